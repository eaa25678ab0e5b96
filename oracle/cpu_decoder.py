"""ORACLE (test infrastructure). fp32 CPU restatement of the decoder the B200
engine runs (the reference has none: its phases are virtual-time charges,
engine.py:251,270,296,358). Same random-init weights (the product's bf16 draw,
upcast to fp32), standard Llama math: RMSNorm, rotate-half RoPE (theta,
fp32 inverse frequencies from a float64 pow, fp32 angle pos*inv_freq), GQA
causal attention, SwiGLU MLP, untied LM head; Qwen3 qk-norm (per-head RMSNorm of q
and k before RoPE) for qk_norm shapes. Each sequence keeps a
contiguous fp32 K/V cache; `forward` appends rows at `start` and returns the
logits of the requested rows. Pinned to HuggingFace transformers' Llama / Qwen3 / GptOss
models on the same weights (tests/test_oracle_vs_hf.py: ~1e-6 relative).

gpt-oss family (config C4, HF GptOss restated): QKV / O biases, per-head attention sinks (an extra
softmax logit with no value row), sliding-window attention on even layers (key j visible from
position p iff p - window < j <= p), YaRN rotary frequencies with cos/sin scaled by the attention
factor, and a routed MoE MLP: router logits + bias, top-k (ties -> lower expert id), softmax over
the selected logits, experts = clamped SwiGLU (gate <= 7, |up| <= 7, (up + 1) * gate *
sigmoid(1.702 gate), gate / up = even / odd rows) with biases, weights MXFP4 — quantised here by
an independent restatement of the OCP MX rule (`mxfp4_roundtrip`) from the same bf16 draws, or,
for the full-size canary, dequantised from the engine's packed tiles (`unpack_mxfp4_tiles`).
"""

from __future__ import annotations

import math
import zlib

import numpy as np
import torch


def draw(shape, seed: int, name: str, norm: bool) -> torch.Tensor:
    """Same generator rule as the product's weights.draw (cpu), upcast to fp32."""
    g = torch.Generator(device="cpu")
    g.manual_seed((seed * 1000003 + zlib.crc32(name.encode())) & 0x7FFFFFFFFFFFFFFF)
    t = torch.randn(shape, generator=g, dtype=torch.float32)
    t = 1.0 + 0.1 * t if norm else 0.02 * t
    return t.to(torch.bfloat16).to(torch.float32)


ROUTE_TIE = 1e-2  # near-tie band of the router arbitration, as a fraction of the token's logit range


class RouteHints:
    """The engine's per-forward expert choices keyed by (rid, start, ids), FIFO per key, built from
    record-mode flights (`Runtime.flights[i]["items"]` / `["routes"]`)."""

    def __init__(self):
        self.q: dict = {}

    def add_flights(self, flights) -> "RouteHints":
        for f in flights:
            if not f.get("routes"):
                continue
            off = 0
            for rid, start, ids, _rows in f["items"]:
                n = len(ids)
                self.q.setdefault((rid, start, tuple(ids)), []).append([r[off:off + n] for r in f["routes"]])
                off += n
        return self

    def take(self, rid, start, ids):
        lst = self.q.get((rid, start, tuple(ids)))
        return lst.pop(0) if lst else None


E2M1 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=np.float32)


def mxfp4_roundtrip(w: torch.Tensor) -> torch.Tensor:
    """OCP MX e2m1 quantise + dequantise of w [N][K] (fp32 values of a bf16 draw), per 32 along K:
    scale 2^e, e = floor(log2(amax)) - 2 clamped to [-13, 12] (amax == 0 -> -13); |v| / 2^e to
    the nearest e2m1 magnitude, a tie to the lower one, saturating at 6; the sign kept for
    non-zero magnitudes. Any torch device (the canary runs it where the weights were drawn)."""
    N, K = w.shape
    x = w.float().reshape(N, K // 32, 32)
    amax = x.abs().amax(-1)
    safe = torch.where(amax > 0, amax, torch.ones_like(amax))
    e = torch.where(amax > 0, torch.floor(torch.log2(safe)) - 2, torch.full_like(amax, -13.0)).clamp(-13, 12)
    v = (x / torch.exp2(e)[..., None]).abs()
    grid = torch.tensor(E2M1, device=w.device)
    # nearest magnitude, ties to the lower: first grid point whose upper midpoint is >= |v|
    mids = (grid[1:] + grid[:-1]) / 2
    idx = (v[..., None] > mids).sum(-1)
    q = grid[idx] * torch.sign(x)
    return (q * torch.exp2(e)[..., None]).reshape(N, K)


def unpack_mxfp4_tiles(tiles: np.ndarray, N: int, K: int) -> np.ndarray:
    """Engine tiles uint8 [NT][K/64][4352] (runtime/weights.py layout: per tile 128 rows x 32
    code bytes, value 2j in the low nibble of byte j, then 128 rows x 2 ue8m0 scale bytes) ->
    fp32 [N][K]."""
    NT, KB = tiles.shape[0], tiles.shape[1]
    codes = tiles[:, :, :4096].reshape(NT, KB, 128, 32)
    scales = tiles[:, :, 4096:].reshape(NT, KB, 128, 2).astype(np.int32) - 127
    lo, hi = codes & 15, codes >> 4
    c = np.stack([lo, hi], axis=-1).reshape(NT, KB, 128, 64)
    mag = E2M1[c & 7] * np.where(c & 8, -1.0, 1.0).astype(np.float32)
    val = mag.reshape(NT, KB, 128, 2, 32) * np.exp2(scales.astype(np.float32))[..., None]
    full = val.reshape(NT, KB, 128, 64).transpose(0, 2, 1, 3).reshape(NT * 128, KB * 64)
    return full[:N].astype(np.float32)


def yarn_inv_freq(d: int, base: float, yarn) -> tuple[torch.Tensor, float]:
    """Rotary inverse frequencies and cos/sin scale (HF `_compute_yarn_parameters`, truncate False,
    float64 then fp32). yarn None: plain theta^(-2i/d), scale 1."""
    pos = np.array([base ** (2.0 * i / d) for i in range(d // 2)], dtype=np.float64)
    if not yarn:
        return torch.tensor((1.0 / pos).astype(np.float32)), 1.0
    factor, bfast, bslow, orig = yarn
    cd = lambda rot: (d * math.log(orig / (rot * 2 * math.pi))) / (2 * math.log(base))  # noqa: E731
    low, high = max(cd(bfast), 0.0), min(cd(bslow), d - 1.0)
    if low == high:
        high += 0.001
    ramp = np.clip((np.arange(d // 2, dtype=np.float64) - low) / (high - low), 0.0, 1.0)
    extra = 1.0 - ramp
    inv = (1.0 / (factor * pos)) * (1.0 - extra) + (1.0 / pos) * extra
    return torch.tensor(inv.astype(np.float32)), float(np.float32(0.1 * math.log(factor) + 1.0))


class CpuDecoder:
    """`source(name, shape, norm)` -> fp32 tensor supplies the weights (default: `draw` on the
    CPU); `stream=True` keeps no layer resident: each forward rebuilds every layer from
    `source` (full-size canaries of shapes whose fp32 weights exceed host memory)."""

    def __init__(self, shape, seed: int = 0, layers: int | None = None, threads: int | None = None,
                 source=None, stream: bool = False, expert_source=None):
        self.s = shape
        # MoE experts: expert_source(layer, e) -> (w_gate_up, b_gate_up, w_down, b_down) fp32,
        # default = the CPU bf16 draw through mxfp4_roundtrip
        self.expert_source = expert_source or (lambda i, e: default_expert(shape, seed, i, e))
        self.L = shape.layers if layers is None else layers
        if threads:
            torch.set_num_threads(threads)
        self.source = source or (lambda name, shp, norm: draw(shp, seed, name, norm))
        self.stream = stream
        self.bf16_points = False
        d, V = shape.d_model, shape.vocab
        self.embed = self.source("embed", (V, d), False)
        self.layers = [] if stream else [self.layer(i) for i in range(self.L)]
        self.fn = self.source("final_norm", (d,), True)
        self.head = self.source("lm_head", (V, d), False)
        half = shape.d_head // 2
        inv = np.array([1.0 / math.pow(shape.rope_theta, 2.0 * i / shape.d_head) for i in range(half)])
        self.inv_freq = torch.tensor(inv.astype(np.float32))
        self.rope_scale = 1.0
        if getattr(shape, "yarn", None):
            self.inv_freq, self.rope_scale = yarn_inv_freq(shape.d_head, shape.rope_theta, shape.yarn)
        self.cache: dict[str, list] = {}
        self.routes: list | None = None  # debug: per MoE layer call, the (experts, weights) chosen
        # near-tie arbitration (parity tests): `route_hints.take(rid, start, ids)` -> per layer the
        # engine's expert ids [n, k]; the oracle adopts the engine's experts for a token only where
        # they differ from its own top-k by a near-tie (`ROUTE_TIE` of the token's logit range) and
        # raises otherwise. Storage rounding upstream of the router (the bf16 attention output, the
        # bf16 norm output) moves router logits by ~1e-3; a tie closer than that is decided by
        # rounding on either side, and following the engine there keeps the comparison meaningful.
        self.route_hints = None
        self.arbitrated = 0       # token-layers where the engine's near-tie choice was adopted
        self.routed = 0           # token-layers routed

    def layer(self, i: int) -> dict:
        s, src = self.s, self.source
        d = s.d_model
        qd, kvd = s.n_q * s.d_head, s.n_kv * s.d_head
        w = {
            "an": src(f"l{i}.attn_norm", (d,), True),
            "qkv": src(f"l{i}.wqkv", (qd + 2 * kvd, d), False),
            "o": src(f"l{i}.wo", (d, qd), False),
            "mn": src(f"l{i}.mlp_norm", (d,), True),
        }
        if not getattr(s, "n_experts", 0):
            w["gu"] = src(f"l{i}.w_gate_up", (2 * s.d_ff, d), False)
            w["dn"] = src(f"l{i}.w_down", (d, s.d_ff), False)
        if s.qk_norm:  # Qwen3: per-head RMSNorm of q and k before RoPE
            w["qn"] = src(f"l{i}.q_norm", (s.d_head,), True)
            w["kn"] = src(f"l{i}.k_norm", (s.d_head,), True)
        if getattr(s, "attn_bias", False):
            w["bqkv"] = src(f"l{i}.bqkv", (qd + 2 * kvd,), False)
            w["bo"] = src(f"l{i}.bo", (d,), False)
        if getattr(s, "sinks", False):
            w["sinks"] = src(f"l{i}.sinks", (s.n_q,), True)
        w["window"] = s.window(i) if hasattr(s, "window") else 0
        if getattr(s, "n_experts", 0):
            w["router"] = src(f"l{i}.router", (s.n_experts, d), False)
            w["router_b"] = src(f"l{i}.router_b", (s.n_experts,), False)
            cache: dict = {}

            def expert(e, i=i, cache=cache):
                if e not in cache:
                    cache[e] = self.expert_source(i, e)
                return cache[e]

            w["expert"] = expert
        return w

    def iter_layers(self):
        if not self.stream:
            yield from enumerate(self.layers)
        else:
            for i in range(self.L):
                yield i, self.layer(i)

    def _norm(self, x, w):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + self.s.rms_eps) * w

    def _qk(self, w, q, k):
        if "qn" in w:
            q, k = self._norm(q, w["qn"]), self._norm(k, w["kn"])
        return q, k

    def _rope(self, x, pos):
        # x [T, H, D]; pos [T]
        ang = pos.to(torch.float32)[:, None] * self.inv_freq[None, :]  # fp32 angle, as on the GPU
        a64 = ang.to(torch.float64)
        c, s = torch.cos(a64).to(torch.float32)[:, None, :], torch.sin(a64).to(torch.float32)[:, None, :]
        if getattr(self, "rope_scale", 1.0) != 1.0:  # YaRN attention factor
            c, s = c * self.rope_scale, s * self.rope_scale
        h = x.shape[-1] // 2
        x1, x2 = x[..., :h], x[..., h:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def truncate(self, rid: str, n: int) -> None:
        if rid in self.cache:
            self.cache[rid] = [(k[:n], v[:n]) for k, v in self.cache[rid]]

    def drop(self, rid: str) -> None:
        self.cache.pop(rid, None)

    def layer_forward(self, w: dict, x: torch.Tensor, pos: torch.Tensor, start: int, kv: tuple, hint=None):
        """One decoder layer: x [T, d] fp32 at absolute positions `pos` (= start..start+T-1), kv =
        this layer's (K, V) cache rows; returns (new x, new kv). Also the per-layer teacher-forced
        check of the full-size canary (tests/test_gpu_canary.py) feeds it the engine's own layer
        inputs."""
        s = self.s
        T = x.shape[0]
        r = (lambda t: t.to(torch.bfloat16).float()) if self.bf16_points else (lambda t: t)
        H, G, D = s.n_q, s.n_kv, s.d_head
        h = r(self._norm(x, w["an"]))
        qkv = h @ w["qkv"].T
        if "bqkv" in w:
            qkv = qkv + w["bqkv"]
        q = qkv[:, : H * D].view(T, H, D)
        k = qkv[:, H * D: (H + G) * D].view(T, G, D)
        v = qkv[:, (H + G) * D:].view(T, G, D)
        q, k = self._qk(w, q, k)
        q, k = self._rope(q, pos), self._rope(k, pos)
        q, k, v = r(q), r(k), r(v)
        kc, vc = kv
        kc = torch.cat([kc[:start], k])
        vc = torch.cat([vc[:start], v])
        n = kc.shape[0]
        rep = H // G
        kk = kc.repeat_interleave(rep, dim=1)  # [n, H, D]
        vv = vc.repeat_interleave(rep, dim=1)
        scores = torch.einsum("thd,nhd->htn", q, kk) / math.sqrt(D)
        keys = torch.arange(n)[None, :]
        mask = keys > pos[:, None]
        if w.get("window", 0):
            mask = mask | (keys <= pos[:, None] - w["window"])
        scores = scores.masked_fill(mask[None], float("-inf"))
        if "sinks" in w:  # the sink logit joins the softmax, its column is dropped
            sink = w["sinks"][:, None, None].expand(H, T, 1)
            p = torch.softmax(torch.cat([scores, sink], dim=-1), dim=-1)[..., :n]
        else:
            p = torch.softmax(scores, dim=-1)
        attn = r(torch.einsum("htn,nhd->thd", p, vv).reshape(T, H * D))
        x = x + attn @ w["o"].T
        if "bo" in w:
            x = x + w["bo"]
        h = r(self._norm(x, w["mn"]))
        if "router" in w:
            x = x + self._moe(w, h, hint)
        else:
            gu = h @ w["gu"].T
            g, u = gu[:, : s.d_ff], gu[:, s.d_ff:]
            x = x + r(torch.nn.functional.silu(g) * u) @ w["dn"].T
        return x, (kc, vc)

    def _moe(self, w: dict, h: torch.Tensor, hint=None) -> torch.Tensor:
        """Routed experts (gpt-oss): top-k of router logits + bias (ties -> lower id, a stable
        sort), softmax over the k, clamped SwiGLU experts with biases, weighted sum in rank order."""
        s = self.s
        T, k, lim = h.shape[0], s.top_k, s.swiglu_limit
        logits = (h @ w["router"].T + w["router_b"]).numpy()
        order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
        self.routed += T
        if hint is not None:
            for t in range(T):
                mine, theirs = set(order[t].tolist()), set(hint[t].tolist())
                if mine == theirs:
                    continue
                kth = float(np.sort(logits[t])[::-1][k - 1])
                tie = ROUTE_TIE * float(logits[t].max() - logits[t].min())
                for e in theirs ^ mine:
                    if abs(float(logits[t, e]) - kth) > tie:
                        raise AssertionError(f"router: engine chose {sorted(theirs)}, oracle {sorted(mine)}; "
                                             f"expert {e} is {float(logits[t, e]) - kth:+.4f} from the k-th logit "
                                             f"(tie band {tie:.4f})")
                chosen = np.array(sorted(theirs, key=lambda e: (-logits[t, e], e)))
                order[t] = chosen
                self.arbitrated += 1
        top = np.take_along_axis(logits, order, axis=1)
        ex = np.exp(top - top[:, :1])
        wts = ex / ex.sum(1, keepdims=True)
        if self.routes is not None:
            self.routes.append((order.copy(), wts.copy(), logits.copy()))
        ys = torch.zeros(T, k, s.d_model)
        for e in np.unique(order):
            tok, rk = np.nonzero(order == e)
            wg, bg, wd, bd = w["expert"](int(e))
            gu = h[torch.tensor(tok)] @ wg.T + bg
            g, u = gu[:, 0::2].clamp(max=lim), gu[:, 1::2].clamp(-lim, lim)
            act = (u + 1) * (g * torch.sigmoid(1.702 * g))
            if self.bf16_points:  # the engine stores the activation as fp16
                act = act.to(torch.float16).float()
            ys[torch.tensor(tok), torch.tensor(rk)] = act @ wd.T + bd
        out = torch.zeros(T, s.d_model)
        wt = torch.tensor(wts, dtype=torch.float32)
        for r_ in range(k):
            out = out + wt[:, r_:r_ + 1] * ys[:, r_]
        return out

    def forward(self, rid: str, ids: list[int], start: int, rows: list[int]) -> torch.Tensor:
        """fp32 forward; with `self.bf16_points` set, values are rounded to bf16 exactly where the
        B200 engine STORES bf16 (GEMM inputs, the rotated q and the K/V cache rows, the attention
        output, the SwiGLU product, the final-norm rows) — all arithmetic stays fp32. That mode
        separates the intrinsic error of bf16 storage (which grows ~sqrt(depth) on the random-init
        models: 0.8% at 1 layer, 3.9% at 32 layers of Llama-3-8B width) from kernel error."""
        s = self.s
        T = len(ids)
        r = (lambda t: t.to(torch.bfloat16).float()) if self.bf16_points else (lambda t: t)
        H, G, D = s.n_q, s.n_kv, s.d_head
        cache = self.cache.setdefault(rid, [(torch.zeros(0, G, D), torch.zeros(0, G, D)) for _ in range(self.L)])
        pos = torch.arange(start, start + T)
        x = self.embed[torch.tensor(ids, dtype=torch.long)]
        hints = self.route_hints.take(rid, start, ids) if self.route_hints is not None else None
        for i, w in self.iter_layers():
            x, cache[i] = self.layer_forward(w, x, pos, start, cache[i], hints[i] if hints else None)
        sel = x[torch.tensor(rows, dtype=torch.long)]
        return r(self._norm(sel, self.fn)) @ self.head.T


def decode_batch(dec: CpuDecoder, caches: list, ids: list[int], positions: list[int]) -> torch.Tensor:
    """One batched decode step (bench CPU baseline only): B sequences, one new token each.

    `caches[b][layer]` = (K, V) fp32 [ctx, n_kv, d]; GEMMs run batched over B (as a CPU
    server would), attention per sequence. Returns logits [B, V]."""
    s = dec.s
    H, G, D = s.n_q, s.n_kv, s.d_head
    B = len(ids)
    pos = torch.tensor(positions)
    x = dec.embed[torch.tensor(ids, dtype=torch.long)]
    for i, w in enumerate(dec.layers):
        h = dec._norm(x, w["an"])
        qkv = h @ w["qkv"].T
        q, k = dec._qk(w, qkv[:, : H * D].view(B, H, D), qkv[:, H * D: (H + G) * D].view(B, G, D))
        q, k = dec._rope(q, pos), dec._rope(k, pos)
        v = qkv[:, (H + G) * D:].view(B, G, D)
        outs = []
        for b in range(B):
            kc, vc = caches[b][i]
            kc = torch.cat([kc, k[b:b + 1]])
            vc = torch.cat([vc, v[b:b + 1]])
            caches[b][i] = (kc, vc)
            kk = kc.repeat_interleave(H // G, dim=1)
            vv = vc.repeat_interleave(H // G, dim=1)
            p = torch.softmax(torch.einsum("hd,nhd->hn", q[b], kk) / math.sqrt(D), dim=-1)
            outs.append(torch.einsum("hn,nhd->hd", p, vv).reshape(H * D))
        x = x + torch.stack(outs) @ w["o"].T
        h = dec._norm(x, w["mn"])
        gu = h @ w["gu"].T
        x = x + (torch.nn.functional.silu(gu[:, : s.d_ff]) * gu[:, s.d_ff:]) @ w["dn"].T
    return dec._norm(x, dec.fn) @ dec.head.T


def default_expert(shape, seed: int, layer: int, e: int):
    """Expert e of `layer` from the CPU bf16 draws (the product's generator rule), MXFP4 round trip."""
    d, f = shape.d_model, shape.d_ff
    p = f"l{layer}.e{e}."
    return (mxfp4_roundtrip(draw((2 * f, d), seed, p + "w_gate_up", False)), draw((2 * f,), seed, p + "b_gate_up", False),
            mxfp4_roundtrip(draw((d, f), seed, p + "w_down", False)), draw((d,), seed, p + "b_down", False))
