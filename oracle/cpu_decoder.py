"""ORACLE (test infrastructure). fp32 CPU restatement of the decoder the B200
engine runs (the reference has none: its phases are virtual-time charges,
engine.py:251,270,296,358). Same random-init weights (the product's bf16 draw,
upcast to fp32), standard Llama math: RMSNorm, rotate-half RoPE (theta,
fp32 inverse frequencies from a float64 pow, fp32 angle pos*inv_freq), GQA
causal attention, SwiGLU MLP, untied LM head; Qwen3 qk-norm (per-head RMSNorm of q
and k before RoPE) for qk_norm shapes. Each sequence keeps a
contiguous fp32 K/V cache; `forward` appends rows at `start` and returns the
logits of the requested rows.
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


class CpuDecoder:
    """`source(name, shape, norm)` -> fp32 tensor supplies the weights (default: `draw` on the
    CPU); `stream=True` keeps no layer resident: each forward rebuilds every layer from
    `source` (full-size canaries of shapes whose fp32 weights exceed host memory)."""

    def __init__(self, shape, seed: int = 0, layers: int | None = None, threads: int | None = None,
                 source=None, stream: bool = False):
        self.s = shape
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
        self.cache: dict[str, list] = {}

    def layer(self, i: int) -> dict:
        s, src = self.s, self.source
        d = s.d_model
        qd, kvd = s.n_q * s.d_head, s.n_kv * s.d_head
        w = {
            "an": src(f"l{i}.attn_norm", (d,), True),
            "qkv": src(f"l{i}.wqkv", (qd + 2 * kvd, d), False),
            "o": src(f"l{i}.wo", (d, qd), False),
            "mn": src(f"l{i}.mlp_norm", (d,), True),
            "gu": src(f"l{i}.w_gate_up", (2 * s.d_ff, d), False),
            "dn": src(f"l{i}.w_down", (d, s.d_ff), False),
        }
        if s.qk_norm:  # Qwen3: per-head RMSNorm of q and k before RoPE
            w["qn"] = src(f"l{i}.q_norm", (s.d_head,), True)
            w["kn"] = src(f"l{i}.k_norm", (s.d_head,), True)
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
        h = x.shape[-1] // 2
        x1, x2 = x[..., :h], x[..., h:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def truncate(self, rid: str, n: int) -> None:
        if rid in self.cache:
            self.cache[rid] = [(k[:n], v[:n]) for k, v in self.cache[rid]]

    def drop(self, rid: str) -> None:
        self.cache.pop(rid, None)

    def layer_forward(self, w: dict, x: torch.Tensor, pos: torch.Tensor, start: int, kv: tuple):
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
        mask = torch.arange(n)[None, :] > pos[:, None]
        scores = scores.masked_fill(mask[None], float("-inf"))
        p = torch.softmax(scores, dim=-1)
        attn = r(torch.einsum("htn,nhd->thd", p, vv).reshape(T, H * D))
        x = x + attn @ w["o"].T
        h = r(self._norm(x, w["mn"]))
        gu = h @ w["gu"].T
        g, u = gu[:, : s.d_ff], gu[:, s.d_ff:]
        x = x + r(torch.nn.functional.silu(g) * u) @ w["dn"].T
        return x, (kc, vc)

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
        for i, w in self.iter_layers():
            x, cache[i] = self.layer_forward(w, x, pos, start, cache[i])
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
