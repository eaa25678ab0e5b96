"""The GPU decoder: one forward pass over a packed step of resident sequences.

A step packs T tokens: first the B_dec decode sequences (one token each), then
S append-prefill runs (prefill chunks, verify passes, tool-output ingests),
each a contiguous token range. Per layer:

  rmsnorm -> K5 QKV GEMM -> fused RoPE + K1 commit into the paged pool ->
  K3 decode attention (rows [0, B_dec)) + K2 append-prefill (rows [B_dec, T)) ->
  K5 O GEMM -> residual + rmsnorm -> K5 gate-up GEMM -> SiLU*up -> K5 down GEMM

then the final norm on the R sampled rows only, the K5 LM-head GEMM on those
rows, and script-forced greedy sampling. Everything is launched through the
C ABI on the current torch stream; the only torch ops are buffer allocation
and the metadata H2D copy. Host metadata for a step is one pinned int32
buffer, uploaded with a single async copy.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from ..modelcfg import ModelShape
from . import lib

FORCE_BIAS = 1.0e4  # >> any logit spread of the random-init models (|logit| < 10)


class KVPool:
    """Owner of the library's paged pool + host-side allocator handle."""

    def __init__(self, shape: ModelShape, num_blocks: int, max_slots: int, max_blocks_per_slot: int, device: int = 0):
        self.shape = shape
        self.num_blocks = num_blocks
        self.max_slots = max_slots
        self.max_bps = max_blocks_per_slot
        h = C.c_void_p()
        lib.call("stb_kv_pool_create", device, shape.layers, shape.n_kv, shape.d_head, 16, num_blocks,
                 max_slots, max_blocks_per_slot, C.byref(h))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and lib._lib is not None:
            lib._lib.stb_kv_pool_destroy(h)
            self.h = None

    def reserve(self, slot: int, n: int) -> None:
        lib.call("stb_kv_reserve", self.h, slot, n)

    def truncate(self, slot: int, n: int) -> None:
        lib.call("stb_kv_truncate", self.h, slot, n)

    def release(self, slot: int) -> None:
        lib.call("stb_kv_release", self.h, slot)

    def free_blocks(self) -> int:
        return lib.call("stb_kv_free_blocks", self.h)

    def blocks(self, slot: int) -> list[int]:
        n = lib.call("stb_kv_slot_blocks", self.h, slot, None, 0)
        buf = (C.c_int32 * max(n, 1))()
        lib.call("stb_kv_slot_blocks", self.h, slot, C.cast(buf, C.c_void_p), n)
        return list(buf[:n])

    def sync(self, stream: int) -> None:
        lib.call("stb_kv_sync", self.h, C.c_void_p(stream))

    def layer_ptrs(self, layer: int) -> tuple[int, int]:
        k, v = C.c_void_p(), C.c_void_p()
        lib.call("stb_kv_layer_ptrs", self.h, layer, C.byref(k), C.byref(v))
        return k.value, v.value


@dataclass
class StepBatch:
    """Host description of one packed forward (all arrays int32)."""

    ids: np.ndarray          # [T]
    pos: np.ndarray          # [T] absolute position of each token
    slot_of: np.ndarray      # [T] pool slot of each token's sequence
    dec_slots: np.ndarray    # [B_dec]
    dec_ctx: np.ndarray      # [B_dec] context length incl. the new token
    pre_slots: np.ndarray    # [S]
    pre_qstart: np.ndarray   # [S+1] offsets into the prefill rows
    pre_ctx: np.ndarray      # [S]
    sample_rows: np.ndarray  # [R] rows of the packed step whose logits are sampled
    targets: np.ndarray      # [R] forced ids (-1: unforced)

    @property
    def T(self) -> int:
        return int(self.ids.shape[0])

    @property
    def B_dec(self) -> int:
        return int(self.dec_slots.shape[0])

    @property
    def S(self) -> int:
        return int(self.pre_slots.shape[0])

    @property
    def R(self) -> int:
        return int(self.sample_rows.shape[0])


def _p(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


class Decoder:
    def __init__(self, shape: ModelShape, weights: dict[str, torch.Tensor], pool: KVPool, device: str = "cuda"):
        self.shape = shape
        self.w = weights
        self.pool = pool
        self.device = device
        self.scale = 1.0 / math.sqrt(shape.d_head)
        self._cap_t = 0
        self._cap_r = 0
        self._cap_b = 0
        self.keep_logits = False
        self.timers: dict[str, list] | None = None  # kernel -> [(ev0, ev1, algorithmic bytes|flops)]
        self.last_logits: torch.Tensor | None = None
        self.last_raw_argmax: torch.Tensor | None = None

    # -- buffers ----------------------------------------------------------------

    def _ensure(self, T: int, R: int, B: int) -> None:
        s, dev = self.shape, self.device
        if T > self._cap_t:
            cap = max(T, 2 * self._cap_t, 64)
            f32, bf = torch.float32, torch.bfloat16
            self.x = torch.empty(cap, s.d_model, dtype=f32, device=dev)
            self.h = torch.empty(cap, s.d_model, dtype=bf, device=dev)
            self.qkv = torch.empty(cap, s.q_dim + 2 * s.kv_dim, dtype=f32, device=dev)
            self.q = torch.empty(cap, s.q_dim, dtype=bf, device=dev)
            self.attn = torch.empty(cap, s.q_dim, dtype=bf, device=dev)
            self.proj = torch.empty(cap, s.d_model, dtype=f32, device=dev)
            self.gu = torch.empty(cap, 2 * s.d_ff, dtype=f32, device=dev)
            self.act = torch.empty(cap, s.d_ff, dtype=bf, device=dev)
            self._cap_t = cap
        if R > self._cap_r:
            cap = max(R, 2 * self._cap_r, 16)
            self.rows = torch.empty(cap, s.d_model, dtype=torch.bfloat16, device=dev)
            self.logits = torch.empty(cap, s.vocab, dtype=torch.float32, device=dev)
            self.sampled = torch.empty(cap, dtype=torch.int32, device=dev)
            self.raw_arg = torch.empty(cap, dtype=torch.int32, device=dev)
            self.raw_max = torch.empty(cap, dtype=torch.float32, device=dev)
            self._cap_r = cap
        if B > self._cap_b:
            cap = max(B, 2 * self._cap_b, 16)
            nbytes = lib.load().stb_attn_decode_workspace(cap, s.n_q, s.d_head)
            self.work = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
            self._cap_b = cap

    def _upload(self, b: StepBatch) -> dict[str, torch.Tensor]:
        parts = [("ids", b.ids), ("pos", b.pos), ("slot_of", b.slot_of), ("dec_slots", b.dec_slots),
                 ("dec_ctx", b.dec_ctx), ("pre_slots", b.pre_slots), ("pre_qstart", b.pre_qstart),
                 ("pre_ctx", b.pre_ctx), ("sample_rows", b.sample_rows), ("targets", b.targets)]
        total = sum(int(a.shape[0]) for _, a in parts)
        host = torch.empty(max(total, 1), dtype=torch.int32, pin_memory=True)
        hv = host.numpy()
        off = 0
        spans = {}
        for name, a in parts:
            n = int(a.shape[0])
            hv[off:off + n] = a
            spans[name] = (off, n)
            off += n
        dev = host.to(self.device, non_blocking=True)
        self._pinned = host  # keep alive until the copy lands
        self.h2d_bytes = 4 * total
        return {k: dev[o:o + n] for k, (o, n) in spans.items()}

    # -- forward ----------------------------------------------------------------

    def forward(self, b: StepBatch) -> torch.Tensor:
        """Run one packed step; returns the sampled ids [R] (device int32)."""
        s, w = self.shape, self.w
        T, R, B, S = b.T, b.R, b.B_dec, b.S
        self._ensure(T, R, B)
        stream = torch.cuda.current_stream().cuda_stream
        st = C.c_void_p(stream)
        self.pool.sync(stream)
        m = self._upload(b)
        d = s.d_model
        x, h = self.x[:T], self.h[:T]
        call = lib.call
        call("stb_embed", _p(m["ids"]), _p(w["embed"]), _p(x), T, d, st)
        call("stb_add_rmsnorm", _p(x), None, _p(w["l0.attn_norm"]), _p(h), T, d, s.rms_eps, st)
        max_q = int(np.max(np.diff(b.pre_qstart))) if S else 0
        max_ctx = int(b.dec_ctx.max()) if B else 0
        # K3 algorithmic bytes per launch: every context row's K and V once + q in + out
        dec_bytes = (int(b.dec_ctx.sum()) * 2 * s.kv_dim * 2 + 2 * B * s.q_dim * 2) if B else 0
        for i in range(s.layers):
            self.gemm(h, w[f"l{i}.wqkv"], self.qkv[:T], st)
            call("stb_qkv_rope_commit", self.pool.h, i, _p(self.qkv), _p(self.q), _p(m["slot_of"]), _p(m["pos"]),
                 T, s.n_q, s.rope_theta, st)
            if B:
                ev = self._tick()
                call("stb_attn_decode", self.pool.h, i, _p(self.q), _p(self.attn), _p(m["dec_slots"]),
                     _p(m["dec_ctx"]), B, s.n_q, self.scale, max_ctx, _p(self.work), st)
                self._tock("attn_decode", ev, dec_bytes)
            if S:
                call("stb_attn_prefill", self.pool.h, i, C.c_void_p(self.q[B:].data_ptr()),
                     C.c_void_p(self.attn[B:].data_ptr()), _p(m["pre_slots"]), _p(m["pre_qstart"]),
                     _p(m["pre_ctx"]), S, T - B, s.n_q, self.scale, max_q, st)
            self.gemm(self.attn[:T], w[f"l{i}.wo"], self.proj[:T], st)
            call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w[f"l{i}.mlp_norm"]), _p(h), T, d, s.rms_eps, st)
            self.gemm(h, w[f"l{i}.w_gate_up"], self.gu[:T], st)
            call("stb_silu_mul", _p(self.gu), _p(self.act), T, s.d_ff, st)
            self.gemm(self.act[:T], w[f"l{i}.w_down"], self.proj[:T], st)
            if i + 1 < s.layers:
                call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w[f"l{i + 1}.attn_norm"]), _p(h), T, d,
                     s.rms_eps, st)
            else:  # residual add only; the final norm runs on the sampled rows
                call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w["final_norm"]), None, T, d, s.rms_eps, st)
        rows = self.rows[:R]
        call("stb_gather_rmsnorm", _p(x), _p(m["sample_rows"]), _p(w["final_norm"]), _p(rows), R, d, s.rms_eps, st)
        logits = self.logits[:R]
        self.gemm(rows, w["lm_head"], logits, st)
        call("stb_sample_forced", _p(logits), s.vocab, _p(m["targets"]), R, s.vocab, FORCE_BIAS,
             _p(self.sampled), _p(self.raw_arg), _p(self.raw_max), st)
        if self.keep_logits:
            self.last_logits = logits.clone()
            self.last_raw_argmax = self.raw_arg[:R].clone()
        return self.sampled[:R]

    def _tick(self):
        if self.timers is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def _tock(self, name: str, ev0, work: int) -> None:
        if ev0 is None:
            return
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        self.timers.setdefault(name, []).append((ev0, ev1, work))

    def gemm(self, a: torch.Tensor, wt: torch.Tensor, out: torch.Tensor, st: C.c_void_p) -> None:
        M, K = a.shape
        N = wt.shape[0]
        ev = self._tick()
        lib.call("stb_gemm_bf16", _p(a), a.stride(0), _p(wt), wt.stride(0), _p(out), out.stride(0), M, N, K, 0, st)
        # K5 algorithmic bytes: weights + activations in + fp32 out (HBM-bound when M is small)
        self._tock("gemm", ev, N * K * 2 + M * K * 2 + M * N * 4)
