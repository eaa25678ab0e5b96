"""The GPU decoder: one forward pass over a packed step of resident sequences.

A step packs T tokens: first the B_dec decode sequences (one token each), then
S append-prefill runs (prefill chunks, verify passes, tool-output ingests),
each a contiguous token range. Per layer:

  rmsnorm -> K5 QKV GEMM -> fused (qk-norm +) RoPE + K1 commit into the paged pool ->
  K3 decode attention (rows [0, B_dec)) + K2 append-prefill (rows [B_dec, T)) ->
  K5 O GEMM -> residual + rmsnorm -> K5 gate-up GEMM -> SiLU*up -> K5 down GEMM

(with STB200_FUSED=1: five launches per layer, every row op inside the GEMM that
produces its input; the norm weights are folded into the QKV / gate-up weights once
at load, and the 1/rms of each row — known only after the whole row is reduced —
scales the GEMM's finished sums. Parity-green but measured slower than the default
separate-kernel path: rmsnorm -> QKV -> RoPE+commit -> attention -> O -> add+rmsnorm
-> gate-up [SiLU fused for whole-tile schedules] -> down -> add+rmsnorm.)

then the final norm on the R sampled rows only, the K5 LM-head GEMM on those
rows, and script-forced greedy sampling. Every launch goes through the C ABI
on the current torch stream.

Step metadata (ids, positions, slots, contexts, sample rows, targets) is one
int32 record written into a pinned host buffer and copied with a single H2D
into a static device buffer. Decode-only steps (the common case) replay a
CUDA graph captured once per batch size: all launch parameters of such a step
depend on B alone (the K3 split count is B-derived, GEMM tensor maps point at
static buffers), so the graph is valid for every step of that size.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from ..modelcfg import ModelShape
from . import lib

_NVTX = os.environ.get("STB200_NVTX", "1") != "0"  # one NVTX range per packed step (the phase marks: engine._log)
FORCE_BIAS = 1.0e4  # >> any logit spread of the random-init models (|logit| < 10)
# timing experiments only: comma-separated C-ABI entry points the step does not launch
# (outputs are garbage; tools/profile_step.py uses it to attribute in-step time under PDL)
_SKIP = frozenset(k for k in os.environ.get("STB200_SKIP_KERNELS", "").split(",") if k)
GEMM_C_ZEROED = 1
GEMM_SILU_MUL = 2   # include/stb200.h STB_GEMM_SILU_MUL


def interleave_gate_up(w: torch.Tensor, d_ff: int) -> None:
    """In place: rows [gate_0..gate_F-1, up_0..up_F-1] -> [gate_0, up_0, gate_1, up_1, ...]
    (stb_silu_mul / STB_GEMM_SILU_MUL layout). Idempotent per tensor object (marked, not
    keyed by address: the caching allocator reuses addresses of freed weights)."""
    if getattr(w, "_stb_gate_up_interleaved", False):
        return
    w.copy_(w.view(2, d_ff, -1).transpose(0, 1).reshape(2 * d_ff, -1))
    w._stb_gate_up_interleaved = True   # include/stb200.h STB_GEMM_C_ZEROED
GEMM_W_TILED = 4    # include/stb200.h STB_GEMM_W_TILED
CLEAR_MAX = 256     # consumers clear up to this many rows they read (decode-sized steps)
# Mixed steps (verify passes, small ingests) can be replayed from CUDA graphs too, but their
# shapes keep changing with the batch (B, T, R, max_q), so captures — each a ~10 ms host stall
# the GPU idles through — outnumber the replays that pay them back; measured on C2: no gain
# in the verify steps (their host launch is hidden behind the previous step), 0.25 ms/step of
# device idle from captures. Off by default (STB200_GRAPH_MIXED=1 enables).
GRAPH_MAX_T = 192 if os.environ.get("STB200_GRAPH_MIXED") == "1" else 0
GRAPH_MAX_RUNS = 2
GRAPH_CACHE = 48    # captured graphs kept
PROJECTIONS = ("wqkv", "wo", "w_gate_up", "w_down")
MOE_PROJECTIONS = ("wqkv", "wo", "router")   # gpt-oss: the experts are MXFP4 tiles (weights.MoELayer)
MOE_GATE_UP, MOE_DOWN = 1, 2                 # include/stb200.h STB_MOE_*
# MoE GEMMs on the block-scaled tensor-core path (stb_moe_quant + stb_moe_gemm_mx);
# STB200_MOE_MX=0 keeps the dequantising kernel (stb_moe_gemm_mxfp4) for A/B
from .weights import MOE_MX  # noqa: E402  (the experts' packing follows the same switch)
# STB200_MOE_FUSED_SPLIT=1: the gate-up epilogue splits the down projection's input itself
# (stb_moe_gemm_mx_q) instead of writing fp16 rows for stb_moe_quant — parity-green but slower
# (in-step A/B, profiles/r2n_c4_fused_split_ab.txt: decode 8.83 -> 9.22 ms, a 400-token ingest step
# 19.9 -> 23.4 ms: the per-element byte stores and pair barriers lengthen the epilogue past the
# weight stream), so off by default
MOE_FUSED_SPLIT = os.environ.get("STB200_MOE_FUSED_SPLIT", "0") == "1"
MOE_TILE_BYTES = 4352                        # one 128 x 64 MXFP4 tile (weights.TILE_BYTES)


class _MoeWork:
    """Algorithmic HBM bytes of one grouped-GEMM launch, known only after the step ran: the
    touched experts' MXFP4 tiles (every weight byte once) + the token rows in + the rows out.
    Evaluated by Decoder.fold from the per-layer expert offsets the step copied to pinned memory."""

    __slots__ = ("host", "layer", "N", "K", "rows", "in_b", "out_b")

    def __init__(self, host, layer, N, K, rows, in_b, out_b):
        self.host, self.layer, self.N, self.K, self.rows, self.in_b, self.out_b = host, layer, N, K, rows, in_b, out_b

    def __call__(self) -> int:
        offs = self.host[self.layer].numpy()
        touched = int(np.count_nonzero(np.diff(offs)))
        w = touched * (-(-self.N // 128)) * (self.K // 64) * MOE_TILE_BYTES
        n_out = self.N // 2 if self.out_b == 2 else self.N   # gate-up emits N/2 fp16 activations
        return w + self.rows * self.K * self.in_b + self.rows * n_out * self.out_b


class GemmEpi(C.Structure):
    """include/stb200.h stb_gemm_epi."""

    _fields_ = [("kind", C.c_int), ("ss_in", C.c_void_p), ("ss_parts", C.c_int), ("inv_dim", C.c_float),
                ("eps", C.c_float),
                ("out", C.c_void_p), ("ldo", C.c_int64), ("x", C.c_void_p), ("ldx", C.c_int64),
                ("ss_out", C.c_void_p), ("pool", C.c_void_p), ("layer", C.c_int), ("n_q", C.c_int),
                ("slot_of", C.c_void_p), ("pos_of", C.c_void_p), ("rope_theta", C.c_float),
                ("q_norm", C.c_void_p), ("k_norm", C.c_void_p), ("qk_eps", C.c_float)]


EPI_SILU, EPI_QKV, EPI_RESID = 1, 2, 3   # include/stb200.h STB_EPI_*


class BlockOp(C.Structure):
    """include/stb200.h stb_block_op: one phase of a decode-block chain (stb_gemm_block)."""

    _fields_ = [("kind", C.c_int), ("x", C.c_void_p), ("ldx", C.c_int64), ("w", C.c_void_p), ("c", C.c_void_p),
                ("ldc", C.c_int64), ("n", C.c_int), ("k", C.c_int), ("x_res", C.c_void_p), ("y", C.c_void_p),
                ("eps", C.c_float), ("pool", C.c_void_p), ("layer", C.c_int), ("n_q", C.c_int),
                ("slot_of", C.c_void_p), ("pos_of", C.c_void_p), ("rope_theta", C.c_float),
                ("q_norm", C.c_void_p), ("k_norm", C.c_void_p)]


OP_GEMM, OP_NORM, OP_SILU, OP_ROPE = 1, 2, 3, 4   # include/stb200.h STB_OP_*
# Decode block (stb_gemm_block, opt-in STB200_GEMM_BLOCK=1): decode-only steps of dense models
# as [attention, block] per layer, the O / gate-up / down / next QKV projections and the row ops
# between them in one launch with grid barriers. Parity-green but measured slower than the
# PDL-chained per-op launches (C2 decode step at ctx 2k 4.93 -> 5.5-6.2 ms): a grid barrier plus a
# row-op phase costs 6-7 us where a programmatic-dependent kernel boundary plus the row kernel
# costs 3-4, and merging two GEMMs into one launch saves nothing.
BLOCK_MAX_T = 64 if os.environ.get("STB200_GEMM_BLOCK", "0") == "1" else 0


def fusable(shape: ModelShape) -> bool:
    """The fused QKV epilogue needs 128-aligned q / kv widths and d_head <= 128."""
    return shape.d_head in (32, 64, 128) and shape.q_dim % 128 == 0 and shape.kv_dim % 128 == 0


def fold_norm(w: torch.Tensor, g: torch.Tensor) -> None:
    """In place: W[n][k] <- bf16(W[n][k] * g[k]) (fp32 product): the RMSNorm weight of the
    GEMM's input folded into the GEMM (the fused epilogue applies only 1/rms)."""
    w.copy_((w.float() * g.float()[None, :]).to(w.dtype))


class TiledWeight:
    """A projection weight re-laid out once by stb_weight_tile: each 128 x 64 tile one
    contiguous, pre-swizzled 16 KiB block, so every GEMM pipeline stage is a single
    linear bulk copy of whole DRAM pages (STB_GEMM_W_TILED)."""

    __slots__ = ("t", "N", "K")

    def __init__(self, w: torch.Tensor):
        self.N, self.K = int(w.shape[0]), int(w.shape[1])
        self.t = torch.empty(lib.load().stb_weight_tiled_elems(self.N, self.K), dtype=torch.bfloat16,
                             device=w.device)
        lib.call("stb_weight_tile", C.c_void_p(w.data_ptr()), w.stride(0), self.N, self.K,
                 C.c_void_p(self.t.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))

    def data_ptr(self) -> int:
        return self.t.data_ptr()


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
        self.log: list | None = None  # record mode: every allocator op, for an oracle replay

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and lib._lib is not None:
            lib._lib.stb_kv_pool_destroy(h)
            self.h = None

    def reserve(self, slot: int, n: int) -> None:
        lib.call("stb_kv_reserve", self.h, slot, n)
        if self.log is not None:
            self.log.append(("reserve", slot, n))

    def truncate(self, slot: int, n: int) -> None:
        lib.call("stb_kv_truncate", self.h, slot, n)
        if self.log is not None:
            self.log.append(("truncate", slot, n))

    def release(self, slot: int) -> None:
        lib.call("stb_kv_release", self.h, slot)
        if self.log is not None:
            self.log.append(("release", slot, 0))

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
    # multi-query K3 entries (filled by Decoder._forward, not by the caller): packed first row and
    # query count of every K3 entry — decode rows first, then the short runs folded into K3
    dec_qrow: np.ndarray | None = None
    dec_nq: np.ndarray | None = None

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


FIELDS = ("ids", "pos", "slot_of", "dec_slots", "dec_ctx", "pre_slots", "pre_qstart", "pre_ctx", "sample_rows",
          "targets", "dec_qrow", "dec_nq")
# Short runs (verify passes: the last sampled token + the draft) ride in the decode attention
# launch as multi-query K3 entries (stb_attn_decode_mq: 16 / group queries per 16-row tile)
# instead of a separate K2 launch + split merge — when every run of the step has at most this
# many queries and the model has plain attention (no sliding window, no sinks).
# STB200_MQ_MAX=0 keeps them on K2.
MQ_MAX_N = int(os.environ.get("STB200_MQ_MAX", "40"))
MQ_MIN_DECODE = 16  # decode rows the step must carry for its short runs to ride in K3
# K3 partition computed once per step (layer 0) and reused by the later layers; STB200_K3_PLAN=0
# has every launch compute its own
K3_PLAN = os.environ.get("STB200_K3_PLAN", "1") != "0"


_EMPTY_I32 = np.zeros(0, dtype=np.int32)


def _p(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t if isinstance(t, int) else t.data_ptr())


class Decoder:
    META_CAP = 1 << 20  # int32 entries of the static step record

    def __init__(self, shape: ModelShape, weights: dict[str, torch.Tensor], pool: KVPool, device: str = "cuda",
                 use_graphs: bool = True):
        self.shape = shape
        self.w = weights
        for i in range(shape.layers if not shape.moe else 0):
            gu = weights[f"l{i}.w_gate_up"]
            if not isinstance(gu, TiledWeight):  # (gate, up) pairs in adjacent rows: fused SiLU epilogue
                interleave_gate_up(gu, shape.d_ff)
            del gu
        # fused epilogues: correct (tests/test_gpu_parity.py) but measured slower on B200 — the
        # epilogue's global round trips sit on the GEMM's critical path; opt in
        self.fused = os.environ.get("STB200_FUSED", "") == "1" and fusable(shape) and not shape.moe
        # projections in the tiled HBM layout (once; a shared dict is converted in place —
        # the first Decoder over a dict decides whether the norm weights are folded in)
        if "_stb_fused" not in weights:
            weights["_stb_fused"] = self.fused
            for i in range(shape.layers):
                if self.fused:
                    fold_norm(weights[f"l{i}.wqkv"], weights[f"l{i}.attn_norm"])
                    fold_norm(weights[f"l{i}.w_gate_up"], weights[f"l{i}.mlp_norm"])
        self.fused = bool(weights["_stb_fused"])
        projections = MOE_PROJECTIONS if shape.moe else PROJECTIONS
        for name in [f"l{i}.{p}" for i in range(shape.layers) for p in projections] + ["lm_head"]:
            if not isinstance(weights[name], TiledWeight):
                weights[name] = TiledWeight(weights[name])
        # rotary table (YaRN for gpt-oss: frequencies + cos/sin scale, modelcfg.rope_table)
        self.rope_inv, self.rope_scale = None, 1.0
        if shape.yarn:
            inv, self.rope_scale = shape.rope_table()
            self.rope_inv = torch.tensor(inv, dtype=torch.float32, device=device)
        self.pool = pool
        self.device = device
        self.scale = 1.0 / math.sqrt(shape.d_head)
        self._cap_t = self._cap_r = self._cap_b = 0
        self.keep_logits = False
        self.use_graphs = use_graphs
        self.graphs: dict[tuple, tuple] = {}
        self.graph_sizes: dict[tuple, int] = {}  # kernels captured per graph
        self._seen: set = set()                  # mixed-step shapes already run eagerly once
        self.timers: dict[str, list] | None = None  # name -> [ms, work, launches] totals
        self.timer_filter: set | None = None  # time only these kernel classes (None: all)
        self._pre_flops = 0
        self._pre_work = (0, 0)  # (flops, bytes) of one K2 launch: verify runs are HBM-bound, ingests tensor-bound
        self._pre_work_win = (0, 0)  # the same on a sliding-window layer
        self._dec_bytes_win = 0      # K3's algorithmic bytes on a sliding-window layer
        self._pre_units = 0
        self.run_log: list | None = None
        self._pending: list | None = []             # (name, ev0, ev1, work) awaiting a sync
        self._graph_timed = False
        self.last_logits: torch.Tensor | None = None
        self.last_raw_argmax: torch.Tensor | None = None
        # double-buffered pinned step records: the runtime keeps one step in flight, so the
        # record of step k+1 is written while step k's upload may still be pending
        self.meta_host = [torch.empty(self.META_CAP, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self.meta_ev: list = [None, None]
        self.meta_flip = 0
        self.meta_dev = torch.empty(self.META_CAP, dtype=torch.int32, device=device)
        self.h2d_bytes = 0
        self.graph_replays = 0
        self.graph_kernels = 0   # kernels launched by graph replays (captured launches x replays)
        self._timed_parity = 0
        self.step_events: list | None = None  # (ev0, ev1, graphed, T) bracketing each step's kernels
        # leading rows of each GEMM output that may be non-zero (rows at and past it are zero)
        self._dirty = {"qkv": 0, "proj": 0, "gu": 0, "logits": 0}
        self._stream_cache: dict = {}
        self._blk_cache: dict = {}   # (T, buffers, metadata pointers) -> decode-block op arrays
        self._mq_B = 0               # K3 entries of the current step when its short runs ride in K3
        self.last_step_tokens = 0
        self.taps: list | None = None  # debug (canary): residual stream after the embedding and each layer
        # MoE routing statistics for the grouped GEMM's algorithmic bytes: each timed step copies the
        # per-layer expert offsets to pinned memory (4 buffers: eager / graph x 2 flight parities)
        self._moe_host = None
        self._moe_flip = 0
        self.route_log: list | None = None  # debug / parity: per layer, the step's expert ids [T*k] (device)

    # -- buffers ----------------------------------------------------------------

    def _ensure(self, T: int, R: int, B: int) -> None:
        s, dev = self.shape, self.device
        if T > self._cap_t:
            cap = max(T, 2 * self._cap_t, 64)
            f32, bf = torch.float32, torch.bfloat16
            self.x = torch.empty(cap, s.d_model, dtype=f32, device=dev)
            self.h = torch.empty(cap, s.d_model, dtype=bf, device=dev)
            # GEMM outputs start zeroed and are cleared by their consumers, so decode-shaped
            # (stream-K) GEMMs accumulate into them with no memset (see _dirty)
            self.qkv = torch.zeros(cap, s.q_dim + 2 * s.kv_dim, dtype=f32, device=dev)
            self.q = torch.empty(cap, s.q_dim, dtype=bf, device=dev)
            self.attn = torch.empty(cap, s.q_dim, dtype=bf, device=dev)
            self.proj = torch.zeros(cap, s.d_model, dtype=f32, device=dev)
            self.gu = torch.zeros(cap, 2 * s.d_ff, dtype=f32, device=dev)
            self.act = torch.empty(cap, s.d_ff, dtype=bf, device=dev)
            # fused path: per-row partial sums of squares (one per 128-feature tile of d) of
            # every norm input (2 per layer + 1)
            self.ss = torch.zeros(2 * s.layers + 1, cap, -(-s.d_model // 512) * 4, dtype=f32, device=dev)
            if s.moe:  # routed rows: T * top_k, plus one token tile of TMA overhang
                rows = cap * s.top_k + 64
                i32 = torch.int32
                self.rlog = torch.zeros(cap, s.n_experts, dtype=f32, device=dev)
                self.m_counts = torch.zeros(s.n_experts, dtype=i32, device=dev)   # zero at rest
                self.m_expert = torch.empty(cap * s.top_k, dtype=i32, device=dev)
                self.m_rank = torch.empty(cap * s.top_k, dtype=i32, device=dev)
                self.m_wt = torch.empty(cap * s.top_k, dtype=f32, device=dev)
                self.m_perm = torch.empty(cap * s.top_k, dtype=i32, device=dev)
                self.m_offs = torch.zeros(s.layers, s.n_experts + 1, dtype=i32, device=dev)
                self.m_x = torch.zeros(rows, s.d_model, dtype=torch.float16, device=dev)
                self.m_act = torch.zeros(rows, s.d_ff, dtype=torch.float16, device=dev)
                self.m_y = torch.empty(rows, s.d_model, dtype=f32, device=dev)
                if MOE_MX:  # e4m3 hi / lo halves + scale words of the gate-up input, and of the down
                    # input (written by the gate-up epilogue while the gate-up GEMM still reads the first)
                    kq = max(s.d_model, s.d_ff)
                    L = lib.load()
                    self.m_xq = torch.zeros(L.stb_moe_quant_bytes(rows, kq), dtype=torch.uint8, device=dev)
                    self.m_xsf = torch.zeros(L.stb_moe_quant_scale_words(rows, kq), dtype=torch.int32, device=dev)
                    self.m_aq = torch.zeros(L.stb_moe_quant_bytes(rows, s.d_ff), dtype=torch.uint8, device=dev)
                    self.m_asf = torch.zeros(L.stb_moe_quant_scale_words(rows, s.d_ff), dtype=torch.int32,
                                             device=dev)
                self._moe_rows = rows
            self._cap_t = cap
            self._dirty.update(qkv=0, proj=0, gu=0)
            self.graphs.clear()  # captured graphs point at the old buffers
            self._blk_cache.clear()
        if R > self._cap_r:
            cap = max(R, 2 * self._cap_r, 64)
            self.rows = torch.empty(cap, s.d_model, dtype=torch.bfloat16, device=dev)
            self.logits = torch.zeros(cap, s.vocab, dtype=torch.float32, device=dev)
            self.sampled = torch.empty(cap, dtype=torch.int32, device=dev)
            self.raw_arg = torch.empty(cap, dtype=torch.int32, device=dev)
            self.raw_max = torch.empty(cap, dtype=torch.float32, device=dev)
            self._cap_r = cap
            self._dirty["logits"] = 0
            self.graphs.clear()
        if B > self._cap_b:
            cap = max(B, 2 * self._cap_b, 64)
            nbytes = lib.load().stb_attn_decode_workspace(cap, s.n_q, s.n_kv, s.d_head)
            # zeroed once: the tail holds K3's merge tickets, which every launch leaves zero
            self.work = torch.zeros(-(-nbytes // 4), dtype=torch.float32, device=dev)
            self._cap_b = cap
            self.graphs.clear()

    def _upload(self, b: StepBatch) -> dict[str, int]:
        """Write the step record into pinned memory, one async H2D into the static buffer."""
        k = self.meta_flip
        self.meta_flip ^= 1
        if self.meta_ev[k] is not None:
            self.meta_ev[k].synchronize()
        hv = self.meta_host[k].numpy()
        off, spans = 0, {}
        for name in FIELDS:
            a = getattr(b, name)
            if a is None:
                a = _EMPTY_I32
            n = int(a.shape[0])
            hv[off:off + n] = a
            spans[name] = off
            off += n
        if off > self.META_CAP:
            raise ValueError("step record exceeds the static metadata buffer")
        self.meta_dev[:off].copy_(self.meta_host[k][:off], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.meta_ev[k] = ev
        self.h2d_bytes = 4 * off
        base = self.meta_dev.data_ptr()
        return {k: base + 4 * o for k, o in spans.items()}

    # -- forward ----------------------------------------------------------------

    def forward(self, b: StepBatch) -> torch.Tensor:
        """Run one packed step; returns the sampled ids [R] (device int32)."""
        if _NVTX:
            torch.cuda.nvtx.range_push(f"step T={b.T} decode={b.B_dec} runs={b.S}")
        try:
            return self._forward(b)
        finally:
            if _NVTX:
                torch.cuda.nvtx.range_pop()

    def _mq_entries(self, b: StepBatch) -> StepBatch | None:
        """Fold the step's short runs into K3 as multi-query entries (MQ_MAX_N): entry j of a run of
        n queries holds queries [QE j, min(QE (j+1), n)) at packed rows B + q_start + QE j, QE = 16 /
        group; decode rows are single-query entries. None when the step keeps K2."""
        s = self.shape
        if not (b.S and MQ_MAX_N and not s.moe and not s.sinks and not s.sliding_window):
            return None
        n = np.diff(b.pre_qstart)
        # the folded entries re-read their run's pages from L2 ceil(n / QE) times: worth it when the
        # launch is dominated by decode rows (measured: B=31 + a 33-query run 62 us vs 76 us for K3 +
        # K2; a lone run 55 us vs 21 us on K2)
        if int(n.max()) > MQ_MAX_N or b.B_dec < MQ_MIN_DECODE:
            return None
        qe = 16 // (s.n_q // s.n_kv)
        B = b.B_dec
        slots, ctxs, rows, nqs = [b.dec_slots], [b.dec_ctx], [np.arange(B, dtype=np.int32)], [np.ones(B, np.int32)]
        for i in range(b.S):
            ni, c = int(n[i]), int(b.pre_ctx[i])
            j = np.arange(0, ni, qe, dtype=np.int32)
            nq = np.minimum(qe, ni - j).astype(np.int32)
            slots.append(np.full(len(j), b.pre_slots[i], np.int32))
            ctxs.append((c - ni + j + nq).astype(np.int32))
            rows.append((B + int(b.pre_qstart[i]) + j).astype(np.int32))
            nqs.append(nq)
        return dataclasses.replace(b, dec_slots=np.concatenate(slots), dec_ctx=np.concatenate(ctxs),
                                   dec_qrow=np.concatenate(rows), dec_nq=np.concatenate(nqs))

    def _forward(self, b: StepBatch) -> torch.Tensor:
        T, R, B, S = b.T, b.R, b.B_dec, b.S
        self.last_step_tokens = T
        dec_bytes = (int(b.dec_ctx.sum()) * 2 * self.shape.kv_dim * 2 + 2 * B * self.shape.q_dim * 2) if B else 0
        # sliding-window layers (gpt-oss, every other layer) read only the last `window` keys
        W = self.shape.sliding_window
        self._dec_bytes_win = ((int(np.minimum(b.dec_ctx, W).sum()) * 2 * self.shape.kv_dim * 2
                                + 2 * B * self.shape.q_dim * 2) if B else 0) if W else dec_bytes
        mq = self._mq_entries(b)
        self._mq_B = 0
        if mq is not None:
            # K3's algorithmic bytes gain each folded run's K/V once (its entries re-read them from
            # L2) plus its q and o rows
            n = np.diff(b.pre_qstart)
            dec_bytes += int(np.sum(b.pre_ctx)) * 2 * self.shape.kv_dim * 2 + int(np.sum(n)) * 2 * self.shape.q_dim * 2
            self._mq_B = int(mq.dec_slots.shape[0])
            b = mq
        self._ensure(T, R, max(B, self._mq_B))
        stream = torch.cuda.current_stream().cuda_stream
        self.pool.sync(stream)
        m = self._upload(b)
        max_q = int(np.max(np.diff(b.pre_qstart))) if S else 0
        if S:  # K2 algorithmic flops per layer: 4 H_q d (n ctx_prev + n(n+1)/2) per run
            n = np.diff(b.pre_qstart).astype(np.float64)
            prev = b.pre_ctx.astype(np.float64) - n
            self._pre_flops = int(4 * self.shape.q_dim * float(np.sum(n * prev + n * (n + 1) / 2)))
            # algorithmic bytes: every run's K/V read once plus its q and o rows
            pre_bytes = int(np.sum(b.pre_ctx)) * 2 * self.shape.kv_dim * 2 + int(np.sum(n)) * 2 * self.shape.q_dim * 2
            self._pre_work = (self._pre_flops, pre_bytes)
            if W:  # a window layer: query at position p attends min(p + 1, W) keys; keys read once
                pos = [prev_i + np.arange(n_i) for prev_i, n_i in zip(prev, n)]
                keys = sum(int(np.minimum(p_ + 1, W).sum()) for p_ in pos)
                kread = int(np.sum(np.minimum(b.pre_ctx, n + W - 1)))
                self._pre_work_win = (int(4 * self.shape.q_dim * keys),
                                      kread * 2 * self.shape.kv_dim * 2 + int(np.sum(n)) * 2 * self.shape.q_dim * 2)
            else:
                self._pre_work_win = self._pre_work
            # K2 work units holding queries: (query-tile pair of 2*128/G tokens, kv head, run)
            pair = 2 * 128 // (self.shape.n_q // self.shape.n_kv)
            self._pre_units = int(np.sum(np.ceil(n / pair))) * self.shape.n_kv
            if self.run_log is not None:  # (n, ctx) of every K2 run of the step (diagnostics)
                self.run_log.append([(int(a), int(c)) for a, c in zip(n, b.pre_ctx)])
        # CUDA graphs: decode-only steps (one per batch size) and small mixed steps (verify
        # passes: the same (B, T, R, S, max_q) shape recurs every few steps), whose ~300
        # eager launches would otherwise be paced by the host
        graphable = (self.use_graphs and B > 0 and not self.keep_logits
                     and (S == 0 or (T <= GRAPH_MAX_T and S <= GRAPH_MAX_RUNS)))
        e0 = torch.cuda.Event(enable_timing=True) if self.step_events is not None else None
        shape_key = (B, T, R, S, max_q, self._mq_B)
        if graphable and S > 0 and shape_key not in self._seen:
            # first occurrence of a mixed-step shape runs eagerly (it also initialises every
            # launch's one-time state); the graph is captured, without a warm-up run, only
            # when the shape recurs
            self._seen.add(shape_key)
            graphable = False
        if not graphable:
            if e0 is not None:
                e0.record()
            self._launch(m, T, R, B, S, max_q, int(b.dec_ctx.max()) if len(b.dec_ctx) else 0, dec_bytes)
        else:
            # decode graphs assume (and leave) zeroed every GEMM output they accumulate into
            # (stream-K); a whole-tile LM head overwrites the logits, so those stay as they are
            V, d = self.shape.vocab, self.shape.d_model
            lm_stream = self._stream_cache.get((R, V, d))
            if lm_stream is None:
                lm_stream = self._stream_cache[(R, V, d)] = bool(lib.load().stb_gemm_is_stream(R, V, d))
            timed = self.timers is not None
            # timed graphs carry their own event nodes: two copies alternate so a step's
            # events are not re-recorded while the runtime still has that step in flight
            par = 0
            if timed:
                par = self._timed_parity
                self._timed_parity ^= 1
            key = (B, T, R, S, max_q, timed, par, self._mq_B)
            if key not in self.graphs:
                if len(self.graphs) >= GRAPH_CACHE:  # drop the oldest mixed-step graph
                    old = next((k for k in self.graphs if k[3] > 0), None)
                    if old is not None:
                        del self.graphs[old]
                self._capture(key, m, T, R, B, S, max_q, dec_bytes, warm=S == 0)
            graph, events = self.graphs[key]
            if e0 is not None:  # after any capture: host-side capture time is not device work
                e0.record()
            for name, rows in self._dirty.items():  # part of the step: inside the timed bracket
                if rows and (name != "logits" or lm_stream):
                    getattr(self, name)[:rows].zero_()
                    self._dirty[name] = 0
            graph.replay()
            self.graph_replays += 1
            self.graph_kernels += self.graph_sizes.get(key, 0)
            if timed:
                live = {"attn_decode": (dec_bytes, self._dec_bytes_win),
                        "attn_prefill": (self._pre_work, self._pre_work_win)}
                seen: dict = {}
                for name, a0, a1, work in events:
                    if name in live:  # one launch per layer, in layer order
                        layer = seen.get(name, 0)
                        seen[name] = layer + 1
                        work = live[name][1 if self.shape.window(layer) else 0]
                    self._pending.append((name, a0, a1, work))
        if self.step_events is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            self.step_events.append((e0, e1, S == 0, T))  # (.., decode-only step, tokens)
        if self.keep_logits:
            self.last_logits = self.logits[:R].clone()
            self.logits[:R].zero_()
            self._dirty["logits"] = 0
            self.last_raw_argmax = self.raw_arg[:R].clone()
        return self.sampled[:R]

    def _capture(self, key, m: dict[str, int], T: int, R: int, B: int, S: int, max_q: int, dec_bytes: int,
                 warm: bool = True) -> None:
        timed = key[5]
        saved, saved_timers = self._pending, self.timers
        self.timers, self._pending = None, []
        if warm:
            # warm once eagerly (first-call allocations, tensor-map encodes, attributes); untimed.
            # It runs the step's kernels for real: KV commits are idempotent and the replay
            # overwrites every output
            self._launch(m, T, R, B, S, max_q, 0, dec_bytes)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        events: list = []
        self._pending = events
        self._graph_timed = timed
        n0 = lib.load().stb_launch_count()
        with torch.cuda.graph(graph):
            self._launch(m, T, R, B, S, max_q, 0, dec_bytes)
        self.graph_sizes[key] = int(lib.load().stb_launch_count() - n0)
        self._pending, self.timers = saved, saved_timers
        self._graph_timed = False
        self.graphs[key] = (graph, events)

    def _launch(self, m: dict[str, int], T: int, R: int, B: int, S: int, max_q: int, max_ctx: int,
                dec_bytes: int) -> None:
        if self.shape.moe:
            return self._launch_moe(m, T, R, B, S, max_q, max_ctx, dec_bytes)
        if self.fused:
            return self._launch_fused(m, T, R, B, S, max_q, max_ctx, dec_bytes)
        if S == 0 and T == B and T <= BLOCK_MAX_T and not _SKIP:
            for name in ("qkv", "proj", "gu"):  # the block's stream-K phases accumulate into zeroed rows
                if self._dirty[name]:
                    getattr(self, name)[:self._dirty[name]].zero_()
                    self._dirty[name] = 0
            return self._launch_blocks(m, T, R, B, max_ctx, dec_bytes)
        s, w = self.shape, self.w
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        d = s.d_model
        x, h = self.x, self.h
        call = lib.call if not _SKIP else (lambda name, *a: None if name in _SKIP else lib.call(name, *a))
        for _ in range(2):  # empty pairs: the timers' own overhead, subtracted by the reader
            self._tock("event_overhead", self._tick("event_overhead"), 0)
        call("stb_embed", _p(m["ids"]), _p(w["embed"]), _p(x), T, d, st)
        call("stb_add_rmsnorm", _p(x), None, _p(w["l0.attn_norm"]), _p(h), T, d, s.rms_eps, 0, st)
        clr = T if T <= CLEAR_MAX else 0
        if self.taps is not None:
            self.taps.append(x[:T].clone())
        for i in range(s.layers):
            self.gemm(h[:T], w[f"l{i}.wqkv"], "qkv", st, "wqkv")
            if s.qk_norm:
                call("stb_qkv_norm_rope_commit", self.pool.h, i, _p(self.qkv), _p(self.q), _p(m["slot_of"]),
                     _p(m["pos"]), T, s.n_q, s.rope_theta, _p(w[f"l{i}.q_norm"]), _p(w[f"l{i}.k_norm"]), s.rms_eps,
                     clr, st)
            else:
                call("stb_qkv_rope_commit", self.pool.h, i, _p(self.qkv), _p(self.q), _p(m["slot_of"]),
                     _p(m["pos"]), T, s.n_q, s.rope_theta, clr, st)
            self._cleared("qkv", clr)
            self._attention(call, m, i, T, B, S, max_q, max_ctx, dec_bytes, st)
            self.gemm(self.attn[:T], w[f"l{i}.wo"], "proj", st, "wo")
            call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w[f"l{i}.mlp_norm"]), _p(h), T, d, s.rms_eps, clr, st)
            self._cleared("proj", clr)
            if not self.gemm(h[:T], w[f"l{i}.w_gate_up"], "gu", st, "w_gate_up", fuse_silu=True):
                call("stb_silu_mul", _p(self.gu), _p(self.act), T, s.d_ff, clr, st)
                self._cleared("gu", clr)
            self.gemm(self.act[:T], w[f"l{i}.w_down"], "proj", st, "w_down")
            if i + 1 < s.layers:
                call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w[f"l{i + 1}.attn_norm"]), _p(h), T, d,
                     s.rms_eps, clr, st)
            else:  # residual add only; the final norm runs on the sampled rows
                call("stb_add_rmsnorm", _p(x), _p(self.proj), _p(w["final_norm"]), None, T, d, s.rms_eps, clr, st)
            self._cleared("proj", clr)
            if self.taps is not None:
                self.taps.append(x[:T].clone())
        rows = self.rows[:R]
        call("stb_gather_rmsnorm", _p(x), _p(m["sample_rows"]), _p(w["final_norm"]), _p(rows), R, d, s.rms_eps, st)
        self.gemm(rows, w["lm_head"], "logits", st, "lm_head")
        # the sampler re-zeroes the logits only when the LM head accumulated them (stream-K);
        # whole-tile LM heads (any decode batch) overwrite them with plain stores
        clear = 0 if self.keep_logits or not self._stream_cache[(R, s.vocab, d)] else 1
        call("stb_sample_forced", _p(self.logits), s.vocab, _p(m["targets"]), R, s.vocab, FORCE_BIAS,
             _p(self.sampled), _p(self.raw_arg), _p(self.raw_max), clear, st)
        if clear:
            self._cleared("logits", R)

    def _block_ops(self, m: dict[str, int], T: int) -> list:
        """The decode-block chains of one decode step (stb_gemm_block op arrays), built once per
        (T, buffer set, step-record pointers): [norm, QKV_0, RoPE_0] before the first attention,
        then per layer i [O_i, norm, gate-up_i, SiLU, down_i, norm, QKV_{i+1}, RoPE_{i+1}] (the
        last layer ends with the residual add). Returns [(ops array, n_ops, algorithmic bytes)]."""
        key = (T, m["slot_of"], m["pos"], self.x.data_ptr(), self.qkv.data_ptr(), self.h.data_ptr())
        hit = self._blk_cache.get(key)
        if hit is not None:
            return hit
        s, w = self.shape, self.w
        d = s.d_model
        x, h = self.x, self.h

        def gemm(a, wt, out):
            return BlockOp(kind=OP_GEMM, x=a.data_ptr(), ldx=a.stride(0), w=wt.data_ptr(), c=out.data_ptr(),
                           ldc=out.stride(0), n=wt.N, k=wt.K), wt.N * wt.K * 2 + T * wt.K * 2 + T * wt.N * 4

        def norm(delta, weight, y):
            return BlockOp(kind=OP_NORM, c=delta.data_ptr() if delta is not None else None,
                           w=weight.data_ptr() if weight is not None else None, n=d, x_res=x.data_ptr(),
                           y=y.data_ptr() if y is not None else None, eps=s.rms_eps), 0

        def rope(i):
            qn = w[f"l{i}.q_norm"].data_ptr() if s.qk_norm else None
            kn = w[f"l{i}.k_norm"].data_ptr() if s.qk_norm else None
            return BlockOp(kind=OP_ROPE, c=self.qkv.data_ptr(), y=self.q.data_ptr(), pool=self.pool.h, layer=i,
                           n_q=s.n_q, slot_of=m["slot_of"], pos_of=m["pos"], rope_theta=s.rope_theta, q_norm=qn,
                           k_norm=kn, eps=s.rms_eps), 0

        def qkv(i):
            return [norm(None if i == 0 else self.proj, w[f"l{i}.attn_norm"], h),
                    gemm(h[:T], w[f"l{i}.wqkv"], self.qkv), rope(i)]

        chains = [qkv(0)]
        for i in range(s.layers):
            ops = [gemm(self.attn[:T], w[f"l{i}.wo"], self.proj), norm(self.proj, w[f"l{i}.mlp_norm"], h),
                   gemm(h[:T], w[f"l{i}.w_gate_up"], self.gu),
                   (BlockOp(kind=OP_SILU, c=self.gu.data_ptr(), y=self.act.data_ptr(), n=s.d_ff), 0),
                   gemm(self.act[:T], w[f"l{i}.w_down"], self.proj)]
            if i + 1 < s.layers:
                ops += qkv(i + 1)
            else:
                ops.append(norm(self.proj, None, None))  # residual add only (the final norm: sampled rows)
            chains.append(ops)
        out = []
        for ops in chains:
            arr = (BlockOp * len(ops))(*[o for o, _ in ops])
            out.append((arr, len(ops), sum(b for _, b in ops)))
        if len(self._blk_cache) > 64:
            self._blk_cache.clear()
        self._blk_cache[key] = out
        return out

    def _launch_blocks(self, m: dict[str, int], T: int, R: int, B: int, max_ctx: int, dec_bytes: int) -> None:
        """A decode-only step as 2 launches per layer: attention (K3) and one decode block."""
        s, w = self.shape, self.w
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        d = s.d_model
        call = lib.call
        for _ in range(2):  # empty pairs: the timers' own overhead, subtracted by the reader
            self._tock("event_overhead", self._tick("event_overhead"), 0)
        call("stb_embed", _p(m["ids"]), _p(w["embed"]), _p(self.x), T, d, st)
        chains = self._block_ops(m, T)
        if self.taps is not None:
            self.taps.append(self.x[:T].clone())

        def block(k):
            arr, n, nbytes = chains[k]
            ev = self._tick()
            call("stb_gemm_block", C.cast(arr, C.c_void_p), n, T, st)
            self._tock("gemm_decode", ev, nbytes)

        block(0)
        for i in range(s.layers):
            ev = self._tick("attn_decode")
            call("stb_attn_decode", self.pool.h, i, _p(self.q), _p(self.attn), _p(m["dec_slots"]), _p(m["dec_ctx"]),
                 B, s.n_q, self.scale, max_ctx, _p(self.work), st)
            self._tock("attn_decode", ev, dec_bytes)
            block(i + 1)
            if self.taps is not None:
                self.taps.append(self.x[:T].clone())
        rows = self.rows[:R]
        call("stb_gather_rmsnorm", _p(self.x), _p(m["sample_rows"]), _p(w["final_norm"]), _p(rows), R, d, s.rms_eps,
             st)
        self.gemm(rows, w["lm_head"], "logits", st, "lm_head")
        clear = 0 if self.keep_logits or not self._stream_cache[(R, s.vocab, d)] else 1
        call("stb_sample_forced", _p(self.logits), s.vocab, _p(m["targets"]), R, s.vocab, FORCE_BIAS,
             _p(self.sampled), _p(self.raw_arg), _p(self.raw_max), clear, st)
        if clear:
            self._cleared("logits", R)

    def _launch_moe(self, m: dict[str, int], T: int, R: int, B: int, S: int, max_q: int, max_ctx: int,
                    dec_bytes: int) -> None:
        """gpt-oss family (config C4), per layer: rmsnorm -> QKV GEMM -> bias + YaRN RoPE + K1
        commit -> K3 / K2 with the layer's sliding window and sinks -> O GEMM -> + bias, residual,
        rmsnorm -> router GEMM -> route -> gather -> MXFP4 gate-up (clamped SwiGLU) -> MXFP4 down
        -> weighted combine + residual + the next rmsnorm (moe.cu)."""
        s, w = self.shape, self.w
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        d, E, k = s.d_model, s.n_experts, s.top_k
        x, h = self.x, self.h
        call = lib.call if not _SKIP else (lambda name, *a: None if name in _SKIP else lib.call(name, *a))
        for _ in range(2):
            self._tock("event_overhead", self._tick("event_overhead"), 0)
        call("stb_embed", _p(m["ids"]), _p(w["embed"]), _p(x), T, d, st)
        call("stb_add_rmsnorm", _p(x), None, _p(w["l0.attn_norm"]), _p(h), T, d, s.rms_eps, 0, st)
        clr = T if T <= CLEAR_MAX else 0
        if self.taps is not None:
            self.taps.append(x[:T].clone())
        rows = T * k
        timed = self.timers is not None or self._graph_timed
        offs_host = None
        if timed:
            if self._moe_host is None:
                self._moe_host = [torch.empty(s.layers, E + 1, dtype=torch.int32, pin_memory=True) for _ in range(4)]
            if self._graph_timed:
                slot = self._timed_parity  # graphs: the capture's parity (key[6])
            else:
                self._moe_flip ^= 1
                slot = 2 + self._moe_flip
            offs_host = self._moe_host[slot]
        inv = _p(self.rope_inv) if self.rope_inv is not None else None
        for i in range(s.layers):
            self.gemm(h[:T], w[f"l{i}.wqkv"], "qkv", st, "wqkv")
            call("stb_qkv_rope_commit_ex", self.pool.h, i, _p(self.qkv), _p(self.q), _p(m["slot_of"]), _p(m["pos"]),
                 T, s.n_q, s.rope_theta, inv, C.c_float(self.rope_scale),
                 _p(w.get(f"l{i}.bqkv")), clr, st)
            self._cleared("qkv", clr)
            win, sinks = s.window(i), _p(w.get(f"l{i}.sinks"))
            if B:
                ev = self._tick("attn_decode")
                call("stb_attn_decode_ex", self.pool.h, i, _p(self.q), _p(self.attn), _p(m["dec_slots"]),
                     _p(m["dec_ctx"]), B, s.n_q, self.scale, max_ctx, win, sinks, _p(self.work), st)
                self._tock("attn_decode", ev, self._dec_bytes_win if win else dec_bytes)
            if S:
                ev = self._tick("attn_prefill")
                call("stb_attn_prefill_ex", self.pool.h, i, _p(self.q[B:].data_ptr()), _p(self.attn[B:].data_ptr()),
                     _p(m["pre_slots"]), _p(m["pre_qstart"]), _p(m["pre_ctx"]), S, T - B, s.n_q, self.scale, max_q,
                     self._pre_units, win, sinks, st)
                self._tock("attn_prefill", ev, self._pre_work_win if win else self._pre_work)
            self.gemm(self.attn[:T], w[f"l{i}.wo"], "proj", st, "wo")
            call("stb_add_bias_rmsnorm", _p(x), _p(self.proj), _p(w.get(f"l{i}.bo")), _p(w[f"l{i}.mlp_norm"]), _p(h),
                 T, d, s.rms_eps, clr, st)
            self._cleared("proj", clr)
            # router: fp32 logits, zeroed by the GEMM itself (flags 0)
            rt_w = w[f"l{i}.router"]
            ev = self._tick()
            if "stb_gemm_bf16" not in _SKIP:
                lib.call("stb_gemm_bf16", _p(h), h.stride(0), _p(rt_w), 0, _p(self.rlog), self.rlog.stride(0), T, E, d,
                         0, GEMM_W_TILED, st)
            self._tock("gemm_decode" if T <= 128 else "gemm_prefill", ev,
                       E * d * 2 + T * d * 2 + T * E * 4 if T <= 128 else 2 * T * E * d)
            call("stb_moe_route", _p(self.rlog), self.rlog.stride(0), _p(w[f"l{i}.router_b"]), T, E, k,
                 _p(self.m_counts), _p(self.m_expert), _p(self.m_rank), _p(self.m_wt), st)
            if self.route_log is not None:
                self.route_log.append(self.m_expert[:rows].clone())
            offs = self.m_offs[i]
            ex = w[f"l{i}.experts"]
            cap_r = self._moe_rows
            if MOE_MX:  # block-scaled tensor-core path: the gather splits the rows into e4m3 halves
                call("stb_moe_gather_mx", _p(h), h.stride(0), T, d, k, E, _p(self.m_counts), _p(self.m_expert),
                     _p(self.m_rank), _p(offs), _p(self.m_perm), cap_r, _p(self.m_xq), _p(self.m_xsf), st)
                ev = self._tick()
                # the epilogue splits the SwiGLU rows into the down projection's e4m3 halves itself
                fuse = MOE_FUSED_SPLIT and s.d_ff % 64 == 0
                call("stb_moe_gemm_mx_q", _p(self.m_xq), _p(self.m_xsf), cap_r, _p(ex.gate_up), _p(ex.b_gate_up),
                     _p(self.m_counts), E, 2 * s.d_ff, d, MOE_GATE_UP, C.c_float(s.swiglu_limit),
                     None if fuse else _p(self.m_act), self.m_act.stride(0), rows,
                     _p(self.m_aq) if fuse else None, _p(self.m_asf) if fuse else None, cap_r, st)
            else:
                call("stb_moe_gather", _p(h), h.stride(0), T, d, k, E, _p(self.m_counts), _p(self.m_expert),
                     _p(self.m_rank), _p(offs), _p(self.m_perm), _p(self.m_x), st)
                ev = self._tick()
                call("stb_moe_gemm_mxfp4", _p(self.m_x), cap_r, _p(ex.gate_up), _p(ex.b_gate_up),
                     _p(self.m_counts), E, 2 * s.d_ff, d, MOE_GATE_UP, C.c_float(s.swiglu_limit), _p(self.m_act),
                     self.m_act.stride(0), rows, st)
            self._tock("moe_gemm", ev, _MoeWork(offs_host, i, 2 * s.d_ff, d, rows, 2, 2) if timed else 0)
            if MOE_MX:
                if not fuse:
                    call("stb_moe_quant", _p(self.m_act), self.m_act.stride(0), rows, s.d_ff, cap_r, _p(self.m_aq),
                         _p(self.m_asf), st)
                ev = self._tick()
                call("stb_moe_gemm_mx", _p(self.m_aq), _p(self.m_asf), cap_r, _p(ex.down), _p(ex.b_down),
                     _p(self.m_counts), E, d, s.d_ff, MOE_DOWN, C.c_float(0.0), _p(self.m_y), self.m_y.stride(0),
                     rows, st)
            else:
                ev = self._tick()
                call("stb_moe_gemm_mxfp4", _p(self.m_act), cap_r, _p(ex.down), _p(ex.b_down),
                     _p(self.m_counts), E, d, s.d_ff, MOE_DOWN, C.c_float(0.0), _p(self.m_y), self.m_y.stride(0),
                     rows, st)
            self._tock("moe_gemm", ev, _MoeWork(offs_host, i, d, s.d_ff, rows, 2, 4) if timed else 0)
            last = i + 1 == s.layers
            call("stb_moe_combine", _p(x), _p(self.m_y), T, d, k, _p(self.m_perm), _p(self.m_wt),
                 None if last else _p(w[f"l{i + 1}.attn_norm"]), None if last else _p(h), s.rms_eps,
                 _p(self.m_counts), E, st)
            if self.taps is not None:
                self.taps.append(x[:T].clone())
        if offs_host is not None:
            offs_host.copy_(self.m_offs, non_blocking=True)
        rows_b = self.rows[:R]
        call("stb_gather_rmsnorm", _p(x), _p(m["sample_rows"]), _p(w["final_norm"]), _p(rows_b), R, d, s.rms_eps, st)
        self.gemm(rows_b, w["lm_head"], "logits", st, "lm_head")
        clear = 0 if self.keep_logits or not self._stream_cache[(R, s.vocab, d)] else 1
        call("stb_sample_forced", _p(self.logits), s.vocab, _p(m["targets"]), R, s.vocab, FORCE_BIAS,
             _p(self.sampled), _p(self.raw_arg), _p(self.raw_max), clear, st)
        if clear:
            self._cleared("logits", R)

    def _attention(self, call, m, i: int, T: int, B: int, S: int, max_q: int, max_ctx: int, dec_bytes: int, st):
        s = self.shape
        # K3's work partition depends only on the step's entries: layer 0 computes and stores it,
        # the later layers load it (plan_mode 1 / 2, stb_attn_decode_planned)
        plan = (1 if i == 0 else 2) if K3_PLAN else 0
        if self._mq_B:  # decode rows + the step's short runs in one multi-query K3 launch
            ev = self._tick("attn_decode")
            call("stb_attn_decode_planned", self.pool.h, i, _p(self.q), _p(self.attn), _p(m["dec_slots"]),
                 _p(m["dec_ctx"]), _p(m["dec_qrow"]), _p(m["dec_nq"]), self._mq_B, s.n_q, self.scale, max_ctx,
                 plan, _p(self.work), st)
            self._tock("attn_decode", ev, dec_bytes)
            return
        if B:
            ev = self._tick("attn_decode")
            call("stb_attn_decode_planned", self.pool.h, i, _p(self.q), _p(self.attn), _p(m["dec_slots"]),
                 _p(m["dec_ctx"]), None, None, B, s.n_q, self.scale, max_ctx, plan, _p(self.work), st)
            self._tock("attn_decode", ev, dec_bytes)
        if S:
            ev = self._tick("attn_prefill")
            call("stb_attn_prefill_split", self.pool.h, i, _p(self.q[B:].data_ptr()), _p(self.attn[B:].data_ptr()),
                 _p(m["pre_slots"]), _p(m["pre_qstart"]), _p(m["pre_ctx"]), S, T - B, s.n_q, self.scale, max_q,
                 self._pre_units, st)
            self._tock("attn_prefill", ev, self._pre_work)

    def _launch_fused(self, m: dict[str, int], T: int, R: int, B: int, S: int, max_q: int, max_ctx: int,
                      dec_bytes: int) -> None:
        """Five launches per layer; row ops live in the GEMM epilogues (module docstring)."""
        s, w = self.shape, self.w
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        d = s.d_model
        x, xb, ss = self.x, self.h, self.ss
        ld_ss = ss.stride(0)
        call = lib.call if not _SKIP else (lambda name, *a: None if name in _SKIP else lib.call(name, *a))
        for _ in range(2):  # empty pairs: the timers' own overhead, subtracted by the reader
            self._tock("event_overhead", self._tick("event_overhead"), 0)
        parts = ss.shape[2]
        call("stb_embed_prep", _p(m["ids"]), _p(w["embed"]), _p(x), _p(xb), _p(ss), parts, T, d, st)
        inv_d = 1.0 / d
        ss_at = lambda j: ss.data_ptr() + 4 * j * ld_ss  # noqa: E731
        for i in range(s.layers):
            e = GemmEpi(kind=EPI_QKV, ss_in=ss_at(2 * i), ss_parts=parts, inv_dim=inv_d, eps=s.rms_eps,
                        out=self.q.data_ptr(), ldo=self.q.stride(0), pool=self.pool.h.value, layer=i, n_q=s.n_q, slot_of=m["slot_of"],
                        pos_of=m["pos"], rope_theta=s.rope_theta,
                        q_norm=w[f"l{i}.q_norm"].data_ptr() if s.qk_norm else None,
                        k_norm=w[f"l{i}.k_norm"].data_ptr() if s.qk_norm else None, qk_eps=s.rms_eps)
            self.gemm_fused(xb[:T], w[f"l{i}.wqkv"], self.qkv, e, st, "wqkv")
            self._attention(call, m, i, T, B, S, max_q, max_ctx, dec_bytes, st)
            e = GemmEpi(kind=EPI_RESID, out=xb.data_ptr(), ldo=xb.stride(0), x=x.data_ptr(), ldx=x.stride(0),
                        ss_out=ss_at(2 * i + 1), ss_parts=parts)
            self.gemm_fused(self.attn[:T], w[f"l{i}.wo"], self.proj, e, st, "wo")
            e = GemmEpi(kind=EPI_SILU, ss_in=ss_at(2 * i + 1), ss_parts=parts, inv_dim=inv_d, eps=s.rms_eps,
                        out=self.act.data_ptr(), ldo=self.act.stride(0))
            self.gemm_fused(xb[:T], w[f"l{i}.w_gate_up"], self.gu, e, st, "w_gate_up")
            e = GemmEpi(kind=EPI_RESID, out=xb.data_ptr(), ldo=xb.stride(0), x=x.data_ptr(), ldx=x.stride(0),
                        ss_out=ss_at(2 * i + 2), ss_parts=parts)
            self.gemm_fused(self.act[:T], w[f"l{i}.w_down"], self.proj, e, st, "w_down")
        rows = self.rows[:R]
        call("stb_gather_rmsnorm", _p(x), _p(m["sample_rows"]), _p(w["final_norm"]), _p(rows), R, d, s.rms_eps, st)
        self.gemm(rows, w["lm_head"], "logits", st, "lm_head")
        clear = 0 if self.keep_logits or not self._stream_cache[(R, s.vocab, d)] else 1
        call("stb_sample_forced", _p(self.logits), s.vocab, _p(m["targets"]), R, s.vocab, FORCE_BIAS,
             _p(self.sampled), _p(self.raw_arg), _p(self.raw_max), clear, st)
        if clear:
            self._cleared("logits", R)

    def gemm_fused(self, a: torch.Tensor, wt: "TiledWeight", work: torch.Tensor, epi: GemmEpi, st, tag: str):
        """K5 with a fused epilogue; `work` is a zeroed fp32 accumulator the kernel leaves zeroed."""
        M, K = a.shape
        N = wt.N
        if "stb_gemm_bf16_fused" in _SKIP or f"gemm:{tag}" in _SKIP:
            return
        ev = self._tick()
        lib.call("stb_gemm_bf16_fused", _p(a), a.stride(0), _p(wt), 0, _p(work), work.stride(0), M, N, K,
                 GEMM_W_TILED, C.byref(epi), st)
        if ev is not None:
            if M <= 128:
                self._tock("gemm_decode", ev, N * K * 2 + M * K * 2 + M * N * 4)
            else:
                self._tock("gemm_prefill", ev, 2 * M * N * K)

    def _cleared(self, name: str, rows: int) -> None:
        if rows >= self._dirty[name]:
            self._dirty[name] = 0

    # -- timing (CUDA events on the launching stream; graph-safe) ----------------

    def _tick(self, name: str | None = None):
        if self.timers is None and not self._graph_timed:
            return None
        if self.timer_filter is not None and name not in self.timer_filter:
            return None
        ev = torch.cuda.Event(enable_timing=True, external=True)
        ev.record()
        return ev

    def _tock(self, name: str, ev0, work: int) -> None:
        if ev0 is None:
            return
        ev1 = torch.cuda.Event(enable_timing=True, external=True)
        ev1.record()
        self._pending.append((name, ev0, ev1, work))

    def take_pending(self) -> list:
        """Detach the event pairs of the step just launched (completed later)."""
        pend, self._pending = self._pending, []
        return pend

    def fold(self, pending: list, sink: dict | None = None) -> None:
        """Fold finished event pairs into `sink` (default `timers`) after their step synchronised."""
        sink = self.timers if sink is None else sink
        if sink is not None:
            for name, e0, e1, work in pending:
                if callable(work):  # known after the step (MoE: the touched experts)
                    work = work()
                t = sink.setdefault(name, [0.0, 0, 0])
                ms = e0.elapsed_time(e1)
                t[0] += ms
                t[2] += 1
                if isinstance(work, tuple):  # (flops, bytes): per-launch list for a max(tensor, hbm) roofline
                    t[1] += work[0]
                    sink.setdefault(name + ":launches", []).append((ms, *work))
                else:
                    t[1] += work

    def collect(self) -> None:
        self.fold(self.take_pending())

    def gemm(self, a: torch.Tensor, wt: torch.Tensor, out_name: str, st: C.c_void_p, tag: str = "",
             fuse_silu: bool = False) -> bool:
        """Launch K5; returns True when the SiLU-gate epilogue was fused (output in self.act)."""
        M, K = a.shape
        N = wt.N
        key = (M, N, K)
        stream = self._stream_cache.get(key)
        if stream is None:
            stream = self._stream_cache[key] = bool(lib.load().stb_gemm_is_stream(M, N, K))
        fused = fuse_silu and not stream  # whole tiles: the epilogue sees finished sums
        if fused:
            out, flags = self.act[:M], GEMM_SILU_MUL
        else:
            out = getattr(self, out_name)[:M]
            flags = GEMM_C_ZEROED if (stream and self._dirty[out_name] == 0) else 0
        if "stb_gemm_bf16" in _SKIP or f"gemm:{tag}" in _SKIP:
            return fused
        ev = self._tick()
        lib.call("stb_gemm_bf16", _p(a), a.stride(0), _p(wt), 0, _p(out), out.stride(0), M, N, K, 0,
                 flags | GEMM_W_TILED, st)
        if not fused:
            self._dirty[out_name] = max(self._dirty[out_name], M)
        if M <= 128:  # decode-shaped: HBM-bound on the weights; work = algorithmic bytes
            self._tock("gemm_decode", ev, N * K * 2 + M * K * 2 + M * N * 4)
        else:  # prefill / ingest: tensor-bound; work = FLOPs
            self._tock("gemm_prefill", ev, 2 * M * N * K)
        return fused
