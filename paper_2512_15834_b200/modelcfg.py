"""Decoder shapes of the benchmark configs.

The reference has no model: its engine charges `rate x tokens` per phase
(`engine.py:251,270,296,358`). The B200 engine runs a random-init decoder of
a named shape so those phases are real GEMMs and paged attention. Weights are
N(0, 0.02) from a seeded generator (`runtime/weights.py`); the oracle builds
the same weights bit-for-bit on the CPU and upcasts them to fp32.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelShape:
    name: str
    layers: int
    d_model: int
    n_q: int
    n_kv: int
    d_head: int
    d_ff: int
    vocab: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    qk_norm: bool = False  # Qwen3: per-head RMSNorm of q and k (weights [d_head]) before RoPE
    # gpt-oss family (config C4). n_experts > 0: the MLP is a routed mixture of experts (router
    # [n_experts][d] + bias, top_k, softmax over the selected logits), each expert a clamped
    # SwiGLU of width d_ff with biases, expert weights stored MXFP4 (e2m1 values, one ue8m0 scale
    # per 32 along K — the released checkpoint's format)
    n_experts: int = 0
    top_k: int = 0
    swiglu_limit: float = 0.0     # gpt-oss: gate <= limit, |up| <= limit, out = (up+1) * gate*sigmoid(1.702 gate)
    sliding_window: int = 0       # > 0: even layers attend to the last `sliding_window` keys only
    sinks: bool = False           # per-head learned logit added to every softmax denominator
    attn_bias: bool = False       # biases on the QKV and O projections
    yarn: tuple | None = None     # (factor, beta_fast, beta_slow, original_max_position): YaRN RoPE

    @property
    def moe(self) -> bool:
        return self.n_experts > 0

    def window(self, layer: int) -> int:
        """Sliding window of `layer` (0 = full causal attention); gpt-oss alternates, layer 0 sliding."""
        return self.sliding_window if (self.sliding_window and layer % 2 == 0) else 0

    @property
    def q_dim(self) -> int:
        return self.n_q * self.d_head

    @property
    def kv_dim(self) -> int:
        return self.n_kv * self.d_head

    @property
    def kv_bytes_per_token(self) -> int:
        """bf16 K+V bytes one token occupies across all layers."""
        return 2 * self.layers * self.kv_dim * 2

    @property
    def expert_bytes(self) -> int:
        """HBM bytes of ONE expert's MXFP4 weights (gate-up + down, N padded to 128 rows): 4 bits
        per value + one scale byte per 32 values."""
        def mx(n, k):
            return -(-n // 128) * 128 * k * 17 // 32
        return mx(2 * self.d_ff, self.d_model) + mx(self.d_model, self.d_ff)

    @property
    def weight_bytes(self) -> int:
        d = self.d_model
        per_layer = d * (self.q_dim + 2 * self.kv_dim) + self.q_dim * d + 2 * d
        per_layer += 2 * self.d_head if self.qk_norm else 0
        if self.moe:
            per_layer += self.n_experts * d  # router
            extra = self.layers * self.n_experts * self.expert_bytes
        else:
            per_layer += 3 * d * self.d_ff
            extra = 0
        return 2 * (self.layers * per_layer + 2 * self.vocab * d + d) + extra

    def with_layers(self, layers: int) -> "ModelShape":
        return replace(self, name=f"{self.name}[L={layers}]", layers=layers)

    def rope_table(self) -> tuple[list[float], float]:
        """(inverse frequencies [d_head/2], cos/sin scale). Plain RoPE: theta^(-2i/d), scale 1.
        YaRN (gpt-oss, HF `_compute_yarn_parameters`, truncate=False): interpolated / extrapolated
        frequencies blended by a linear ramp between the correction dims of beta_fast / beta_slow
        rotations at the original context, cos and sin scaled by 0.1 ln(factor) + 1. All float64,
        rounded to fp32 once (the engine uploads this table; the oracle restates the formula)."""
        d, base = self.d_head, self.rope_theta
        pos_freqs = [base ** (2.0 * i / d) for i in range(d // 2)]
        if not self.yarn:
            return [float(_f32(1.0 / p)) for p in pos_freqs], 1.0
        factor, beta_fast, beta_slow, orig = self.yarn

        def corr_dim(rot):
            return (d * math.log(orig / (rot * 2 * math.pi))) / (2 * math.log(base))

        low, high = max(corr_dim(beta_fast), 0.0), min(corr_dim(beta_slow), d - 1.0)
        if low == high:
            high += 0.001
        inv = []
        for i, p in enumerate(pos_freqs):
            ramp = min(max((i - low) / (high - low), 0.0), 1.0)
            extra = 1.0 - ramp
            inv.append(float(_f32((1.0 / (factor * p)) * (1.0 - extra) + (1.0 / p) * extra)))
        return inv, float(_f32(0.1 * math.log(factor) + 1.0))


def _f32(x: float) -> float:
    import struct

    return struct.unpack("f", struct.pack("f", x))[0]


# C1: the reference CPU run's "tiny random-init decoder (2 layers, d=256)"
TINY = ModelShape("tiny-c1", layers=2, d_model=256, n_q=4, n_kv=2, d_head=64, d_ff=1024, vocab=512)
# C2: Llama-3-8B shape
LLAMA3_8B = ModelShape("llama3-8b", layers=32, d_model=4096, n_q=32, n_kv=8, d_head=128,
                       d_ff=14336, vocab=128256, rope_theta=500000.0)
# C3: Qwen3-32B shape, qk-norm included
QWEN3_32B = ModelShape("qwen3-32b", layers=64, d_model=5120, n_q=64, n_kv=8, d_head=128,
                       d_ff=25600, vocab=151936, rope_theta=1000000.0, rms_eps=1e-6, qk_norm=True)
# C3 family at CPU-oracle size (parity tests): Qwen3 attention geometry (d_head 128, GQA 8,
# qk-norm), two layers
QWEN3_MINI = ModelShape("qwen3-mini", layers=2, d_model=1024, n_q=16, n_kv=2, d_head=128,
                        d_ff=2048, vocab=1024, rope_theta=1000000.0, rms_eps=1e-6, qk_norm=True)

# C4: gpt-oss-120b shape (HF GptOssConfig): 36 layers, d 2880, 64 q heads / 8 kv heads of 64,
# 128 experts top-4 of width 2880 (MXFP4), SWA-128 on alternate layers, attention sinks, QKV / O
# biases, YaRN RoPE (theta 150k, factor 32 over 4096), clamped SwiGLU (limit 7), V = 201,088
GPT_OSS_120B = ModelShape("gpt-oss-120b", layers=36, d_model=2880, n_q=64, n_kv=8, d_head=64, d_ff=2880,
                          vocab=201088, rope_theta=150000.0, rms_eps=1e-5, n_experts=128, top_k=4,
                          swiglu_limit=7.0, sliding_window=128, sinks=True, attn_bias=True,
                          yarn=(32.0, 32.0, 1.0, 4096))
# C4 family at CPU-oracle size (parity tests): same attention geometry (d_head 64, GQA 8, sinks,
# biases, YaRN), a short window so both layer kinds are exercised, 16 experts top-4
GPT_OSS_MINI = ModelShape("gpt-oss-mini", layers=2, d_model=512, n_q=16, n_kv=2, d_head=64, d_ff=256,
                          vocab=1024, rope_theta=150000.0, rms_eps=1e-5, n_experts=16, top_k=4,
                          swiglu_limit=7.0, sliding_window=32, sinks=True, attn_bias=True,
                          yarn=(32.0, 32.0, 1.0, 4096))

SHAPES = {s.name: s for s in (TINY, LLAMA3_8B, QWEN3_32B, QWEN3_MINI, GPT_OSS_120B, GPT_OSS_MINI)}
