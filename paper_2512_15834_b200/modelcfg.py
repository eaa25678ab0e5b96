"""Decoder shapes of the benchmark configs.

The reference has no model: its engine charges `rate x tokens` per phase
(`engine.py:251,270,296,358`). The B200 engine runs a random-init decoder of
a named shape so those phases are real GEMMs and paged attention. Weights are
N(0, 0.02) from a seeded generator (`runtime/weights.py`); the oracle builds
the same weights bit-for-bit on the CPU and upcasts them to fp32.
"""

from __future__ import annotations

from dataclasses import dataclass


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
    def weight_bytes(self) -> int:
        d = self.d_model
        per_layer = d * (self.q_dim + 2 * self.kv_dim) + self.q_dim * d + 3 * d * self.d_ff + 2 * d
        per_layer += 2 * self.d_head if self.qk_norm else 0
        return 2 * (self.layers * per_layer + 2 * self.vocab * d + d)

    def with_layers(self, layers: int) -> "ModelShape":
        return ModelShape(f"{self.name}[L={layers}]", layers, self.d_model, self.n_q, self.n_kv,
                          self.d_head, self.d_ff, self.vocab, self.rope_theta, self.rms_eps, self.qk_norm)


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

SHAPES = {s.name: s for s in (TINY, LLAMA3_8B, QWEN3_32B, QWEN3_MINI)}
