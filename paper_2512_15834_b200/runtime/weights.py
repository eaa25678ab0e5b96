"""Deterministic random-init decoder weights (BASELINE configs are random-init).

Every tensor is drawn from its own generator seeded by (seed, tensor name), so
any subset of layers can be rebuilt identically — the oracle rebuilds the
same bf16 values on the CPU and upcasts them to fp32. `device="cpu"` draws on
the CPU (parity runs); `device="cuda"` draws on the GPU (large shapes, where a
CPU draw of 8B values would dominate start-up); both are bf16 in HBM.

Layout (rows = output features, so every projection is X @ W^T, K-major):
  embed [V][d]; per layer: attn_norm [d], wqkv [(n_q+2n_kv)*dh][d] (q rows,
  then k rows, then v rows), q_norm / k_norm [dh] (qk-norm shapes only),
  wo [d][n_q*dh], mlp_norm [d], w_gate_up [2ff][d] (gate rows, then up rows),
  w_down [d][ff]; final_norm [d]; lm_head [V][d].
"""

from __future__ import annotations

import zlib

import torch

from ..modelcfg import ModelShape

STD = 0.02


def _gen(seed: int, name: str, device: str) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1000003 + zlib.crc32(name.encode())) & 0x7FFFFFFFFFFFFFFF)
    return g


def draw(shape: tuple, seed: int, name: str, device: str = "cpu", norm: bool = False) -> torch.Tensor:
    g = _gen(seed, name, device)
    t = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    t = 1.0 + 0.1 * t if norm else STD * t
    return t.to(torch.bfloat16)


def tensor_specs(shape: ModelShape):
    d, V = shape.d_model, shape.vocab
    yield "embed", (V, d), False
    for i in range(shape.layers):
        yield f"l{i}.attn_norm", (d,), True
        yield f"l{i}.wqkv", (shape.q_dim + 2 * shape.kv_dim, d), False
        if shape.qk_norm:
            yield f"l{i}.q_norm", (shape.d_head,), True
            yield f"l{i}.k_norm", (shape.d_head,), True
        yield f"l{i}.wo", (d, shape.q_dim), False
        yield f"l{i}.mlp_norm", (d,), True
        yield f"l{i}.w_gate_up", (2 * shape.d_ff, d), False
        yield f"l{i}.w_down", (d, shape.d_ff), False
    yield "final_norm", (d,), True
    yield "lm_head", (V, d), False


def build(shape: ModelShape, seed: int = 0, init_device: str = "cpu", device: str = "cuda") -> dict[str, torch.Tensor]:
    out = {}
    for name, shp, norm in tensor_specs(shape):
        out[name] = draw(shp, seed, name, init_device, norm).to(device).contiguous()
    return out
