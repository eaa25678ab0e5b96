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

MoE shapes (gpt-oss, config C4) replace the MLP with: router [E][d] + router_b [E]; per expert
j: e{j}.w_gate_up [2ff][d] (rows interleaved gate_0, up_0, gate_1, ... as in gpt-oss'
gate_up_proj[..., ::2] / [..., 1::2]) + e{j}.b_gate_up [2ff], e{j}.w_down [d][ff] + e{j}.b_down
[d]; and attention biases bqkv [(n_q+2n_kv)*dh], bo [d], sinks [n_q]. Expert weights are drawn
bf16 like every other tensor and stored MXFP4 (`quantize_mxfp4`, the released checkpoint's
format: SURVEY H7) in the tiled layout the grouped GEMM streams (`pack_mxfp4_tiles`).
"""

from __future__ import annotations

import zlib

import os

import numpy as np

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
    """Every dense tensor (name, shape, norm-like); MoE expert tensors are in `expert_specs`."""
    d, V = shape.d_model, shape.vocab
    qkv = shape.q_dim + 2 * shape.kv_dim
    yield "embed", (V, d), False
    for i in range(shape.layers):
        yield f"l{i}.attn_norm", (d,), True
        yield f"l{i}.wqkv", (qkv, d), False
        if shape.attn_bias:
            yield f"l{i}.bqkv", (qkv,), False
            yield f"l{i}.bo", (d,), False
        if shape.sinks:
            yield f"l{i}.sinks", (shape.n_q,), True
        if shape.qk_norm:
            yield f"l{i}.q_norm", (shape.d_head,), True
            yield f"l{i}.k_norm", (shape.d_head,), True
        yield f"l{i}.wo", (d, shape.q_dim), False
        yield f"l{i}.mlp_norm", (d,), True
        if shape.moe:
            yield f"l{i}.router", (shape.n_experts, d), False
            yield f"l{i}.router_b", (shape.n_experts,), False
        else:
            yield f"l{i}.w_gate_up", (2 * shape.d_ff, d), False
            yield f"l{i}.w_down", (d, shape.d_ff), False
    yield "final_norm", (d,), True
    yield "lm_head", (V, d), False


def expert_specs(shape: ModelShape, layer: int, e: int):
    d, f = shape.d_model, shape.d_ff
    p = f"l{layer}.e{e}."
    return ((p + "w_gate_up", (2 * f, d)), (p + "b_gate_up", (2 * f,)), (p + "w_down", (d, f)), (p + "b_down", (d,)))


# ---------------------------------------------------------------- MXFP4 (OCP MX, e2m1 + ue8m0 / 32)
E2M1 = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)
_MID = (0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0)
SCALE_EXP_MIN, SCALE_EXP_MAX = -13, 12  # keeps every e2m1 x 2^e a normal fp16 (the GEMM's operand type)
TILE_ROWS, TILE_K = 128, 64
TILE_BYTES = TILE_ROWS * TILE_K // 2 + TILE_ROWS * TILE_K // 32  # 4096 B of codes + 256 B of scales


def quantize_mxfp4(w: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """w [N][K] (K % 32 == 0) -> (codes uint8 [N][K] in 0..15: sign << 3 | e2m1 magnitude index,
    scale exponents int8 [N][K/32]). Per 32-value block along K: e = floor(log2(amax)) - 2 (the e2m1
    emax), clamped to [-13, 12] (an all-zero block takes -13); values / 2^e rounded to the nearest
    e2m1 magnitude (a value exactly between two takes the lower), saturating at 6."""
    N, K = w.shape
    x = w.float().reshape(N, K // 32, 32)
    amax = x.abs().amax(-1)
    e = torch.floor(torch.log2(torch.where(amax > 0, amax, torch.ones_like(amax)))) - 2
    e = torch.where(amax > 0, e, torch.full_like(e, SCALE_EXP_MIN)).clamp(SCALE_EXP_MIN, SCALE_EXP_MAX)
    v = x / torch.exp2(e)[..., None]
    mid = torch.tensor(_MID, dtype=torch.float32, device=w.device)
    mag = torch.bucketize(v.abs(), mid, right=False).to(torch.uint8)  # mid[i-1] < |v| <= mid[i] -> i
    sign = ((v < 0) & (mag > 0)).to(torch.uint8) << 3
    return (mag | sign).reshape(N, K), e.to(torch.int8)


def dequantize_mxfp4(codes: torch.Tensor, exps: torch.Tensor) -> torch.Tensor:
    lut = torch.tensor(E2M1, dtype=torch.float32, device=codes.device)
    v = lut[(codes & 7).long()] * torch.where((codes & 8) > 0, -1.0, 1.0)
    N, K = codes.shape
    return (v.reshape(N, K // 32, 32) * torch.exp2(exps.float())[..., None]).reshape(N, K)


def pack_mxfp4_tiles(codes: torch.Tensor, exps: torch.Tensor) -> torch.Tensor:
    """(codes [N][K], exps [N][K/32]) -> uint8 [ceil(N/128)][K/64][4352]: tile (n, k) = 128 rows x 64
    values as [128 rows][32 bytes] (byte j of a row: value 2j in the low nibble, 2j+1 in the high)
    followed by [128 rows][2] ue8m0 scale bytes (exponent + 127); rows past N are zero. One tile is
    one pipeline stage of stb_moe_gemm_mxfp4: a single linear bulk copy."""
    N, K = codes.shape
    if K % TILE_K:
        raise ValueError("MXFP4 tiles need K % 64 == 0")
    NT, KB = -(-N // TILE_ROWS), K // TILE_K
    c = torch.zeros(NT * TILE_ROWS, K, dtype=torch.uint8, device=codes.device)
    c[:N] = codes
    s = torch.full((NT * TILE_ROWS, K // 32), SCALE_EXP_MIN + 127, dtype=torch.uint8, device=codes.device)
    s[:N] = (exps.to(torch.int16) + 127).to(torch.uint8)
    byte = c[:, 0::2] | (c[:, 1::2] << 4)                                      # [NT*128][K/2]
    byte = byte.reshape(NT, TILE_ROWS, KB, 32).permute(0, 2, 1, 3).reshape(NT, KB, TILE_ROWS * 32)
    sc = s.reshape(NT, TILE_ROWS, KB, 2).permute(0, 2, 1, 3).reshape(NT, KB, TILE_ROWS * 2)
    return torch.cat([byte, sc], dim=2).contiguous()


MX_STAGE_K = 128
MX_STAGE_BYTES = TILE_ROWS * MX_STAGE_K // 2 + 512  # 8192 B of codes + 32 x 4 scale words
# experts in the block-scaled GEMM's stage format (csrc/moe.cu stb_moe_gemm_mx); STB200_MOE_MX=0 keeps
# the dequantising kernel's tiles (stb_moe_gemm_mxfp4) for A/B
MOE_MX = os.environ.get("STB200_MOE_MX", "1") != "0"


def pack_mx_stages(codes: torch.Tensor, exps: torch.Tensor) -> torch.Tensor:
    """(codes [N][K], exps [N][K/32]) -> uint8 [ceil(N/128)][ceil(K/128)][8704]: stage (n, s) = 128
    rows x 128 values of K as [128 rows][64 bytes] (byte j of a row: value 2j in the low nibble, 2j+1
    in the high; the tensor-memory accelerator unpacks them to 16-byte chunks) followed by 32 x 4
    scale words, word (l, j) = the four ue8m0 bytes (exponent + 127) of row 32 j + l, K slice t in
    byte t (the tcgen05.cp source layout). Rows past N and K past K are zero codes with scale 127."""
    N, K = codes.shape
    if K % TILE_K:
        raise ValueError("MX stages need K % 64 == 0")
    NT, KS = -(-N // TILE_ROWS), -(-K // MX_STAGE_K)
    c = torch.zeros(NT * TILE_ROWS, KS * MX_STAGE_K, dtype=torch.uint8, device=codes.device)
    c[:N, :K] = codes
    s = torch.full((NT * TILE_ROWS, KS * 4), 127, dtype=torch.uint8, device=codes.device)
    s[:N, :K // 32] = (exps.to(torch.int16) + 127).to(torch.uint8)
    byte = c[:, 0::2] | (c[:, 1::2] << 4)                                         # [NT*128][KS*64]
    byte = byte.reshape(NT, TILE_ROWS, KS, 64).permute(0, 2, 1, 3).reshape(NT, KS, TILE_ROWS * 64)
    sc = s.reshape(NT, 4, 32, KS, 4).permute(0, 3, 2, 1, 4).reshape(NT, KS, 512)  # [n][s][l][j][t]
    return torch.cat([byte, sc], dim=2).contiguous()


def pack_experts(codes: torch.Tensor, exps: torch.Tensor) -> torch.Tensor:
    """The product's expert packing: MX stages (block-scaled GEMM) or MXFP4 tiles (STB200_MOE_MX=0)."""
    return pack_mx_stages(codes, exps) if MOE_MX else pack_mxfp4_tiles(codes, exps)


class MoELayer:
    """One layer's experts on the device: packed MXFP4 gate-up / down experts (uint8 [E][NT][KS][8704]
    MX stages, or [E][NT][KB][4352] tiles with STB200_MOE_MX=0) and fp32 biases [E][2ff] / [E][d]."""

    __slots__ = ("gate_up", "b_gate_up", "down", "b_down")

    def __init__(self, gate_up, b_gate_up, down, b_down):
        self.gate_up, self.b_gate_up, self.down, self.b_down = gate_up, b_gate_up, down, b_down


def build_experts(shape: ModelShape, layer: int, seed: int, init_device: str, device: str) -> MoELayer:
    """Draw every expert of `layer` (bf16, per-tensor generators like the dense weights), quantize
    to MXFP4 on `init_device` and pack the tiles; one expert at a time, so the fp32 temporaries of
    a gpt-oss-120b layer never exceed one expert's."""
    gu, bgu, dn, bdn = [], [], [], []
    for e in range(shape.n_experts):
        (n_gu, s_gu), (n_bgu, s_bgu), (n_dn, s_dn), (n_bdn, s_bdn) = expert_specs(shape, layer, e)
        gu.append(pack_experts(*quantize_mxfp4(draw(s_gu, seed, n_gu, init_device))).to(device))
        dn.append(pack_experts(*quantize_mxfp4(draw(s_dn, seed, n_dn, init_device))).to(device))
        bgu.append(draw(s_bgu, seed, n_bgu, init_device).float().to(device))
        bdn.append(draw(s_bdn, seed, n_bdn, init_device).float().to(device))
    return MoELayer(torch.stack(gu), torch.stack(bgu), torch.stack(dn), torch.stack(bdn))


def build(shape: ModelShape, seed: int = 0, init_device: str = "cpu", device: str = "cuda") -> dict[str, torch.Tensor]:
    out = {}
    for name, shp, norm in tensor_specs(shape):
        t = draw(shp, seed, name, init_device, norm).to(device).contiguous()
        if name.endswith((".bqkv", ".bo", ".sinks", ".router_b")):
            t = t.float()  # consumed as fp32 by the kernels
        out[name] = t
    if shape.moe:
        for i in range(shape.layers):
            out[f"l{i}.experts"] = build_experts(shape, i, seed, init_device, device)
    return out
