// RoPE + KV commit of one (token, head, group-of-8-rotation-pairs) element of a fused QKV
// projection row: optional per-head RMSNorm of q and k (Qwen3 qk-norm), optional bias
// (gpt-oss), rotate-half RoPE of q and k, q written as bf16, k and v committed into the
// pre-swizzled pool pages at (slot_of[t], pos_of[t]). Shared by qkv_rope_commit_kernel
// (kv.cu) and the decode-block kernel's ROPE phase (gemm.cu). The d_head/16 threads of one
// head row must be adjacent lanes of one warp, and every lane of the warp must call this
// (valid or not): the qk-norm row reduction is a few xor-shuffles. The qkv row is read
// with ld.global.cg: in the decode block it was just reduced in L2 by other SMs.
#pragma once
#include "common.cuh"
#include "pool.cuh"

namespace stb {

__device__ __forceinline__ void rope_commit_elem(int64_t gid, float* __restrict__ qkv,
                                                 __nv_bfloat16* __restrict__ q_out,
                                                 const int32_t* __restrict__ slot_of,
                                                 const int32_t* __restrict__ pos_of, int n, int n_q, int n_kv,
                                                 int d_head, const float* __restrict__ inv_freq,
                                                 const int32_t* __restrict__ table, int max_bps,
                                                 __nv_bfloat16* __restrict__ kpages, __nv_bfloat16* __restrict__ vpages,
                                                 int clear_rows, const __nv_bfloat16* __restrict__ q_norm,
                                                 const __nv_bfloat16* __restrict__ k_norm, float eps,
                                                 const float* __restrict__ bias, float rope_scale) {
  const int half = d_head / 2;
  const int groups = half / 8;
  const int heads = n_q + 2 * n_kv;
  const bool valid = gid < (int64_t)n * heads * groups;
  const int g = gid % groups;
  const int h = (gid / groups) % heads;
  const int t = valid ? (int)(gid / ((int64_t)groups * heads)) : 0;
  float x1[8], x2[8];
  float* row = qkv + ((int64_t)t * heads + h) * d_head;
  if (valid) {
    const float4 a0 = __ldcg(reinterpret_cast<const float4*>(row + g * 8));
    const float4 a1 = __ldcg(reinterpret_cast<const float4*>(row + g * 8 + 4));
    const float4 b0 = __ldcg(reinterpret_cast<const float4*>(row + half + g * 8));
    const float4 b1 = __ldcg(reinterpret_cast<const float4*>(row + half + g * 8 + 4));
    x1[0] = a0.x, x1[1] = a0.y, x1[2] = a0.z, x1[3] = a0.w, x1[4] = a1.x, x1[5] = a1.y, x1[6] = a1.z, x1[7] = a1.w;
    x2[0] = b0.x, x2[1] = b0.y, x2[2] = b0.z, x2[3] = b0.w, x2[4] = b1.x, x2[5] = b1.y, x2[6] = b1.z, x2[7] = b1.w;
    if (bias != nullptr) {  // gpt-oss QKV bias (added before RoPE)
      const float* br = bias + h * d_head;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x1[j] += br[g * 8 + j];
        x2[j] += br[half + g * 8 + j];
      }
    }
    if (t < clear_rows) {  // leave the GEMM accumulator zeroed for the next stream-K product
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(row + g * 8) = z;
      *reinterpret_cast<float4*>(row + g * 8 + 4) = z;
      *reinterpret_cast<float4*>(row + half + g * 8) = z;
      *reinterpret_cast<float4*>(row + half + g * 8 + 4) = z;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) x1[j] = x2[j] = 0.f;
  }
  if (q_norm != nullptr) {  // uniform over the launch: every lane takes the shuffles
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) ss = fmaf(x1[j], x1[j], fmaf(x2[j], x2[j], ss));
    for (int o = 1; o < groups; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (h < n_q + n_kv) {
      const float r = rsqrtf(ss / (float)d_head + eps);
      const __nv_bfloat16* w = h < n_q ? q_norm : k_norm;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x1[j] = x1[j] * r * __bfloat162float(w[g * 8 + j]);
        x2[j] = x2[j] * r * __bfloat162float(w[half + g * 8 + j]);
      }
    }
  }
  if (!valid) return;
  float y1[8], y2[8];
  int pos = pos_of[t];
  if (h < n_q + n_kv) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float s, c;
      sincosf((float)pos * inv_freq[g * 8 + j], &s, &c);
      s *= rope_scale;  // YaRN attention factor (1 for plain RoPE)
      c *= rope_scale;
      y1[j] = x1[j] * c - x2[j] * s;
      y2[j] = x2[j] * c + x1[j] * s;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) { y1[j] = x1[j]; y2[j] = x2[j]; }
  }
  uint4 lo = make_uint4(pack_bf16(y1[0], y1[1]), pack_bf16(y1[2], y1[3]), pack_bf16(y1[4], y1[5]), pack_bf16(y1[6], y1[7]));
  uint4 hi = make_uint4(pack_bf16(y2[0], y2[1]), pack_bf16(y2[2], y2[3]), pack_bf16(y2[4], y2[5]), pack_bf16(y2[6], y2[7]));
  __nv_bfloat16* dst;
  int c_lo = g, c_hi = half / 8 + g;  // 16-byte chunks of the row
  if (h < n_q) {
    dst = q_out + ((int64_t)t * n_q + h) * d_head;
  } else {
    int kvh = (h < n_q + n_kv) ? h - n_q : h - n_q - n_kv;
    __nv_bfloat16* pages = (h < n_q + n_kv) ? kpages : vpages;
    int blk = table[(int64_t)slot_of[t] * max_bps + (pos >> 4)];
    dst = pages + (((int64_t)blk * n_kv + kvh) * 16 + (pos & 15)) * d_head;
    c_lo = kv_phys_chunk(pos & 15, c_lo);  // pre-swizzled page layout (pool.cuh)
    c_hi = kv_phys_chunk(pos & 15, c_hi);
  }
  *reinterpret_cast<uint4*>(dst + c_lo * 8) = lo;
  *reinterpret_cast<uint4*>(dst + c_hi * 8) = hi;
}

}  // namespace stb
