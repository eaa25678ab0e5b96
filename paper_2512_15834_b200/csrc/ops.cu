// Small fused row ops around the GEMMs (HBM-bound, one pass each) and K4, the
// speculation-validation kernel.
//
// K4 replaces `validate_draft` (`engine.py:96-111`) and the consume rule
// (`engine.py:291`): greedy longest-common-prefix of the drafted call ids against
// the ids the verify pass produced at the same positions, as int32 compares —
// bit-exact by construction. One warp per sequence: ballot of mismatches, ffs.
#include <cfloat>

#include "../../include/stb200.h"
#include "common.cuh"

using namespace stb;

namespace {

__global__ void embed_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ table,
                             float* __restrict__ x, int n, int d) {
  pdl_wait();
  pdl_launch();
  int t = blockIdx.x;
  const __nv_bfloat16* row = table + (int64_t)ids[t] * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    uint4 v = *reinterpret_cast<const uint4*>(row + c);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    float4 a, b;
    float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
    float2 f2 = __bfloat1622float2(h[2]), f3 = __bfloat1622float2(h[3]);
    a = make_float4(f0.x, f0.y, f1.x, f1.y);
    b = make_float4(f2.x, f2.y, f3.x, f3.y);
    *reinterpret_cast<float4*>(x + (int64_t)t * d + c) = a;
    *reinterpret_cast<float4*>(x + (int64_t)t * d + c + 4) = b;
  }
}

// block-wide sum with warp shuffles + one smem hop
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.f;
  t = warp_sum(t);
  __syncthreads();
  return t;
}

// embed + the first layer's fused-norm inputs: x = embed row (fp32), xb = bf16(x),
// ss[t][0] = sum x^2, ss[t][p] = 0 for the other partial slots
__global__ void embed_prep_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ table,
                                  float* __restrict__ x, __nv_bfloat16* __restrict__ xb, float* __restrict__ ss,
                                  int parts, int d) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[32];
  const int t = blockIdx.x;
  const __nv_bfloat16* row = table + (int64_t)ids[t] * d;
  float acc = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + c);
    *reinterpret_cast<uint4*>(xb + (int64_t)t * d + c) = v;  // bf16(x) == the embedding row
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    float f[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 p = __bfloat1622float2(h[j]);
      f[2 * j] = p.x;
      f[2 * j + 1] = p.y;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = fmaf(f[j], f[j], acc);
    *reinterpret_cast<float4*>(x + (int64_t)t * d + c) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(x + (int64_t)t * d + c + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
  acc = block_sum(acc, red);
  for (int j = threadIdx.x; j < parts; j += blockDim.x) ss[(int64_t)t * parts + j] = j == 0 ? acc : 0.f;
}

// one CTA per row, the row held in registers (VPT float4 per thread, blockDim*4*VPT == d):
// x (+)= delta; y = bf16(x * rsqrt(mean(x^2) + eps) * w). One global read of x (and
// delta), one write of x and y, a single block reduction.
template <int VPT>
__global__ void add_rmsnorm_kernel(float* __restrict__ x, float* __restrict__ delta,
                                   const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ y, int d,
                                   float eps, const int32_t* __restrict__ gather, int clear_rows,
                                   const float* __restrict__ bias) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[32];
  const int t = blockIdx.x;
  const int src = gather ? gather[t] : t;
  float* xr = x + (int64_t)src * d;
  float4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c >= d) {  // d not a multiple of 4 x threads (gpt-oss d = 2880)
      v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    v[i] = *reinterpret_cast<const float4*>(xr + c);
    if (delta) {
      float4* dp = reinterpret_cast<float4*>(delta + (int64_t)t * d + c);
      float4 e = *dp;
      if (t < clear_rows) *dp = make_float4(0.f, 0.f, 0.f, 0.f);  // GEMM accumulator back to zero
      if (bias) {
        const float4 b = *reinterpret_cast<const float4*>(bias + c);
        e.x += b.x, e.y += b.y, e.z += b.z, e.w += b.w;
      }
      v[i].x += e.x;
      v[i].y += e.y;
      v[i].z += e.z;
      v[i].w += e.w;
      *reinterpret_cast<float4*>(xr + c) = v[i];
    }
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  if (!y) return;  // residual add only
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
  __nv_bfloat16* yr = y + (int64_t)t * d;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c >= d) continue;
    const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + c));
    const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + c + 2));
    *reinterpret_cast<uint2*>(yr + c) = make_uint2(pack_bf16(v[i].x * inv * w01.x, v[i].y * inv * w01.y),
                                                   pack_bf16(v[i].z * inv * w23.x, v[i].w * inv * w23.y));
  }
}

// d = threads * 4 * VPT with threads a multiple of 32 and <= 1024
int launch_rmsnorm(float* x, float* delta, const void* w, void* y, int n, int d, float eps,
                   const int32_t* gather, int clear_rows, cudaStream_t st, const float* bias = nullptr) {
  if (d % 4) return fail(STB_EINVAL, "rmsnorm: d must be a multiple of 4");
  const int v4 = d / 4;
  int vpt = 1;
  while ((v4 + vpt - 1) / vpt > 1024) vpt *= 2;
  if (vpt > 8) return fail(STB_EINVAL, "rmsnorm: d too large");
  const int threads = (((v4 + vpt - 1) / vpt) + 31) / 32 * 32;  // whole warps (block_sum); tail lanes idle
  const auto* wb = (const __nv_bfloat16*)w;
  auto* yb = (__nv_bfloat16*)y;
  cudaError_t e;
  switch (vpt) {
    case 1: e = launch_k(add_rmsnorm_kernel<1>, dim3(n), dim3(threads), 0, st, x, delta, wb, yb, d, eps, gather, clear_rows, bias); break;
    case 2: e = launch_k(add_rmsnorm_kernel<2>, dim3(n), dim3(threads), 0, st, x, delta, wb, yb, d, eps, gather, clear_rows, bias); break;
    case 4: e = launch_k(add_rmsnorm_kernel<4>, dim3(n), dim3(threads), 0, st, x, delta, wb, yb, d, eps, gather, clear_rows, bias); break;
    default: e = launch_k(add_rmsnorm_kernel<8>, dim3(n), dim3(threads), 0, st, x, delta, wb, yb, d, eps, gather, clear_rows, bias); break;
  }
  if (e != cudaSuccess) return fail(STB_ECUDA, "rmsnorm launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

// (gate, up) pairs are interleaved in gu (the gate-up weight rows are interleaved at load,
// so the fused GEMM epilogue finds each pair in adjacent TMEM lanes)
__global__ void silu_mul_kernel(float* __restrict__ gu, __nv_bfloat16* __restrict__ y, int n, int f, int clear_rows) {
  pdl_wait();
  pdl_launch();
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  int64_t total = (int64_t)n * f;
  if (i >= total) return;
  int64_t t = i / f, c = i % f;
  float* p = gu + t * 2 * f + 2 * c;
  float4 a = *reinterpret_cast<const float4*>(p);      // g0 u0 g1 u1
  float4 b = *reinterpret_cast<const float4*>(p + 4);  // g2 u2 g3 u3
  if (t < clear_rows) {
    *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(p + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint2 o = make_uint2(pack_bf16(silu_gate(a.x, a.y), silu_gate(a.z, a.w)),
                       pack_bf16(silu_gate(b.x, b.y), silu_gate(b.z, b.w)));
  *reinterpret_cast<uint2*>(y + i) = o;
}

// Script-forced greedy sampling, split over the vocabulary: grid = R rows x CH chunks.
// Each CTA reduces its chunk to (max, argmax) of the raw and of the biased logits
// (first index wins ties), publishes a partial, and the last CTA of a row to
// finish (atomic ticket) reduces the row's CH partials; the ticket self-resets.
struct ArgPart {
  float best, bbest;
  int bi, bbi;
};

__device__ __forceinline__ void arg_merge(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) {
    v = ov;
    i = oi;
  }
}

__device__ __forceinline__ void block_arg(float& best, int& bi, float& bbest, int& bbi, ArgPart* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    float ob = __shfl_xor_sync(0xffffffffu, bbest, o);
    int obi = __shfl_xor_sync(0xffffffffu, bbi, o);
    arg_merge(best, bi, ov, oi);
    arg_merge(bbest, bbi, ob, obi);
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = {best, bbest, bi, bbi};
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    ArgPart p = l < nw ? sm[l] : ArgPart{-FLT_MAX, -FLT_MAX, 0x7fffffff, 0x7fffffff};
    best = p.best, bi = p.bi, bbest = p.bbest, bbi = p.bbi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      float ob = __shfl_xor_sync(0xffffffffu, bbest, o);
      int obi = __shfl_xor_sync(0xffffffffu, bbi, o);
      arg_merge(best, bi, ov, oi);
      arg_merge(bbest, bbi, ob, obi);
    }
  }
}

__global__ void sample_forced_kernel(float* __restrict__ logits, int64_t ld, const int32_t* __restrict__ target,
                                     int V, float bias, int CH, ArgPart* __restrict__ parts,
                                     int* __restrict__ tickets, int32_t* __restrict__ out,
                                     int32_t* __restrict__ raw_arg, float* __restrict__ raw_max, int clear) {
  pdl_wait();
  pdl_launch();
  __shared__ ArgPart sm[32];
  __shared__ int last;
  const int r = blockIdx.x / CH, ch = blockIdx.x % CH;
  float* row = logits + (int64_t)r * ld;
  const int tgt = target ? target[r] : -1;
  const int span = ((V + CH - 1) / CH + 3) & ~3;
  const int lo = ch * span, hi = min(V, lo + span);
  float best = -FLT_MAX, bbest = -FLT_MAX;
  int bi = 0x7fffffff, bbi = 0x7fffffff;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(logits) & 15) == 0);
  if (vec) {
    // 4 float4 loads in flight per thread before any compare
    constexpr int U = 4;
    const int step = blockDim.x * 4;
    for (int c0 = lo + threadIdx.x * 4; c0 < hi; c0 += U * step) {
      float4 v4[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * step;
        v4[u] = c < hi ? __ldcs(reinterpret_cast<const float4*>(row + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * step;
        if (c >= hi) break;
        if (clear) *reinterpret_cast<float4*>(row + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int idx = c + q;
          if (idx < hi) {
            arg_merge(best, bi, vv[q], idx);
            arg_merge(bbest, bbi, idx == tgt ? vv[q] + bias : vv[q], idx);
          }
        }
      }
    }
  } else {
    for (int c = lo + threadIdx.x; c < hi; c += blockDim.x) {
      const float x = row[c];
      if (clear) row[c] = 0.f;
      arg_merge(best, bi, x, c);
      arg_merge(bbest, bbi, c == tgt ? x + bias : x, c);
    }
  }
  block_arg(best, bi, bbest, bbi, sm);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = {best, bbest, bi, bbi};
    __threadfence();
    last = atomicAdd(&tickets[r], 1) == CH - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  ArgPart p = threadIdx.x < CH ? parts[r * CH + threadIdx.x] : ArgPart{-FLT_MAX, -FLT_MAX, 0x7fffffff, 0x7fffffff};
  best = p.best, bi = p.bi, bbest = p.bbest, bbi = p.bbi;
  block_arg(best, bi, bbest, bbi, sm);
  if (threadIdx.x == 0) {
    out[r] = bbi;
    if (raw_arg) raw_arg[r] = bi;
    if (raw_max) raw_max[r] = best;
    tickets[r] = 0;
  }
}

// K4: one warp per sequence
__global__ void spec_validate_kernel(const int32_t* __restrict__ draft, const int32_t* __restrict__ d_off,
                                     const int32_t* __restrict__ model, const int32_t* __restrict__ m_off,
                                     const int32_t* __restrict__ model_first,
                                     const int32_t* __restrict__ span_len, const int32_t* __restrict__ kv_len,
                                     const int32_t* __restrict__ base_extra, int S, int32_t* __restrict__ accepted,
                                     int32_t* __restrict__ consume, int32_t* __restrict__ new_len) {
  pdl_wait();
  pdl_launch();
  int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (s >= S) return;
  int dl = d_off[s + 1] - d_off[s];
  const int first = model_first ? model_first[s] : -1;
  const int lead = first >= 0 ? 1 : 0;
  int ml = m_off[s + 1] - m_off[s] + lead;
  int sl = span_len[s];
  int n = min(min(dl, ml), sl);
  const int32_t* d = draft + d_off[s];
  const int32_t* m = model + m_off[s];
  int acc = n;
  for (int base = 0; base < n; base += 32) {
    int i = base + lane;
    bool miss = false;
    if (i < n) miss = d[i] != (i < lead ? first : m[i - lead]);
    unsigned bal = __ballot_sync(0xffffffffu, miss);
    if (bal) {
      acc = base + __ffs(bal) - 1;
      break;
    }
  }
  if (lane == 0) {
    accepted[s] = acc;
    consume[s] = acc >= sl ? sl : acc + 1;
    if (new_len) new_len[s] = kv_len[s] + acc + (base_extra ? base_extra[s] : 0);
  }
}

}  // namespace

extern "C" {

int stb_embed(const int32_t* ids, const void* table, float* x, int n, int d, void* stream) {
  if (n <= 0) return STB_OK;
  if (d % 8) return fail(STB_EINVAL, "embed: d must be a multiple of 8");
  launch_k(embed_kernel, dim3(n), dim3(128), 0, (cudaStream_t)stream, ids, (const __nv_bfloat16*)table, x, n, d);
  STB_CHECK_LAUNCH("embed");
  return STB_OK;
}

int stb_embed_prep(const int32_t* ids, const void* table, float* x, void* xb, float* ss, int ss_parts, int n, int d,
                   void* stream) {
  if (n <= 0) return STB_OK;
  if (d % 8) return fail(STB_EINVAL, "embed_prep: d must be a multiple of 8");
  if (ss_parts < 1) return fail(STB_EINVAL, "embed_prep: ss_parts >= 1");
  launch_k(embed_prep_kernel, dim3(n), dim3(128), 0, (cudaStream_t)stream, ids, (const __nv_bfloat16*)table, x,
           (__nv_bfloat16*)xb, ss, ss_parts, d);
  STB_CHECK_LAUNCH("embed_prep");
  return STB_OK;
}

int stb_add_rmsnorm(float* x, float* delta, const void* w, void* y, int n, int d, float eps, int clear_rows,
                    void* stream) {
  if (n <= 0) return STB_OK;
  return launch_rmsnorm(x, delta, w, y, n, d, eps, nullptr, clear_rows, (cudaStream_t)stream);
}

int stb_add_bias_rmsnorm(float* x, float* delta, const float* bias, const void* w, void* y, int n, int d, float eps,
                         int clear_rows, void* stream) {
  if (n <= 0) return STB_OK;
  return launch_rmsnorm(x, delta, w, y, n, d, eps, nullptr, clear_rows, (cudaStream_t)stream, bias);
}

int stb_gather_rmsnorm(const float* x, const int32_t* idx, const void* w, void* y, int n, int d, float eps,
                       void* stream) {
  if (n <= 0) return STB_OK;
  return launch_rmsnorm(const_cast<float*>(x), nullptr, w, y, n, d, eps, idx, 0, (cudaStream_t)stream);
}

int stb_silu_mul(float* gu, void* y, int n, int f, int clear_rows, void* stream) {
  if (n <= 0) return STB_OK;
  if (f % 4) return fail(STB_EINVAL, "silu_mul: f must be a multiple of 4");
  int64_t total = (int64_t)n * f / 4;
  launch_k(silu_mul_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, gu, (__nv_bfloat16*)y, n, f, clear_rows);
  STB_CHECK_LAUNCH("silu_mul");
  return STB_OK;
}

int stb_sample_forced(float* logits, int64_t ld, const int32_t* target, int R, int V, float bias, int32_t* out,
                      int32_t* raw_argmax, float* raw_max, int clear, void* stream) {
  if (R <= 0) return STB_OK;
  constexpr int CH = 32;  // vocabulary chunks per row (<= 32: one warp reduces the partials)
  constexpr int kMaxRows = 65536;
  if (R > kMaxRows) return fail(STB_EINVAL, "sample_forced: at most %d rows per call", kMaxRows);
  // per-(device, stream) scratch: partials + self-resetting tickets (first use precedes capture)
  const size_t part_bytes = sizeof(ArgPart) * (size_t)kMaxRows * CH;
  auto* base = (uint8_t*)stream_scratch(kScratchSample, (cudaStream_t)stream, part_bytes + sizeof(int) * kMaxRows);
  if (!base) return fail(STB_ENOMEM, "sample_forced: scratch allocation failed (or first use inside a capture)");
  auto* parts = (ArgPart*)base;
  auto* tickets = (int*)(base + part_bytes);
  launch_k(sample_forced_kernel, dim3(R * CH), dim3(256), 0, (cudaStream_t)stream, logits, ld, target, V, bias, CH, parts, tickets, out,
                                                                 raw_argmax, raw_max, clear);
  STB_CHECK_LAUNCH("sample_forced");
  return STB_OK;
}

}  // extern "C"

namespace {
// K4b: canonical-key digests, bit-exact. One warp per probe: lanes stride over the key table and
// the lowest matching index wins (ballot + ffs per 32-entry block, first block with a match).
__global__ void key_match_kernel(const unsigned long long* __restrict__ probe, const int32_t* __restrict__ probe_rid,
                                 int n, const unsigned long long* __restrict__ keys,
                                 const int32_t* __restrict__ key_rid, int m, int32_t* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= n) return;
  const unsigned long long p0 = probe[2 * i], p1 = probe[2 * i + 1];
  const int rid = probe_rid[i];
  int found = -1;
  for (int base = 0; base < m; base += 32) {
    const int j = base + lane;
    const bool hit = j < m && key_rid[j] == rid && keys[2 * j] == p0 && keys[2 * j + 1] == p1;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (bal) {
      found = base + __ffs(bal) - 1;
      break;
    }
  }
  if (lane == 0) out[i] = found;
}
}  // namespace

extern "C" {

int stb_key_match(const void* probe, const int32_t* probe_rid, int n, const void* keys, const int32_t* key_rid, int m,
                  int32_t* out, void* stream) {
  if (n <= 0) return STB_OK;
  if (m < 0 || !probe || !probe_rid || !out || (m > 0 && (!keys || !key_rid)))
    return fail(STB_EINVAL, "key_match: bad operands");
  const int threads = 128, blocks = (n * 32 + threads - 1) / threads;
  launch_k(key_match_kernel, dim3(blocks), dim3(threads), 0, (cudaStream_t)stream,
           (const unsigned long long*)probe, probe_rid, n, (const unsigned long long*)keys, key_rid, m, out);
  STB_CHECK_LAUNCH("key_match");
  return STB_OK;
}

int stb_spec_validate(const int32_t* draft, const int32_t* d_off, const int32_t* model, const int32_t* m_off,
                      const int32_t* model_first, const int32_t* span_len, const int32_t* kv_len,
                      const int32_t* base_extra, int S, int32_t* accepted, int32_t* consume, int32_t* new_len,
                      void* stream) {
  if (S <= 0) return STB_OK;
  int threads = 128;
  int blocks = (S * 32 + threads - 1) / threads;
  launch_k(spec_validate_kernel, dim3(blocks), dim3(threads), 0, (cudaStream_t)stream, draft, d_off, model, m_off, model_first, span_len, kv_len,
                                                                     base_extra, S, accepted, consume, new_len);
  STB_CHECK_LAUNCH("spec_validate");
  return STB_OK;
}

}  // extern "C"
