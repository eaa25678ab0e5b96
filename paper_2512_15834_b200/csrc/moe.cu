// gpt-oss mixture-of-experts MLP (config C4): routing, token permutation, the MXFP4 grouped
// GEMM on the 5th-gen tensor cores, and the weighted combine fused with the next RMSNorm.
//
// Replaces, for the MoE model family, the MLP part of every `rate x tokens` charge of the
// reference engine (`engine.py:251,270,296,358`); the reference itself has no model
// (SPEC.md:17). Expert weights are MXFP4 — e2m1 values with one ue8m0 scale per 32 along K, the
// released gpt-oss checkpoint's format — which is what lets a 120B replica (~67 GB) live on one
// B200. The default GEMM (moe_gemm_mx_kernel, further down) is block-scaled: the tensor
// core reads the e2m1 codes and applies their scales itself (kind::mxf8f6f4), with the token rows
// split exactly into two e4m3 halves; the description below is the dequantising kernel it replaced
// (kept for A/B, STB200_MOE_MX=0), whose activations stay fp16 (kind::f16 on weights dequantised
// on chip).
//
// Per layer (one stream, programmatic dependent launch throughout):
//   K5 router GEMM (bf16, gemm.cu) -> logits [T][E]
//   moe_route_kernel      warp per token: + bias, top-k (ties -> lower expert id), softmax over
//                         the k selected logits; claims a rank in its expert (atomic count)
//   moe_gather_kernel     expert offsets (prefix of the counts), the permutation, and the
//                         token rows copied expert-contiguous as fp16 (the GEMM's B operand)
//   moe_gemm_mxfp4_kernel gate-up (clamped SwiGLU epilogue -> fp16 act) and down (+bias -> fp32)
//   moe_combine_kernel    x += sum_k w_k * y[perm(t, k)] (fixed k order: deterministic), then
//                         RMSNorm of the new residual row (the next layer's input); zeroes the
//                         counts for the next layer
//
// Grouped GEMM, weight-stationary like K5: UMMA M = 128 expert weight rows, N = BN tokens of
// that expert. Persistent, one CTA per SM; the work list (expert, 128-row tile, token tile) is
// derived on the device from the counts, so the launch (and a CUDA graph of it) does not depend
// on the routing. Per K block of 64 the weight tile is 4352 contiguous bytes (4096 B of codes +
// 256 B of scales, runtime/weights.py pack_mxfp4_tiles): one bulk copy. Dequantisation never
// touches shared memory on the way out: converter thread r (= TMEM lane r = weight row r) reads
// its 32 code bytes, F2FP.F16.E2M1 unpacks two values per instruction, HMUL2 applies the 2^e
// scale (exact), and tcgen05.st writes the 32 fp16x2 columns straight into a TMEM A-operand
// ring; the MMA reads A from TMEM and the fp16 token rows (B) from smem. So shared memory
// carries 4.25 KB of weight bytes per stage instead of 16 KB of dequantised tiles written and
// read again — the MoE is HBM-bound on the weights at every batch the engine runs.
//   warp 0      weight producer: per stage the item's two 128-row tiles of one K block (a
//               work item is 256 weight rows sharing one token tile: twice the bytes per
//               pipeline stage, half the token-tile loads), into a ring the converters free
//               as soon as the tiles are in their registers
//   warp 3      token producer: the expert's fp16 token rows per stage (TMA, L2-resident), a
//               ring the MMA frees
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma kind::f16 per stage, A from TMEM
//   warp 2      TMEM allocator
//   warps 4-11  converters: smem codes -> fp16 -> TMEM A ring, one warp per (tile, lane
//               quarter = warp & 3); per-stage fixed latencies (smem loads, the TMEM store wait,
//               barrier hand-offs) are what paced the single-tile version (0.51 of HBM at the
//               C4 decode shape), so each stage now carries two tiles' worth of bytes
//   warps 12-15 epilogue: TMEM accumulator (double-buffered) -> SwiGLU / bias -> global
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/stb200.h"
#include "common.cuh"

using namespace stb;

namespace {

constexpr int kMaxE = 256;
constexpr int kMaxK = 8;
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int RAW = 4352;  // one MXFP4 tile: 128 rows x 32 code bytes + 128 rows x 2 scale bytes
#ifndef STB_MOE_NTP
#define STB_MOE_NTP 2
#endif
constexpr int NTP = STB_MOE_NTP;  // weight tiles (of 128 rows) per work item: a 256-row item shares
                                  // one token tile and doubles the bytes every pipeline stage carries
#ifndef STB_MOE_CONV_PAR
#define STB_MOE_CONV_PAR 2
#endif
constexpr int CPAR = STB_MOE_CONV_PAR;  // converter warps per (tile, lane quarter), on alternating stages
constexpr int kConvWarps = 4 * NTP * CPAR;
constexpr int kThreads = 32 * (4 + kConvWarps + 4);
// TMEM: accumulators [buffer][tile][BN] in [0, 2 NTP BN), then the A ring: stages of NTP x 32
// columns of fp16x2 (64 K values x 128 rows per tile), as many as fit (at most 8)
template <int BN>
constexpr int a_col0() { return 2 * NTP * BN; }
template <int BN>
constexpr int a_stages() { return std::min(8, (512 - a_col0<BN>()) / (32 * NTP)); }

template <int BN>
struct MCfg {
  static constexpr int X_BYTES = BN * BK * 2;  // fp16 token rows of one K block, SW128 K-major
#ifndef STB_MOE_XS
#define STB_MOE_XS 8
#endif
  static constexpr int XS = STB_MOE_XS;        // token-tile ring (L2-resident rows, freed by the MMA)
#ifndef STB_MOE_RING_KB
#define STB_MOE_RING_KB 196
#endif
  // weight-tile ring: freed by the converters as soon as they have read a tile, so the bytes in
  // flight from HBM never wait behind the dequantise -> MMA pipeline
  static constexpr int WS = std::min(24, (STB_MOE_RING_KB * 1024 - XS * X_BYTES) / (NTP * RAW));
  static constexpr int SMEM = 1024 + XS * X_BYTES + WS * NTP * RAW + 1024;
};

// mbarrier wait that lets the hardware suspend the thread until the phase completes (long waits:
// the epilogue warps, whose spinning otherwise steals issue slots from the converters)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// two e2m1 codes (byte B of x) -> fp16x2 (low nibble -> low half). The byte is named as a .b8
// piece of x, so ptxas folds the selection into the conversion (F2FP.F16.E2M1.UNPACK_B R, x.B1):
// no shift per byte, a quarter of the converters' instructions
template <int B>
__device__ __forceinline__ uint32_t e2m1x2_to_f16x2(uint32_t x) {
  uint32_t d;
  if constexpr (B == 0)
    asm("{\n.reg .b8 b0, b1, b2, b3;\nmov.b32 {b0, b1, b2, b3}, %1;\ncvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(d) : "r"(x));
  else if constexpr (B == 1)
    asm("{\n.reg .b8 b0, b1, b2, b3;\nmov.b32 {b0, b1, b2, b3}, %1;\ncvt.rn.f16x2.e2m1x2 %0, b1;\n}" : "=r"(d) : "r"(x));
  else if constexpr (B == 2)
    asm("{\n.reg .b8 b0, b1, b2, b3;\nmov.b32 {b0, b1, b2, b3}, %1;\ncvt.rn.f16x2.e2m1x2 %0, b2;\n}" : "=r"(d) : "r"(x));
  else
    asm("{\n.reg .b8 b0, b1, b2, b3;\nmov.b32 {b0, b1, b2, b3}, %1;\ncvt.rn.f16x2.e2m1x2 %0, b3;\n}" : "=r"(d) : "r"(x));
  return d;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// ---------------------------------------------------------------- routing
template <int EPL>
__global__ void __launch_bounds__(256) moe_route_kernel(const float* __restrict__ logits, int64_t ld,
                                                        const float* __restrict__ bias, int T, int E, int k,
                                                        int* __restrict__ counts, int* __restrict__ expert,
                                                        int* __restrict__ rank, float* __restrict__ wt) {
  pdl_wait();
  pdl_launch();
  const int t = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (t >= T) return;
  float v[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = j * 32 + lane;
    v[j] = e < E ? logits[(int64_t)t * ld + e] + (bias ? bias[e] : 0.f) : -INFINITY;
  }
  float sv[kMaxK];
  int se[kMaxK];
#pragma unroll
  for (int r = 0; r < kMaxK; ++r) {
    if (r >= k) break;
    float bv = -INFINITY;
    int be = 1 << 30;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = j * 32 + lane;
      if (e < E && (v[j] > bv || (v[j] == bv && e < be))) bv = v[j], be = e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (ov > bv || (ov == bv && oe < be)) bv = ov, be = oe;
    }
    sv[r] = bv;
    se[r] = be;
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (j * 32 + lane == be) v[j] = -INFINITY;
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < kMaxK; ++r)
    if (r < k) s += expf(sv[r] - sv[0]);
#pragma unroll
  for (int r = 0; r < kMaxK; ++r) {
    if (r < k && lane == r) {
      const int64_t p = (int64_t)t * k + r;
      expert[p] = se[r];
      rank[p] = atomicAdd(counts + se[r], 1);
      wt[p] = expf(sv[r] - sv[0]) / s;
    }
  }
}

// exclusive prefix of counts[0..E) into off[0..E] (shared), whole block
__device__ __forceinline__ void block_prefix(const int* __restrict__ counts, int E, int* off) {
  __shared__ int part[kMaxE / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < kMaxE) {
    const int c = tid < E ? counts[tid] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) part[w] = incl;
    off[tid + 1] = incl;  // provisional (warp-local)
  }
  __syncthreads();
  if (tid < kMaxE) {
    int base = 0;
    for (int j = 0; j < w; ++j) base += part[j];
    off[tid + 1] += base;
  }
  if (tid == 0) off[0] = 0;
  __syncthreads();
}

// expert-contiguous fp16 copy of the token rows; perm[t*k + r] = destination row
__global__ void __launch_bounds__(256) moe_gather_kernel(const __nv_bfloat16* __restrict__ h, int64_t ldh, int T,
                                                         int d, int k, int E, const int* __restrict__ counts,
                                                         const int* __restrict__ expert, const int* __restrict__ rank,
                                                         int* __restrict__ offsets, int* __restrict__ perm,
                                                         __half* __restrict__ xperm) {
  pdl_wait();
  pdl_launch();
  __shared__ int off[kMaxE + 1];
  block_prefix(counts, E, off);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += blockDim.x) offsets[e] = off[e];
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < T * k; p += nw) {
    const int t = p / k;
    const int row = off[expert[p]] + rank[p];
    if (lane == 0) perm[p] = row;
    const __nv_bfloat16* src = h + (int64_t)t * ldh;
    __half* dst = xperm + (int64_t)row * d;
    for (int c = lane * 8; c < d; c += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(src + c);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
      uint4 o;
      __half2* oh = reinterpret_cast<__half2*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) oh[q] = __float22half2_rn(__bfloat1622float2(b[q]));
      *reinterpret_cast<uint4*>(dst + c) = o;
    }
  }
}

// x[t] += sum_r wt[t,r] * y[perm[t,r]] (+ the fixed r order), then RMSNorm(x[t]) * w -> hn (bf16)
__global__ void __launch_bounds__(256) moe_combine_kernel(float* __restrict__ x, const float* __restrict__ y, int d,
                                                          int k, const int* __restrict__ perm,
                                                          const float* __restrict__ wt,
                                                          const __nv_bfloat16* __restrict__ w,
                                                          __nv_bfloat16* __restrict__ hn, float eps,
                                                          int* __restrict__ counts, int E) {
  pdl_wait();
  pdl_launch();
  __shared__ float red[32];
  const int t = blockIdx.x;
  if (t == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) counts[e] = 0;  // the next layer's route starts clean
  int rows[kMaxK];
  float ws[kMaxK];
#pragma unroll
  for (int r = 0; r < kMaxK; ++r) {
    rows[r] = r < k ? perm[(int64_t)t * k + r] : 0;
    ws[r] = r < k ? wt[(int64_t)t * k + r] : 0.f;
  }
  float* xr = x + (int64_t)t * d;
  float ss = 0.f;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(xr + c);
#pragma unroll
    for (int r = 0; r < kMaxK; ++r) {
      if (r < k) {
        const float4 yv = __ldcg(reinterpret_cast<const float4*>(y + (int64_t)rows[r] * d + c));
        v.x += ws[r] * yv.x, v.y += ws[r] * yv.y, v.z += ws[r] * yv.z, v.w += ws[r] * yv.w;
      }
    }
    *reinterpret_cast<float4*>(xr + c) = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (hn == nullptr) return;
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / d + eps);
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + c));
    const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + c + 2));
    *reinterpret_cast<uint2*>(hn + (int64_t)t * d + c) =
        make_uint2(pack_bf16(v.x * inv * w01.x, v.y * inv * w01.y), pack_bf16(v.z * inv * w23.x, v.w * inv * w23.y));
  }
}

// ---------------------------------------------------------------- grouped MXFP4 GEMM
struct MoeArgs {
  const uint8_t* w;     // [E][NT][KB][RAW]
  const float* bias;    // [E][N]
  const int* counts;    // [E]
  void* out;            // kind 1: fp16 act [rows][N/2]; kind 2: fp32 y [rows][N]
  int64_t ldo;
  int E, N, K, kind;
  float limit;          // SwiGLU clamp (kind 1)
  uint8_t* qout;        // kind 1, block-scaled path: the down input's e4m3 halves [2][qcap][N/2] (or null)
  uint8_t* qsf;         // ... and its scale words, as bytes ([stages][2][pitch] words)
  int qcap;
};

constexpr float kSwigluAlpha = 1.702f;

__device__ __forceinline__ float gpt_oss_glu(float g, float u, float limit) {
  g = fminf(g, limit);
  u = fminf(fmaxf(u, -limit), limit);
  return (u + 1.f) * (g / (1.f + __expf(-kSwigluAlpha * g)));
}

__device__ __forceinline__ void tmem_st32_wait_fence(uint32_t taddr, const uint32_t* r) {
  tmem_st32(taddr, r);
  tmem_st_wait();
  tc_fence_before();
}

// instruction descriptor: fp16 x fp16 -> fp32, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#ifdef STB_MOE_PROF
// timing experiments only: cycles each role spends in its waits, summed over the grid
__device__ unsigned long long g_moe_prof[16];
#define MPROF_DECL unsigned long long mp_[4] = {0, 0, 0, 0}, mp_t0 = clock64();
#define MPROF_WAIT(slot, call)            \
  {                                       \
    const unsigned long long t_ = clock64(); \
    call;                                 \
    mp_[slot] += clock64() - t_;          \
  }
#define MPROF_FLUSH(base, cond)                                                       \
  if (cond) {                                                                         \
    for (int q_ = 0; q_ < 3; ++q_) atomicAdd(&g_moe_prof[base + q_], mp_[q_]);        \
    atomicAdd(&g_moe_prof[base + 3], clock64() - mp_t0);                             \
  }
#else
#define MPROF_DECL
#define MPROF_WAIT(slot, call) call;
#define MPROF_FLUSH(base, cond)
#endif

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) moe_gemm_mxfp4_kernel(const __grid_constant__ CUtensorMap tm_x,
                                                                     const MoeArgs a) {
  using CF = MCfg<BN>;
  constexpr int XS = CF::XS, WS = CF::WS;
  constexpr int WSTAGE = NTP * RAW;
  constexpr int A_COL0 = a_col0<BN>(), A_STAGES = a_stages<BN>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sx = smem;                              // [XS][X_BYTES], 1024-aligned (SW128)
  uint8_t* sw = sx + XS * CF::X_BYTES;             // [WS][NTP][RAW]
  uint64_t* w_full = reinterpret_cast<uint64_t*>(sw + WS * WSTAGE);
  uint64_t* w_empty = w_full + WS;                 // converters -> weight producer
  uint64_t* x_full = w_empty + WS;
  uint64_t* x_empty = x_full + XS;                 // MMA -> token producer
  uint64_t* a_full = x_empty + XS;                 // [A_STAGES] converters -> MMA
  uint64_t* a_empty = a_full + 8;                  // [A_STAGES] MMA -> converters
  uint64_t* acc_full = a_empty + 8;                // [2]
  uint64_t* acc_empty = acc_full + 2;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  __shared__ int s_off[kMaxE + 1];                 // token-row offset of each expert
  __shared__ int s_item[kMaxE + 1];                // work-item prefix
  __shared__ int s_cnt[kMaxE];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = a.E, NT = ceil_div(a.N, BM), NP = ceil_div(NT, NTP), KB = a.K / BK;
  if (threadIdx.x == 0) {
    tma_prefetch(&tm_x);
    for (int s = 0; s < WS; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 4 * NTP);  // the stage's converter warps (one per tile x quarter)
    }
    for (int s = 0; s < XS; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(&a_full[s], 4 * NTP);
      mbar_init(&a_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  pdl_wait();  // counts (route) and token rows (gather) come from the preceding kernels
  // work list: items of expert e = ceil(count_e / BN) token tiles x NP pairs of weight tiles
  block_prefix(a.counts, E, s_off);
  if (threadIdx.x < kMaxE) s_cnt[threadIdx.x] = threadIdx.x < E ? s_off[threadIdx.x + 1] - s_off[threadIdx.x] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      s_item[e] = run;
      run += ceil_div(s_cnt[e], BN) * NP;
    }
    s_item[E] = run;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch();
  const uint32_t tmem = *tmem_slot;
  const int total = s_item[E];
  // item -> (expert, first weight tile, token tile); m fastest: the token tiles that share a
  // weight slice run on neighbouring CTAs at the same time (the slice is read from HBM once)
  auto decode = [&](int it, int& e, int& nt0, int& m) {
    int lo = 0, hi = E - 1;  // last e with s_item[e] <= it (experts with no items are skipped)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_item[mid] <= it) lo = mid; else hi = mid - 1;
    }
    e = lo;
    const int mt = ceil_div(s_cnt[e], BN);
    const int local = it - s_item[e];
    const int p = local / mt;
    m = local - p * mt;
    nt0 = p * NTP;
  };

  if (warp == 0) {
    // weight producer: the item's NTP tiles of one K block per stage (one bulk copy each)
    if (elect_one()) {
      MPROF_DECL
      int i = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        int e, nt0, m;
        decode(it, e, nt0, m);
        const int nt_n = min(NTP, NT - nt0);
        const uint8_t* wt = a.w + ((int64_t)e * NT + nt0) * KB * RAW;
        for (int kb = 0; kb < KB; ++kb, ++i) {
          const int s = i % WS;
          MPROF_WAIT(0, mbar_wait(&w_empty[s], ((i / WS) & 1) ^ 1));
          mbar_expect_tx(&w_full[s], nt_n * RAW);
          for (int t = 0; t < nt_n; ++t)
            bulk_load(smem_u32(sw + s * WSTAGE + t * RAW), wt + ((int64_t)t * KB + kb) * RAW, RAW, &w_full[s]);
        }
      }
      MPROF_FLUSH(0, true)
    }
    __syncwarp();
  } else if (warp == 3) {
    // token producer: the expert's BN fp16 rows of each K block (TMA, L2-resident)
    if (elect_one()) {
      int i = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        int e, nt0, m;
        decode(it, e, nt0, m);
        const int xrow = s_off[e] + m * BN;
        for (int kb = 0; kb < KB; ++kb, ++i) {
          const int s = i % XS;
          mbar_wait(&x_empty[s], ((i / XS) & 1) ^ 1);
          mbar_expect_tx(&x_full[s], CF::X_BYTES);
          tma_load_2d(sx + s * CF::X_BYTES, &tm_x, &x_full[s], kb * BK, xrow);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16(BM, BN);
#ifndef STB_MOE_MMA_PER_STAGE
#define STB_MOE_MMA_PER_STAGE (BK / 16)  // < 4: timing experiments only (results are wrong)
#endif
      MPROF_DECL
      int i = 0, j = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x, ++j) {
        int e, nt0, m;
        decode(it, e, nt0, m);
        const int nt_n = min(NTP, NT - nt0);
        const int buf = j & 1;
        MPROF_WAIT(0, mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1));
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++i) {
          const int xs = i % XS, as = i % A_STAGES;
          MPROF_WAIT(1, mbar_wait(&x_full[xs], (i / XS) & 1));        // token rows landed (TMA)
          MPROF_WAIT(2, mbar_wait(&a_full[as], (i / A_STAGES) & 1));  // weights dequantised into TMEM
          tc_fence_after();
          const uint64_t bdesc = umma_desc_kmajor_sw128(smem_u32(sx + xs * CF::X_BYTES), 1024);
          for (int t = 0; t < nt_n; ++t) {
            const uint32_t d = tmem + (buf * NTP + t) * BN;
            const uint32_t acol = tmem + A_COL0 + (as * NTP + t) * 32;
#pragma unroll
            for (int kk = 0; kk < STB_MOE_MMA_PER_STAGE; ++kk)  // +32 B along K = +2 in the descriptor
              umma_f16_ts(d, acol + kk * 8, bdesc + 2 * kk, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&x_empty[xs]);
          umma_commit(&a_empty[as]);
        }
        umma_commit(&acc_full[buf]);
      }
      MPROF_FLUSH(4, true)
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + kConvWarps) {
    // converters: warp = (parity p, tile t, lane quarter q); thread = weight row r of tile t = TMEM
    // lane r; the warp takes the stages i with i % CPAR == p
    const int q = warp & 3, t = ((warp - 4) >> 2) % NTP, par = (warp - 4) / (4 * NTP), r = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t sw_u32 = smem_u32(sw);
    MPROF_DECL
    int i = 0;
    for (int it = blockIdx.x; it < total; it += gridDim.x) {
      int e, nt0, m;
      decode(it, e, nt0, m);
      const bool live = nt0 + t < NT;  // the last pair of an odd tile count has one tile
      for (int kb = 0; kb < KB; ++kb, ++i) {
        if (i % CPAR != par) continue;
        const int s = i % WS, as = i % A_STAGES;
        MPROF_WAIT(0, mbar_wait(&w_full[s], (i / WS) & 1));
        uint32_t out[32];
#ifdef STB_MOE_SKIP_CONVERT  // timing experiments only: stream the weights, convert nothing
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_empty[s]);
        mbar_wait(&a_empty[as], ((i / A_STAGES) & 1) ^ 1);
        if (lane == 0) mbar_arrive(&a_full[as]);
        continue;
#endif
        if (live) {
          const uint32_t raw = sw_u32 + s * WSTAGE + t * RAW;
          const uint4 c0 = lds128(raw + r * 32);
          const uint4 c1 = lds128(raw + r * 32 + 16);
          const uint32_t sc = lds16(raw + 4096 + r * 2);
          __syncwarp();
          if (lane == 0) mbar_arrive(&w_empty[s]);  // the tile is in registers: its slot may refill
          // 2^(e) as fp16: exponent field e + 15 = byte - 127 + 15 (byte in [114, 139] by construction)
          const uint32_t h0 = ((sc & 0xFFu) - 112u) << 10, h1 = ((sc >> 8) - 112u) << 10;
          const uint32_t s0 = h0 | (h0 << 16), s1 = h1 | (h1 << 16);
          const uint32_t wv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const uint32_t scl = w < 4 ? s0 : s1;  // bytes 0-15: values 0-31 (scale 0), 16-31: scale 1
            out[w * 4 + 0] = hmul2(e2m1x2_to_f16x2<0>(wv[w]), scl);
            out[w * 4 + 1] = hmul2(e2m1x2_to_f16x2<1>(wv[w]), scl);
            out[w * 4 + 2] = hmul2(e2m1x2_to_f16x2<2>(wv[w]), scl);
            out[w * 4 + 3] = hmul2(e2m1x2_to_f16x2<3>(wv[w]), scl);
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&w_empty[s]);
        }
        MPROF_WAIT(1, mbar_wait(&a_empty[as], ((i / A_STAGES) & 1) ^ 1));
        tc_fence_after();
        if (live) tmem_st32_wait_fence(tmem + lane_addr + A_COL0 + (as * NTP + t) * 32, out);
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
      }
    }
    MPROF_FLUSH(8, lane == 0)
  } else if (warp >= 4 + kConvWarps) {
    // epilogue: thread = weight row (feature) of each of the item's tiles; columns = tokens
    const int q = warp & 3;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int j = 0;
    for (int it = blockIdx.x; it < total; it += gridDim.x, ++j) {
      int e, nt0, m;
      decode(it, e, nt0, m);
      const int nt_n = min(NTP, NT - nt0);
      const int buf = j & 1;
      const int row0 = s_off[e] + m * BN;
      const int nv = min(BN, s_cnt[e] - m * BN);
      mbar_wait_sleep(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      for (int t = 0; t < nt_n; ++t) {
        const int f = (nt0 + t) * BM + q * 32 + lane;
        const float b = f < a.N ? __ldg(a.bias + (int64_t)e * a.N + f) : 0.f;
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          uint32_t rr[16];
          tmem_ld16(tmem + lane_addr + (buf * NTP + t) * BN + c, rr);
          tmem_ld_wait();
          if (a.kind == 2) {
            float* y = reinterpret_cast<float*>(a.out);
            if (f < a.N) {
#pragma unroll
              for (int u = 0; u < 16; ++u)
                if (c + u < nv) y[(int64_t)(row0 + c + u) * a.ldo + f] = __uint_as_float(rr[u]) + b;
            }
          } else {
            // (gate, up) of output feature f/2 in lanes (2i, 2i+1): the even lane emits tokens
            // c..c+7 of the chunk, the odd lane c+8..c+15
            __half* act = reinterpret_cast<__half*>(a.out);
            const bool odd = lane & 1;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float mine = __uint_as_float(odd ? rr[8 + u] : rr[u]) + b;
              const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? rr[u] : rr[8 + u]) + b, 1);
              const int tok = c + (odd ? 8 : 0) + u;
              const float g = odd ? other : mine, up = odd ? mine : other;
              if (f < a.N && tok < nv)
                act[(int64_t)(row0 + tok) * a.ldo + (f >> 1)] = __float2half_rn(gpt_oss_glu(g, up, a.limit));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free(tmem, 512);
}

// ---------------------------------------------------------------- block-scaled MXFP4 grouped GEMM
// tcgen05.mma kind::mxf8f6f4.block_scale: A = the e2m1 expert weights with their own ue8m0 scales
// (one per 32 along K, the checkpoint's), B = the token rows split exactly into two e4m3 halves with
// one ue8m0 scale per 32 (x = hi 2^s_hi + lo 2^s_lo, stb_moe_quant): B carries 2 BN rows (BN hi
// rows, then BN lo rows) and the epilogue adds the two accumulator column halves. No thread touches
// a weight byte: the tensor-memory-accelerator unpacks the packed codes into the operand layout
// (CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B: 16 codes in the low 8 bytes of each 16-byte chunk, 128-byte
// swizzle; the transaction counts the 8 KB read, not the 16 KB written), and the MMA thread moves
// both operands' scale words into tensor memory itself (tcgen05.cp.32x128b.warpx4), in issue order
// with its MMAs. Weight format (runtime/weights.py pack_mx_stages): per (expert, 128-row tile,
// 128-wide K stage) 8704 B = [128 rows][64 B] codes + [32 lanes][4] scale words (word (l, j) = the
// four K-slice scales of row 32 j + l: the tcgen05.cp source layout). Formats settled on a B200 by
// tools/probe_mxf8f6f4.cu and tools/probe_mx_tma.cu.
//   warp 0      weight producer: one 3-D TMA (codes) + one bulk copy (scale words) per stage
//   warp 1      MMA issuer: per stage 2 tcgen05.cp + 4 MMAs (32 of K each), commits free the rings
//   warp 2      TMEM allocator, then token-scale stager: an item's B scale words for every stage,
//               gathered from the [stage][hi|lo][row] words into the tcgen05.cp layout (double-buffered
//               per item, so the L2 round trips overlap the previous item's stream)
//   warp 3      token producer: BN hi rows + BN lo rows per stage (TMA, L2-resident)
//   warps 4-7   epilogue: TMEM accumulator (double-buffered) -> SwiGLU / bias -> global
__host__ __device__ constexpr int sf_pitch(int rows_cap) { return (rows_cap + 3) & ~3; }
constexpr int MX_BK = 128;          // K per pipeline stage
constexpr int MX_STAGE = 8704;      // bytes of one weight stage in HBM (codes + scale words)
constexpr int MX_KS_MAX = 24;       // K <= 3072: an item's token scale words fit one staging buffer
constexpr int kMxThreads = 32 * 8;

template <int BN>
struct MxCfg {
  static constexpr int XB = 2 * BN * MX_BK;  // e4m3 hi + lo rows of one stage
  static constexpr int AB = BM * MX_BK;      // unpacked codes of one 128-row stage (16 KB)
  static constexpr int SFB_COLS = (2 * BN + 31) / 32;
  static constexpr int SFB_ITEM = MX_KS_MAX * 512;  // an item's token scale words, every stage
#ifndef STB_MOE_MX_RING_KB
#define STB_MOE_MX_RING_KB 222
#endif
  // one ring: a stage holds the weight codes, their scale words and the token halves, filled by two
  // producers onto one barrier and freed by one commit (the MMA thread paces the kernel: every
  // barrier operation it saves is issue time)
  static constexpr int WS = std::min(16, (STB_MOE_MX_RING_KB * 1024 - 2 * SFB_ITEM) / (AB + 512 + XB));
  static constexpr int XS = WS;
  static constexpr int SMEM = 1024 + WS * AB + XS * XB + WS * 512 + 2 * SFB_ITEM + 1024;
#ifndef STB_MX_ACC2
#define STB_MX_ACC2 0
#endif
  // independent accumulators per buffer (K slices alternate between them, summed by the epilogue):
  // consecutive MMAs of a stage do not wait on each other's accumulator
  static constexpr int NACC = (STB_MX_ACC2 && BN <= 32) ? 2 : 1;
  static constexpr int ACC_COLS = NACC * 2 * BN;  // one buffer
  static constexpr int SF0 = 2 * ACC_COLS;   // TMEM: after the double-buffered accumulators
  static constexpr int SFS = 8;              // 4 SFA + 4 SFB columns per scale slot
  static constexpr int SLOTS = 4;
  static_assert(SFB_COLS <= 4 && SF0 + SLOTS * SFS <= 512 && WS >= 4, "MX GEMM budget");
};

__device__ __forceinline__ void umma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
// 32 rows x 16 B of shared memory -> TMEM lanes 0-31 x 4 columns, replicated into every lane quarter
__device__ __forceinline__ void tc_cp_sf(uint32_t taddr, uint32_t saddr) {
  const uint64_t desc = (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n" ::"r"(taddr), "l"(desc));
}
// A = e2m1 (format 5), B = e4m3 (0), K-major, ue8m0 scales (bit 23), M, N; scale ids per slice
__host__ __device__ constexpr uint32_t idesc_mx(int M, int N) {
  return (5u << 7) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ int blk_exp(float amax) {
  int e;
  frexpf(amax, &e);  // amax = m 2^e, m in [0.5, 1)
  return amax > 0.f ? e - 8 : 0;
}
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
  uint16_t lo, hi;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %2, %1;" : "=h"(lo) : "f"(a), "f"(b));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %2, %1;" : "=h"(hi) : "f"(c), "f"(d));
  return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ float2 e4m3x2_to_f2(uint16_t v) {
  uint32_t h;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(v));
  return __half22float2(*reinterpret_cast<__half2*>(&h));
}
// gate-up epilogue -> the down projection's B operand (no fp16 act round trip, no quant launch): the
// chunk's 8 SwiGLU values per lane (feature f/2, tokens c..c+7 on even lanes, c+8..c+15 on odd) are
// split like quant_stage, with each 32-feature block's maxima reduced over the 16 same-parity lanes
// and the partner warp holding the block's other 16 features (named barrier per warp pair)
__device__ __forceinline__ void pair_bar(int q) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(1 + (q >> 1)) : "memory");
}
__device__ __forceinline__ void glu_quant_chunk(const float* gv, int q, int lane, int nt, int f, int N, int c, int nv,
                                                int row0, const MoeArgs& a, float (*s_x)[2][8], float (*s_r)[2][8]) {
  const int odd = lane & 1;
  float am[8], sc[8], r[8];
  int eh[8], el[8];
  uint32_t hq[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    float x = fabsf(gv[u]);
#pragma unroll
    for (int o = 2; o < 32; o <<= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    am[u] = x;
  }
  if (lane < 2)
#pragma unroll
    for (int u = 0; u < 8; ++u) s_x[q][lane][u] = am[u];
  pair_bar(q);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    eh[u] = blk_exp(fmaxf(am[u], s_x[q ^ 1][odd][u]));
    sc[u] = ldexpf(gv[u], -eh[u]);
    hq[u] = e4m3x4(sc[u], 0.f, 0.f, 0.f) & 0xFFu;
    r[u] = sc[u] - e4m3x2_to_f2((uint16_t)hq[u]).x;
    float x = fabsf(r[u]);
#pragma unroll
    for (int o = 2; o < 32; o <<= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    am[u] = x;
  }
  if (lane < 2)
#pragma unroll
    for (int u = 0; u < 8; ++u) s_r[q][lane][u] = am[u];
  pair_bar(q);
  const int Kd = a.N >> 1, feat = f >> 1, blk = (nt * BM + (q >> 1) * 64) >> 6;  // 32-feature block
  const int64_t pitch = sf_pitch(a.qcap);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    el[u] = blk_exp(fmaxf(am[u], s_r[q ^ 1][odd][u]));
    const uint32_t lq = e4m3x4(ldexpf(r[u], -el[u]), 0.f, 0.f, 0.f) & 0xFFu;
    const int tok = c + (odd ? 8 : 0) + u;
    if (f < N && tok < nv) {
      a.qout[(int64_t)(row0 + tok) * Kd + feat] = (uint8_t)hq[u];
      a.qout[((int64_t)a.qcap + row0 + tok) * Kd + feat] = (uint8_t)lq;
    }
    if (lane < 2 && (q & 1) == 0 && tok < nv) {  // the block's first feature: its two scale bytes
      const int64_t w = (int64_t)(2 * (blk >> 2)) * pitch + row0 + tok;
      a.qsf[w * 4 + (blk & 3)] = (uint8_t)(eh[u] + 127);
      a.qsf[(w + pitch) * 4 + (blk & 3)] = (uint8_t)(eh[u] + el[u] + 127);
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(kMxThreads, 1) moe_gemm_mx_kernel(const __grid_constant__ CUtensorMap tm_w,
                                                                    const __grid_constant__ CUtensorMap tm_x,
                                                                    const uint32_t* __restrict__ xsf, int rows_cap,
                                                                    const MoeArgs a) {
  using CF = MxCfg<BN>;
  constexpr int WS = CF::WS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                   // [WS][128 rows][128 B] unpacked codes, SW128 (TMA)
  uint8_t* sx = sa + WS * CF::AB;       // [WS][2 BN rows][128 B] token halves, SW128 (TMA)
  uint8_t* ssa = sx + WS * CF::XB;      // [WS][512 B] weight scale words
  uint8_t* ssb = ssa + WS * 512;        // [2 items][KSB stages][512 B] token scale words
  uint64_t* w_full = reinterpret_cast<uint64_t*>(ssb + 2 * CF::SFB_ITEM);  // both producers (TMA bytes)
  uint64_t* w_empty = w_full + WS;      // MMA -> both producers
  uint64_t* b_full = w_empty + WS;      // [2] stager -> MMA (an item's token scale words)
  uint64_t* b_empty = b_full + 2;       // [2] MMA -> stager
  uint64_t* acc_full = b_empty + 2;     // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  __shared__ int s_off[kMaxE + 1];
  __shared__ int s_item[kMaxE + 1];
  __shared__ int s_cnt[kMaxE];
  __shared__ float s_qx[4][2][8], s_qr[4][2][8];  // fused down-input split: block maxima of a warp pair

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = a.E, NT = ceil_div(a.N, BM), KS = ceil_div(a.K, MX_BK);
  const int pitch = sf_pitch(rows_cap);
  if (threadIdx.x == 0) {
    tma_prefetch(&tm_w);
    tma_prefetch(&tm_x);
    for (int s = 0; s < WS; ++s) {
      mbar_init(&w_full[s], 2);
      mbar_init(&w_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&b_full[b], 1);
      mbar_init(&b_empty[b], 1);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  pdl_wait();
  block_prefix(a.counts, E, s_off);
  if (threadIdx.x < kMaxE) s_cnt[threadIdx.x] = threadIdx.x < E ? s_off[threadIdx.x + 1] - s_off[threadIdx.x] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      s_item[e] = run;
      run += ceil_div(s_cnt[e], BN) * NT;
    }
    s_item[E] = run;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch();
  const uint32_t tmem = *tmem_slot;
  const int total = s_item[E];
  // item -> (expert, weight tile, token tile); token tiles of one weight tile on neighbouring CTAs
  auto decode = [&](int it, int& e, int& nt, int& m) {
    int lo = 0, hi = E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_item[mid] <= it) lo = mid; else hi = mid - 1;
    }
    e = lo;
    const int mt = ceil_div(s_cnt[e], BN);
    const int local = it - s_item[e];
    nt = local / mt;
    m = local - nt * mt;
  };

  if (warp == 0) {
    if (elect_one()) {
      int s = 0, ph = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        int e, nt, m;
        decode(it, e, nt, m);
        const int st0 = (e * NT + nt) * KS;
        for (int ks = 0; ks < KS; ++ks, s = s + 1 == WS ? 0 : s + 1, ph ^= s == 0) {
          mbar_wait(&w_empty[s], ph ^ 1);
          mbar_expect_tx(&w_full[s], 8192 + 512);
          tma_load_3d(sa + s * CF::AB, &tm_w, &w_full[s], 0, 0, st0 + ks);
          bulk_load(smem_u32(ssa + s * 512), a.w + (int64_t)(st0 + ks) * MX_STAGE + 8192, 512, &w_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (elect_one()) {
      int s = 0, ph = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        int e, nt, m;
        decode(it, e, nt, m);
        const int xrow = s_off[e] + m * BN;
        for (int ks = 0; ks < KS; ++ks, s = s + 1 == WS ? 0 : s + 1, ph ^= s == 0) {
          mbar_wait(&w_empty[s], ph ^ 1);
          mbar_expect_tx(&w_full[s], CF::XB);
          tma_load_2d(sx + s * CF::XB, &tm_x, &w_full[s], ks * MX_BK, xrow);
          tma_load_2d(sx + s * CF::XB + BN * MX_BK, &tm_x, &w_full[s], ks * MX_BK, rows_cap + xrow);
        }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // token-scale stager: word (l, c) of stage ks = the scale word of B row n = 32 c + l
    int j = 0;
    for (int it = blockIdx.x; it < total; it += gridDim.x, ++j) {
      int e, nt, m;
      decode(it, e, nt, m);
      const int xrow = s_off[e] + m * BN;
      const int ib = j & 1;
      mbar_wait(&b_empty[ib], ((j >> 1) & 1) ^ 1);
      const uint32_t base = smem_u32(ssb + ib * CF::SFB_ITEM);
      // all of a batch's loads in flight at once (one L2 round trip per batch): 24 stages x 1 column
      // at BN = 16, 12 x 2 at BN = 32, 6 x 4 at BN = 64
      constexpr int C = CF::SFB_COLS, U = 24 / C;
      for (int ks0 = 0; ks0 < KS; ks0 += U) {
        uint32_t v[U][C];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int n = 32 * c + lane, h = n >= BN, tok = n - h * BN, row = xrow + tok;
            v[u][c] = (ks0 + u < KS && n < 2 * BN && row < rows_cap)
                          ? __ldg(xsf + (int64_t)(2 * (ks0 + u) + h) * pitch + row) : 0x7f7f7f7fu;
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ks0 + u < KS)
            sts128(base + (ks0 + u) * 512 + lane * 16, v[u][0], C > 1 ? v[u][C > 1 ? 1 : 0] : 0x7f7f7f7fu,
                   C > 2 ? v[u][C > 2 ? 2 : 0] : 0x7f7f7f7fu, C > 3 ? v[u][C > 3 ? 3 : 0] : 0x7f7f7f7fu);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_full[ib]);
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_mx(BM, 2 * BN);
      const uint32_t sa0 = smem_u32(sa), sx0 = smem_u32(sx), ssa0 = smem_u32(ssa);
      int s = 0, ph = 0, slot = 0, j = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x, ++j) {
        const int buf = j & 1;
        mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        mbar_wait(&b_full[buf], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * CF::ACC_COLS;
        uint32_t sbi = smem_u32(ssb + buf * CF::SFB_ITEM);
        for (int ks = 0; ks < KS; ++ks, s = s + 1 == WS ? 0 : s + 1, ph ^= s == 0, sbi += 512) {
          mbar_wait(&w_full[s], ph);
          tc_fence_after();
          const uint32_t sfa = tmem + CF::SF0 + slot * CF::SFS, sfb = sfa + 4;
          slot = (slot + 1) & (CF::SLOTS - 1);
          tc_cp_sf(sfa, ssa0 + s * 512);
          tc_cp_sf(sfb, sbi);
          const uint64_t adesc = umma_desc_kmajor_sw128(sa0 + s * CF::AB, 1024);
          const uint64_t bdesc = umma_desc_kmajor_sw128(sx0 + s * CF::XB, 1024);
          // always 4 slices of 32: a last stage of 64 of K reads zero codes and zero token bytes
#ifdef STB_MX_SKIP_MMA  // timing experiments only (results are wrong)
          if (ks == 0)
#endif
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // +32 B along K in both descriptors
            const int acc = CF::NACC == 2 ? (kk & 1) : 0;
            umma_mx(d + acc * 2 * BN, adesc + 2 * kk, bdesc + 2 * kk,
                    idesc | ((uint32_t)kk << 29) | ((uint32_t)kk << 4), sfa | ((uint32_t)kk << 30),
                    sfb | ((uint32_t)kk << 30), (ks > 0 || kk > acc) ? 1u : 0u);
          }
          umma_commit(&w_empty[s]);
        }
        umma_commit(&acc_full[buf]);
        umma_commit(&b_empty[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: thread = weight row (feature); columns = tokens (hi half + lo half)
    const int q = warp & 3;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int j = 0;
    for (int it = blockIdx.x; it < total; it += gridDim.x, ++j) {
      int e, nt, m;
      decode(it, e, nt, m);
      const int buf = j & 1;
      const int row0 = s_off[e] + m * BN;
      const int nv = min(BN, s_cnt[e] - m * BN);
      mbar_wait_sleep(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      const int f = nt * BM + q * 32 + lane;
      const float b = f < a.N ? __ldg(a.bias + (int64_t)e * a.N + f) : 0.f;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t rr[16], rl[16];
        const uint32_t cb = tmem + lane_addr + buf * CF::ACC_COLS + c;
        tmem_ld16(cb, rr);
        tmem_ld16(cb + BN, rl);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) rr[u] = __float_as_uint(__uint_as_float(rr[u]) + __uint_as_float(rl[u]));
        if constexpr (CF::NACC == 2) {
          tmem_ld16(cb + 2 * BN, rl);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 16; ++u) rr[u] = __float_as_uint(__uint_as_float(rr[u]) + __uint_as_float(rl[u]));
          tmem_ld16(cb + 3 * BN, rl);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 16; ++u) rr[u] = __float_as_uint(__uint_as_float(rr[u]) + __uint_as_float(rl[u]));
        }
        if (a.kind == 2) {
          float* y = reinterpret_cast<float*>(a.out);
          if (f < a.N) {
#pragma unroll
            for (int u = 0; u < 16; ++u)
              if (c + u < nv) y[(int64_t)(row0 + c + u) * a.ldo + f] = __uint_as_float(rr[u]) + b;
          }
        } else {
          __half* act = reinterpret_cast<__half*>(a.out);
          const bool odd = lane & 1;
          float gv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float mine = __uint_as_float(odd ? rr[8 + u] : rr[u]) + b;
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? rr[u] : rr[8 + u]) + b, 1);
            const int tok = c + (odd ? 8 : 0) + u;
            const float g = odd ? other : mine, up = odd ? mine : other;
            const bool ok = f < a.N && tok < nv;
            gv[u] = ok ? gpt_oss_glu(g, up, a.limit) : 0.f;
            if (ok && act) act[(int64_t)(row0 + tok) * a.ldo + (f >> 1)] = __float2half_rn(gv[u]);
          }
          if (a.qout) glu_quant_chunk(gv, q, lane, nt, f, a.N, c, nv, row0, a, s_qx, s_qr);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free(tmem, 512);
}

// fp16 token rows -> two e4m3 halves with one ue8m0 scale per 32 (the B operand of the block-scaled
// GEMM): per 32-wide block, s_hi = floor(log2 amax) - 7 (so |x| / 2^s_hi < 256 <= 448, exact
// power-of-two scaling), hi = e4m3(x / 2^s_hi), r = x / 2^s_hi - hi (exact in fp32), lo the same
// split of r. x = hi 2^s_hi + lo 2^(s_hi + s_lo) to the rounding of lo (about 2^-8 of the block
// maximum). Warp per (row, 128-wide stage); lane = 4 values; xq [2][rows_cap][K] (hi rows, then lo
// rows), xsf [stages][2][pitch] words of four scale bytes (blocks past K: 127, i.e. 1.0), pitch =
// rows_cap rounded up to 4 words (the GEMM reads them with a 2-D TMA box).
// one 128-wide stage of one token row, lane = 4 values (v): hi / lo codes and the scale words
__device__ __forceinline__ void quant_stage(const float* v, int lane, int ks, int K, int row, int rows_cap,
                                            uint8_t* __restrict__ xq, uint32_t* __restrict__ xsf) {
  const int k = ks * MX_BK + lane * 4;
  float am = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const int eh = blk_exp(am);
  float s[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) s[u] = ldexpf(v[u], -eh);
  const uint32_t hq = e4m3x4(s[0], s[1], s[2], s[3]);
  const float2 h01 = e4m3x2_to_f2((uint16_t)(hq & 0xFFFF)), h23 = e4m3x2_to_f2((uint16_t)(hq >> 16));
  float r[4] = {s[0] - h01.x, s[1] - h01.y, s[2] - h23.x, s[3] - h23.y};
  float ar = fmaxf(fmaxf(fabsf(r[0]), fabsf(r[1])), fmaxf(fabsf(r[2]), fabsf(r[3])));
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) ar = fmaxf(ar, __shfl_xor_sync(0xffffffffu, ar, o));
  const int el = blk_exp(ar);
  const uint32_t lq = e4m3x4(ldexpf(r[0], -el), ldexpf(r[1], -el), ldexpf(r[2], -el), ldexpf(r[3], -el));
  if (k < K) {
    *reinterpret_cast<uint32_t*>(xq + (int64_t)row * K + k) = hq;
    *reinterpret_cast<uint32_t*>(xq + ((int64_t)rows_cap + row) * K + k) = lq;
  }
  // block b = lane / 8: scale bytes of the four blocks gathered into lane 0
  const bool live = ks * MX_BK + (lane & ~7) * 4 < K;
  const uint32_t bh = live ? (uint32_t)(eh + 127) : 127u, bl = live ? (uint32_t)(eh + el + 127) : 127u;
  uint32_t wh = 0, wl = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    wh |= __shfl_sync(0xffffffffu, bh, 8 * b) << (8 * b);
    wl |= __shfl_sync(0xffffffffu, bl, 8 * b) << (8 * b);
  }
  if (lane == 0) {
    const int64_t pitch = sf_pitch(rows_cap);
    xsf[((int64_t)ks * 2) * pitch + row] = wh;
    xsf[((int64_t)ks * 2 + 1) * pitch + row] = wl;
  }

}

__global__ void __launch_bounds__(256) moe_quant_kernel(const __half* __restrict__ x, int64_t ldx, int rows, int K,
                                                        int rows_cap, uint8_t* __restrict__ xq,
                                                        uint32_t* __restrict__ xsf) {
  pdl_wait();
  pdl_launch();
  const int KS = (K + MX_BK - 1) / MX_BK;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < (int64_t)rows * KS; w += nw) {
    const int row = (int)(w / KS), ks = (int)(w - (int64_t)row * KS);
    const int k = ks * MX_BK + lane * 4;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (k < K) {
      const uint2 u = *reinterpret_cast<const uint2*>(x + row * ldx + k);
      const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
      const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
      v[0] = a0.x, v[1] = a0.y, v[2] = a1.x, v[3] = a1.y;
    }
    quant_stage(v, lane, ks, K, row, rows_cap, xq, xsf);
  }
}

// stb_moe_gather + stb_moe_quant in one pass for the gate-up input: offsets / perm as the gather,
// and the routed bf16 token rows split straight into the e4m3 halves (no fp16 copy)
__global__ void __launch_bounds__(256) moe_gather_mx_kernel(const __nv_bfloat16* __restrict__ h, int64_t ldh, int T,
                                                            int d, int k, int E, const int* __restrict__ counts,
                                                            const int* __restrict__ expert,
                                                            const int* __restrict__ rank, int* __restrict__ offsets,
                                                            int* __restrict__ perm, int rows_cap,
                                                            uint8_t* __restrict__ xq, uint32_t* __restrict__ xsf) {
  pdl_wait();
  pdl_launch();
  __shared__ int off[kMaxE + 1];
  block_prefix(counts, E, off);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += blockDim.x) offsets[e] = off[e];
  const int KS = (d + MX_BK - 1) / MX_BK;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < (int64_t)T * k * KS; w += nw) {
    const int p = (int)(w / KS), ks = (int)(w - (int64_t)p * KS);
    const int t = p / k;
    const int row = off[expert[p]] + rank[p];
    if (ks == 0 && lane == 0) perm[p] = row;
    const int c = ks * MX_BK + lane * 4;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (c < d) {
      const uint2 u = *reinterpret_cast<const uint2*>(h + (int64_t)t * ldh + c);
      const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
      const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
      v[0] = a0.x, v[1] = a0.y, v[2] = a1.x, v[3] = a1.y;
    }
    quant_stage(v, lane, ks, d, row, rows_cap, xq, xsf);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// token rows [rows][K], box [BN rows][128 B], 128B swizzle: fp16 (esize 2, the dequantising kernel)
// or e4m3 bytes (esize 1, the block-scaled kernel); cached per (base, rows, K, BN, esize, device)
int x_map(CUtensorMap* out, const void* base, int64_t rows, int K, int bn, int esize = 2) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int, int, int, int>, CUtensorMap> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(base, rows, K, bn, esize, dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STB_OK;
  }
  auto fn = encode_fn();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * esize};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esize), (cuuint32_t)bn};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "moe: tensor map encode failed (%d)", (int)r);
  if (cache.size() > 1024) cache.clear();
  cache.emplace(key, *out);
  return STB_OK;
}

template <int BN>
int launch_moe_gemm(const void* xperm, int rows_cap, const MoeArgs& a, cudaStream_t st) {
  CUtensorMap tm;
  if (int rc = x_map(&tm, xperm, rows_cap, a.K, BN)) return rc;
  auto kern = moe_gemm_mxfp4_kernel<BN>;
  smem_attr_once(kern, MCfg<BN>::SMEM);
  cudaError_t e = launch_k(kern, dim3(device_sms()), dim3(kThreads), MCfg<BN>::SMEM, st, tm, a);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_gemm launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

// MX weight stages of every expert of one projection as a 3-D map: [stages][128 rows][128 codes],
// rows 64 B apart, stages 8704 B apart; box = one stage, unpacked to 16-byte chunks (16U4_ALIGN16B)
int w_map(CUtensorMap* out, const void* base, int64_t stages) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int>, CUtensorMap> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(base, stages, dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STB_OK;
  }
  auto fn = encode_fn();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)MX_BK, (cuuint64_t)BM, (cuuint64_t)stages};
  cuuint64_t strides[2] = {(cuuint64_t)(MX_BK / 2), (cuuint64_t)MX_STAGE};
  cuuint32_t box[3] = {(cuuint32_t)MX_BK, (cuuint32_t)BM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "moe: weight tensor map encode failed (%d)", (int)r);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return STB_OK;
}

template <int BN>
int launch_moe_mx(const void* xq, const uint32_t* xsf, int rows_cap, const MoeArgs& a, cudaStream_t st) {
  CUtensorMap tw, tx;
  const int64_t stages = (int64_t)a.E * ((a.N + BM - 1) / BM) * ((a.K + MX_BK - 1) / MX_BK);
  if (int rc = w_map(&tw, a.w, stages)) return rc;
  if (int rc = x_map(&tx, xq, 2 * (int64_t)rows_cap, a.K, BN, 1)) return rc;
  auto kern = moe_gemm_mx_kernel<BN>;
  smem_attr_once(kern, MxCfg<BN>::SMEM);
  cudaError_t e = launch_k(kern, dim3(device_sms()), dim3(kMxThreads), MxCfg<BN>::SMEM, st, tw, tx, xsf, rows_cap, a);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_gemm_mx launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

}  // namespace

extern "C" {

int64_t stb_moe_quant_bytes(int rows_cap, int K) {
  if (rows_cap <= 0 || K <= 0) return 0;
  return 2 * (int64_t)rows_cap * K;
}
int64_t stb_moe_quant_scale_words(int rows_cap, int K) {
  if (rows_cap <= 0 || K <= 0) return 0;
  return (int64_t)((K + MX_BK - 1) / MX_BK) * 2 * sf_pitch(rows_cap) + 72;  // + the last tile's overhang
}

int stb_moe_quant(const void* x, int64_t ldx, int rows, int K, int rows_cap, void* xq, uint32_t* xsf, void* stream) {
  if (rows <= 0) return STB_OK;
  if (K % 4 || ldx % 4 || rows > rows_cap) return fail(STB_EINVAL, "moe_quant: rows=%d cap=%d K=%d", rows, rows_cap, K);
  const int64_t warps = (int64_t)rows * ((K + MX_BK - 1) / MX_BK);
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, (warps + 7) / 8), 8 * device_sms());
  cudaError_t e = launch_k(moe_quant_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, (const __half*)x, ldx,
                           rows, K, rows_cap, (uint8_t*)xq, xsf);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_quant launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

int stb_moe_gather_mx(const void* h, int64_t ldh, int T, int d, int k, int E, const int32_t* counts,
                      const int32_t* expert, const int32_t* rank, int32_t* offsets, int32_t* perm, int rows_cap,
                      void* xq, uint32_t* xsf, void* stream) {
  if (T <= 0) return STB_OK;
  if (E <= 0 || E > kMaxE || d % 4 || ldh % 4 || T * k > rows_cap)
    return fail(STB_EINVAL, "moe_gather_mx: E=%d d=%d rows=%d cap=%d", E, d, T * k, rows_cap);
  const int64_t warps = (int64_t)T * k * ((d + MX_BK - 1) / MX_BK);
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, (warps + 7) / 8), 4 * device_sms());
  cudaError_t e = launch_k(moe_gather_mx_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream,
                           (const __nv_bfloat16*)h, ldh, T, d, k, E, counts, expert, rank, offsets, perm, rows_cap,
                           (uint8_t*)xq, xsf);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_gather_mx launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

int stb_moe_gemm_mx_q(const void* xq, const uint32_t* xsf, int rows_cap, const void* wtiles, const float* bias,
                      const int32_t* counts, int E, int N, int K, int kind, float limit, void* out, int64_t ldo,
                      int rows, void* q_out, uint32_t* q_sf, int q_cap, void* stream) {
  if (rows <= 0) return STB_OK;
  if (E <= 0 || E > kMaxE || K % BK || K > MX_KS_MAX * MX_BK || N <= 0 ||
      (kind != STB_MOE_GATE_UP && kind != STB_MOE_DOWN) || (kind == STB_MOE_GATE_UP && N % 2) ||
      (reinterpret_cast<uintptr_t>(wtiles) & 15))
    return fail(STB_EINVAL, "moe_gemm_mx: E=%d N=%d K=%d kind=%d", E, N, K, kind);
  if (q_out != nullptr && (kind != STB_MOE_GATE_UP || q_sf == nullptr || q_cap < rows || (N / 2) % 64))
    return fail(STB_EINVAL, "moe_gemm_mx: the fused down-input split needs gate-up, N/2 %% 64 == 0, q_cap >= rows");
  if (q_out == nullptr && out == nullptr) return fail(STB_EINVAL, "moe_gemm_mx: no output");
  MoeArgs a{(const uint8_t*)wtiles, bias, counts, out, ldo, E, N, K, kind, limit, (uint8_t*)q_out, (uint8_t*)q_sf,
            q_cap};
  const double avg = (double)rows / E;
  const double busy = avg + 2.0 * std::sqrt(avg);
  cudaStream_t st = (cudaStream_t)stream;
  if (busy <= 16.0) return launch_moe_mx<16>(xq, xsf, rows_cap, a, st);
  if (busy <= 32.0) return launch_moe_mx<32>(xq, xsf, rows_cap, a, st);
  return launch_moe_mx<64>(xq, xsf, rows_cap, a, st);
}

int stb_moe_gemm_mx(const void* xq, const uint32_t* xsf, int rows_cap, const void* wtiles, const float* bias,
                    const int32_t* counts, int E, int N, int K, int kind, float limit, void* out, int64_t ldo, int rows,
                    void* stream) {
  return stb_moe_gemm_mx_q(xq, xsf, rows_cap, wtiles, bias, counts, E, N, K, kind, limit, out, ldo, rows, nullptr,
                           nullptr, 0, stream);
}

int stb_moe_route(const float* logits, int64_t ld, const float* bias, int T, int E, int k, int32_t* counts,
                  int32_t* expert, int32_t* rank, float* weight, void* stream) {
  if (T <= 0) return STB_OK;
  if (E <= 0 || E > kMaxE || k <= 0 || k > kMaxK || k > E) return fail(STB_EINVAL, "moe_route: E=%d k=%d", E, k);
  const int blocks = (T + 7) / 8;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (E <= 32)
    e = launch_k(moe_route_kernel<1>, dim3(blocks), dim3(256), 0, st, logits, ld, bias, T, E, k, counts, expert, rank, weight);
  else if (E <= 64)
    e = launch_k(moe_route_kernel<2>, dim3(blocks), dim3(256), 0, st, logits, ld, bias, T, E, k, counts, expert, rank, weight);
  else if (E <= 128)
    e = launch_k(moe_route_kernel<4>, dim3(blocks), dim3(256), 0, st, logits, ld, bias, T, E, k, counts, expert, rank, weight);
  else
    e = launch_k(moe_route_kernel<8>, dim3(blocks), dim3(256), 0, st, logits, ld, bias, T, E, k, counts, expert, rank, weight);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_route launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

int stb_moe_gather(const void* h, int64_t ldh, int T, int d, int k, int E, const int32_t* counts,
                   const int32_t* expert, const int32_t* rank, int32_t* offsets, int32_t* perm, void* xperm,
                   void* stream) {
  if (T <= 0) return STB_OK;
  if (E <= 0 || E > kMaxE || d % 8 || ldh % 8) return fail(STB_EINVAL, "moe_gather: E=%d d=%d", E, d);
  const int blocks = std::min(std::max(1, (T * k + 7) / 8), 4 * device_sms());
  cudaError_t e = launch_k(moe_gather_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream,
                           (const __nv_bfloat16*)h, ldh, T, d, k, E, counts, expert, rank, offsets, perm,
                           (__half*)xperm);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_gather launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

int stb_moe_gemm_mxfp4(const void* xperm, int rows_cap, const void* wtiles, const float* bias, const int32_t* counts,
                       int E, int N, int K, int kind, float limit, void* out, int64_t ldo, int rows, void* stream) {
  if (rows <= 0) return STB_OK;
  if (E <= 0 || E > kMaxE || K % BK || N <= 0 || (kind != STB_MOE_GATE_UP && kind != STB_MOE_DOWN) ||
      (kind == STB_MOE_GATE_UP && N % 2))
    return fail(STB_EINVAL, "moe_gemm: E=%d N=%d K=%d kind=%d", E, N, K, kind);
  MoeArgs a{(const uint8_t*)wtiles, bias, counts, out, ldo, E, N, K, kind, limit, nullptr, nullptr, 0};
  // token tile from the mean rows per expert: decode steps put ~T k / E <= a few rows on an
  // expert (BN 16); larger tiles only once experts hold tens of rows
  // (a busy expert holds ~mean + 2 sqrt(mean) rows: one token tile should cover it, or its
  // weights are streamed once per tile)
  const double avg = (double)rows / E;
  const double busy = avg + 2.0 * std::sqrt(avg);
  cudaStream_t st = (cudaStream_t)stream;
  if (busy <= 16.0) return launch_moe_gemm<16>(xperm, rows_cap, a, st);
  if (busy <= 32.0) return launch_moe_gemm<32>(xperm, rows_cap, a, st);
  return launch_moe_gemm<64>(xperm, rows_cap, a, st);
}

int stb_moe_combine(float* x, const float* y, int T, int d, int k, const int32_t* perm, const float* weight,
                    const void* norm_w, void* h_out, float eps, int32_t* counts, int E, void* stream) {
  if (T <= 0) return STB_OK;
  if (d % 4 || k > kMaxK) return fail(STB_EINVAL, "moe_combine: d=%d k=%d", d, k);
  cudaError_t e = launch_k(moe_combine_kernel, dim3(T), dim3(256), 0, (cudaStream_t)stream, x, y, d, k, perm, weight,
                           (const __nv_bfloat16*)norm_w, (__nv_bfloat16*)h_out, eps, counts, E);
  if (e != cudaSuccess) return fail(STB_ECUDA, "moe_combine launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

}  // extern "C"

#ifdef STB_MOE_PROF
extern "C" int stb_debug_moe_prof(unsigned long long* host16) {
  cudaMemcpyFromSymbol(host16, g_moe_prof, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_moe_prof, z, sizeof(z));
  return 0;
}
#endif
