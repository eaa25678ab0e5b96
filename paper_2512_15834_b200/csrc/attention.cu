// K3 — paged decode attention (one query per resident sequence), split-K over the
// context with a log-sum-exp merge; and the warp-tile append-prefill attention used
// for short query runs (verify passes, small ingests).
//
// Replaces the reference's decode charges (`engine.py:270,276,302,317`) and, for
// short runs, the validate/ingest charges (`engine.py:296,358`).
//
// HBM layout (include/stb200.h): per layer K and V pages [num_blocks][n_kv][16][D].
// One (block, kv-head) page is 16 x D bf16 = 4 KiB contiguous (D=128), so a page
// is fetched with 16-byte cp.async by one warp into a 128B-swizzled smem tile and
// consumed by ldmatrix + mma.sync (m16n8k16). GQA packing: the G = n_q / n_kv
// query heads that share a kv head are rows of one 16-row MMA tile, so each K/V
// page is read from HBM exactly once per step for the whole group. Softmax is
// online (exp2 domain) with quad shuffles; rows of one warp live in one quad.
#include <algorithm>
#include <cstdlib>

#include "../../include/stb200.h"
#include "common.cuh"
#include "pool.cuh"

using namespace stb;

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// byte offset of 16B chunk `c` of row `r` in a swizzled [16][D] page tile
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)(r * D * 2 + (((c & ~7) | ((c ^ r) & 7)) << 4));
}

// one warp copies a [16][D] K page and the matching V page into smem (swizzled)
template <int D>
__device__ __forceinline__ void load_page(uint32_t ks, uint32_t vs, const __nv_bfloat16* kp,
                                          const __nv_bfloat16* vp, int lane) {
  constexpr int CH = D / 8;            // 16B chunks per row
  constexpr int PER = 16 * CH / 32;    // chunks per lane per tile
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    int idx = i * 32 + lane;
    int r = idx / CH, c = idx % CH;
    // pages are pre-swizzled in HBM (pool.cuh): a linear copy lands them swizzled
    cp_async16(ks + (r * CH + c) * 16, kp + r * D + c * 8);
    cp_async16(vs + (r * CH + c) * 16, vp + r * D + c * 8);
  }
}

// Running softmax state of the 16 packed rows held by one warp (C-fragment layout:
// this lane owns rows lane/4 and lane/4+8).
template <int D>
struct RowState {
  float o[D / 8][4];
  float m[2];
  float l[2];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
  }
};

// S = Q K^T over one 16-key page, mask, online-softmax update, O += P V.
// qf: A fragments of the 16 x D query tile (pre-scaled by scale*log2e).
// lim0/lim1: number of valid keys of this page for rows lane/4 and lane/4+8
// (key k of the page is valid iff k < lim).
template <int D>
__device__ __forceinline__ void page_step(const uint32_t (*qf)[4], uint32_t ks, uint32_t vs, int lim0, int lim1,
                                          RowState<D>& st, int lane) {
  float s[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < D / 8; c0 += 4) {
      int r = nt * 8 + (lane & 7);
      int c = c0 + (lane >> 3);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(ks + swz<D>(r, c), b0, b1, b2, b3);
      mma_bf16_16816(s[nt], qf[c0 / 2], b0, b1);
      mma_bf16_16816(s[nt], qf[c0 / 2 + 1], b2, b3);
    }
  }
  // mask + row max (rows lane/4 -> s[*][0..1], lane/4+8 -> s[*][2..3])
  const int kc = (lane & 3) * 2;
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int k = nt * 8 + kc + j;
      if (k >= lim0) s[nt][j] = -INFINITY;
      if (k >= lim1) s[nt][2 + j] = -INFINITY;
      mx0 = fmaxf(mx0, s[nt][j]);
      mx1 = fmaxf(mx1, s[nt][2 + j]);
    }
  }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  float mn0 = fmaxf(st.m[0], mx0), mn1 = fmaxf(st.m[1], mx1);
  // fully masked rows keep a finite reference so exp2 never sees (-inf) - (-inf)
  float ref0 = mn0 == -INFINITY ? 0.f : mn0, ref1 = mn1 == -INFINITY ? 0.f : mn1;
  float a0 = exp2f(st.m[0] - ref0), a1 = exp2f(st.m[1] - ref1);
  st.m[0] = mn0;
  st.m[1] = mn1;
  float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      s[nt][j] = exp2f(s[nt][j] - ref0);
      s[nt][2 + j] = exp2f(s[nt][2 + j] - ref1);
      rs0 += s[nt][j];
      rs1 += s[nt][2 + j];
    }
  }
  st.l[0] = st.l[0] * a0 + rs0;
  st.l[1] = st.l[1] * a1 + rs1;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    st.o[n][0] *= a0;
    st.o[n][1] *= a0;
    st.o[n][2] *= a1;
    st.o[n][3] *= a1;
  }
  uint32_t pf[4];
  pf[0] = pack_bf16(s[0][0], s[0][1]);
  pf[1] = pack_bf16(s[0][2], s[0][3]);
  pf[2] = pack_bf16(s[1][0], s[1][1]);
  pf[3] = pack_bf16(s[1][2], s[1][3]);
#pragma unroll
  for (int d0 = 0; d0 < D / 8; d0 += 2) {
    int m = lane >> 3;
    int r = (m & 1) * 8 + (lane & 7);
    int c = d0 + (m >> 1);
    uint32_t b0, b1, b2, b3;
    ldsm_x4_t(vs + swz<D>(r, c), b0, b1, b2, b3);
    mma_bf16_16816(st.o[d0], pf, b0, b1);
    mma_bf16_16816(st.o[d0 + 1], pf, b2, b3);
  }
}

// NP consecutive pages (16*NP keys) per online-softmax update: S for all pages,
// one max / exp / rescale, then P V over NP k-steps. `lim0/lim1` count the valid
// keys of the chunk for the two rows this lane holds; full chunks skip masking.
template <int D, int NP>
__device__ __forceinline__ void chunk_step(const uint32_t (*qf)[4], uint32_t ks0, int lim0, int lim1, RowState<D>& st,
                                           int lane, int lo = 0) {
  constexpr int PAGE = 16 * D * 2;
  // pages past both rows' limits were never loaded: no S, no P V for them
  const int lim = lim0 > lim1 ? lim0 : lim1;
  float s[2 * NP][4];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const uint32_t ks = ks0 + p * 2 * PAGE;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      float* acc = s[p * 2 + nt];
      acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
      if (p > 0 && lim <= 16 * p) continue;
#pragma unroll
      for (int c0 = 0; c0 < D / 8; c0 += 4) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks + swz<D>(nt * 8 + (lane & 7), c0 + (lane >> 3)), b0, b1, b2, b3);
        mma_bf16_16816(acc, qf[c0 / 2], b0, b1);
        mma_bf16_16816(acc, qf[c0 / 2 + 1], b2, b3);
      }
    }
  }
  const int kc = (lane & 3) * 2;
  if (lim0 < 16 * NP || lim1 < 16 * NP || lo > 0) {  // lo: sliding-window start inside the chunk
#pragma unroll
    for (int t = 0; t < 2 * NP; ++t)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int k = t * 8 + kc + j;
        if (k >= lim0 || k < lo) s[t][j] = -INFINITY;
        if (k >= lim1 || k < lo) s[t][2 + j] = -INFINITY;
      }
  }
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int t = 0; t < 2 * NP; ++t) {
    mx0 = fmaxf(mx0, fmaxf(s[t][0], s[t][1]));
    mx1 = fmaxf(mx1, fmaxf(s[t][2], s[t][3]));
  }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  const float mn0 = fmaxf(st.m[0], mx0), mn1 = fmaxf(st.m[1], mx1);
  const float ref0 = mn0 == -INFINITY ? 0.f : mn0, ref1 = mn1 == -INFINITY ? 0.f : mn1;
  const float a0 = fast_exp2(st.m[0] - ref0), a1 = fast_exp2(st.m[1] - ref1);
  st.m[0] = mn0;
  st.m[1] = mn1;
  float rs0 = 0.f, rs1 = 0.f;
  uint32_t pf[NP][4];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      float* v = s[p * 2 + nt];
      v[0] = fast_exp2(v[0] - ref0);
      v[1] = fast_exp2(v[1] - ref0);
      v[2] = fast_exp2(v[2] - ref1);
      v[3] = fast_exp2(v[3] - ref1);
      rs0 += v[0] + v[1];
      rs1 += v[2] + v[3];
      pf[p][nt * 2 + 0] = pack_bf16(v[0], v[1]);
      pf[p][nt * 2 + 1] = pack_bf16(v[2], v[3]);
    }
  }
  st.l[0] = st.l[0] * a0 + rs0;
  st.l[1] = st.l[1] * a1 + rs1;
  if (a0 != 1.f || a1 != 1.f) {
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      st.o[n][0] *= a0;
      st.o[n][1] *= a0;
      st.o[n][2] *= a1;
      st.o[n][3] *= a1;
    }
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if (p > 0 && lim <= 16 * p) continue;
    const uint32_t vs = ks0 + p * 2 * PAGE + PAGE;
#pragma unroll
    for (int d0 = 0; d0 < D / 8; d0 += 2) {
      const int m = lane >> 3;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(vs + swz<D>((m & 1) * 8 + (lane & 7), d0 + (m >> 1)), b0, b1, b2, b3);
      mma_bf16_16816(st.o[d0], pf[p], b0, b1);
      mma_bf16_16816(st.o[d0 + 1], pf[p], b2, b3);
    }
  }
}

// Load a 16 x D query tile into A fragments; row r -> (src row pointer or null)
template <int D>
__device__ __forceinline__ void load_q(uint32_t (*qf)[4], const __nv_bfloat16* row_lo, const __nv_bfloat16* row_hi,
                                       float qscale, int lane) {
  const int kc = (lane & 3) * 2;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int col = ks * 16 + h * 8 + kc;
      float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
      if (row_lo) lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(row_lo + col));
      if (row_hi) hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(row_hi + col));
      qf[ks][h * 2 + 0] = pack_bf16(lo.x * qscale, lo.y * qscale);
      qf[ks][h * 2 + 1] = pack_bf16(hi.x * qscale, hi.y * qscale);
    }
  }
}

// ------------------------------------------------------------------ K3 decode
// Stream-K over pages: the units (b, kv-head, page) of the whole step are laid
// out b-major and cut into W equal contiguous ranges, one per warp (W = grid x 4,
// grid = 2 x SMs, persistent). A warp streams its pages through a private
// STAGES-deep cp.async ring *across* segment boundaries, keeping an online
// softmax per (b, kv-head) segment. A segment that covers its whole pair is
// written out directly; a pair split across warps gets a partial (o/l, lse)
// from each contributor and the last one to finish (ticket) merges them, so no
// separate merge launch and no wave tail, whatever the context lengths.
#ifndef STB_K3_MAXB
#define STB_K3_MAXB 1024
#endif
constexpr int kMaxB = STB_K3_MAXB;  // sequences per decode launch (static smem: ~16 B each)
#ifndef STB_K3_PAGES
#define STB_K3_PAGES 1
#endif
#ifndef STB_K3_WARPS
#define STB_K3_WARPS 8
#endif
constexpr int kChunkPages = STB_K3_PAGES;  // pages (16 keys each) per online-softmax update
constexpr int kDecWarps = STB_K3_WARPS;    // warps per CTA (one CTA per SM: smem-bound)
#ifndef STB_K3_MINCH
#define STB_K3_MINCH (8 / STB_K3_PAGES)
#endif
constexpr int kMinChunks = STB_K3_MINCH;  // fewest chunks (128 keys) a warp is given: bounds merge fan-in

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_of(int64_t u, int64_t U, int W) {
  return (int)(((u + 1) * W + U - 1) / U) - 1;  // largest w with floor(U*w/W) <= u
}

// QE > 1 (multi-query entries, stb_attn_decode_mq): entry b holds n_qs[b] <= QE consecutive
// query rows starting at packed row q_rows[b] — the last n_qs[b] positions of its context, each
// attending causally (query i of the entry sees keys < ctx - (n - 1 - i)). The 16-row MMA tile of
// a (entry, kv head) pair is then QE queries x G heads instead of one query's G heads (rows G..15
// of a decode tile are dead), so a short verify run rides in the decode launch: the entries of
// one run re-read the same pages from L2, and no separate prefill launch or merge is needed.
#ifdef STB_K3_TRACE
// timing experiments only: per warp {entry, partition done, first page landed, last chunk done,
// exit} in %globaltimer ns (stb_debug_k3_trace)
__device__ unsigned long long* g_k3t = nullptr;
__device__ unsigned int g_k3t_n = 0, g_k3t_cap = 0;
__device__ __forceinline__ unsigned long long k3_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K3T(i) k3t[i] = k3_now()
#else
#define K3T(i)
#endif
template <int D, int G, int QE, int STAGES>
__global__ void __launch_bounds__(32 * kDecWarps, 1) attn_decode_kernel(
    const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kpages,
    const __nv_bfloat16* __restrict__ vpages, const int32_t* __restrict__ table, int max_bps,
    const int32_t* __restrict__ slots, const int32_t* __restrict__ ctx_lens, int B, int n_kv, float qscale,
    float* __restrict__ o_part, float* __restrict__ lse_part, int* __restrict__ tickets, int window,
    const float* __restrict__ sinks, const int32_t* __restrict__ q_rows, const int32_t* __restrict__ n_qs,
    int32_t* __restrict__ plan, int plan_mode) {
  // plan_mode (the step's later layers reuse layer 0's work partition — same contexts, same grid):
  // 0 compute the partition here; 1 compute it and CTA 0 stores it in `plan`; 2 load it from
  // `plan` (stored by an earlier launch of the step: completed before this launch's prologue, by
  // the programmatic-dependency chain of the layers in between)
  constexpr int R = G * QE;  // live rows of an entry's 16-row tile (query-major: r = i * G + g)
  static_assert(R <= 16, "an entry's rows must fit one 16-row MMA tile");
  constexpr int PAGE = 16 * D * 2;
  constexpr int NP = kChunkPages;
  // sliding window (gpt-oss, window > 0): a sequence's keys are [kst, ctx), kst = max(0, ctx -
  // window); its chunks are counted from the chunk holding kst, so the partition, the page
  // fetches and the merge fan-in only ever see the window
  auto first_chunk = [&](int ctx) { return window > 0 ? max(0, ctx - window) / (16 * NP) : 0; };
  auto nchunks = [&](int ctx) { return (ctx + 16 * NP - 1) / (16 * NP) - first_chunk(ctx); };
  constexpr int STAGE = NP * 2 * PAGE;  // K and V of NP pages
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ int prefix[kMaxB + 1];  // chunk units before sequence b (< 2^31: B * n_kv * ctx/32)
  __shared__ int s_ctx[kMaxB], s_slot[kMaxB];
  __shared__ int s_qrow[QE > 1 ? kMaxB : 1], s_nq[QE > 1 ? kMaxB : 1];
  __shared__ int s_wbase[kMaxB + 1];  // pair-aligned partition: warps before sequence b
  __shared__ int s_wsum[kDecWarps], s_target;
  __shared__ __align__(8) uint64_t full_bars[kDecWarps * STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = n_kv * G;
#ifdef STB_K3_TRACE
  unsigned long long k3t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  K3T(0);
  auto k3_flush = [&]() {
    if (g_k3t != nullptr && lane == 0) {
      K3T(5);
      const unsigned slot = atomicAdd(&g_k3t_n, 1u);
      if (slot < g_k3t_cap)
        for (int j = 0; j < 8; ++j) g_k3t[(size_t)slot * 8 + j] = j == 7 ? (unsigned long long)(blockIdx.x * 64 + warp) : k3t[j];
    }
  };
#endif
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < kDecWarps * STAGES; ++s2) mbar_init(&full_bars[s2], 1);
    fence_mbar_init();
  }
  if (plan_mode == 2) {
    // plan layout: [T_al, W, prefix[0..B], wbase[0..B]]
    for (int b = threadIdx.x; b <= B; b += blockDim.x) {
      if (b < B) {
        s_ctx[b] = ctx_lens[b];
        s_slot[b] = slots[b];
        if constexpr (QE > 1) {
          s_qrow[b] = q_rows[b];
          s_nq[b] = n_qs[b];
        }
      }
      prefix[b] = __ldcg(plan + 2 + b);
      s_wbase[b] = __ldcg(plan + 3 + B + b);
    }
    if (threadIdx.x == 0) s_target = __ldcg(plan);
  } else {
    // step metadata (host-uploaded, not produced by the preceding kernel): all threads load
    // ctx / slot in parallel (a serial loop would chain B global-load latencies in front of
    // the first page copy), then a block scan gives the unit prefix
    const int per = (B + 32 * kDecWarps - 1) / (32 * kDecWarps), b0 = threadIdx.x * per;
    int local = 0;
    for (int j = 0; j < per; ++j) {
      const int b = b0 + j;
      if (b < B) {
        const int c = ctx_lens[b];
        s_ctx[b] = c;
        s_slot[b] = slots[b];
        if constexpr (QE > 1) {
          s_qrow[b] = q_rows[b];
          s_nq[b] = n_qs[b];
        }
        local += n_kv * nchunks(c);
      }
    }
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int run = incl - local;
    for (int w2 = 0; w2 < warp; ++w2) run += s_wsum[w2];
    for (int j = 0; j < per; ++j) {
      const int b = b0 + j;
      if (b < B) {
        prefix[b] = run;
        run += n_kv * nchunks(s_ctx[b]);
      }
    }
    if (threadIdx.x == 32 * kDecWarps - 1) prefix[B] = run;
  }
  __syncthreads();
#ifdef STB_K3_TRACE
  K3T(6);
#endif
  pdl_launch();
  const int64_t U = prefix[B];
  // Work partition. Pair-aligned when it fits: every (sequence, kv head) pair is cut into
  // k_b = ceil(chunks_b / T) equal parts, one per warp, with the smallest chunk target T
  // (>= kMinChunks) for which all parts fit in the grid's warps — so no warp ever switches
  // pairs mid-stream (q reload, partial write, second merge) and merges are k_b-way. The
  // kernel is HBM-bound, so the uneven part lengths (T/2..T chunks) cost nothing while
  // enough pages are in flight. Otherwise (more pairs than warps): equal contiguous ranges
  // of the unit space, segments crossing pair boundaries.
  const int Wmax = gridDim.x * kDecWarps;
  if (warp == 0 && plan_mode != 2) {  // one warp, shuffles only (no block barriers inside the search)
    auto chunks = [&](int b) { return nchunks(s_ctx[b]); };
    auto count = [&](int T) {  // warps the pair-aligned cut with target T needs
      int c = 0;
      for (int b = lane; b < B; b += 32) c += n_kv * ((chunks(b) + T - 1) / T);
      return warp_sum_i(c);
    };
    int maxch = 0;
    for (int b = lane; b < B; b += 32) maxch = max(maxch, chunks(b));
    maxch = warp_max_i(maxch);
    int lo = (int)max((int64_t)kMinChunks, (U + Wmax - 1) / Wmax), hi = max(lo, maxch);
    const bool fits = count(hi) <= Wmax;
    if (fits) {
      while (lo < hi) {  // smallest T with count(T) <= Wmax (count is non-increasing in T)
        const int mid = (lo + hi) >> 1;
        if (count(mid) <= Wmax) hi = mid; else lo = mid + 1;
      }
      int run = 0;  // warps before sequence b, 32 sequences per pass
      for (int b0 = 0; b0 < B; b0 += 32) {
        const int b = b0 + lane;
        const int k = b < B ? n_kv * ((chunks(b) + lo - 1) / lo) : 0;
        int incl = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (b < B) s_wbase[b] = run + incl - k;
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) s_wbase[B] = run;
    }
    if (lane == 0) s_target = fits ? lo : 0;
  }
  __syncthreads();
  const int T_al = s_target;  // > 0: pair-aligned partition with chunk target T_al
  const int W = T_al ? s_wbase[B] : (int)max((int64_t)1, min((int64_t)Wmax, U / kMinChunks));
  if (plan_mode == 1 && blockIdx.x == 0) {  // store the partition for the step's later layers
    for (int b = threadIdx.x; b <= B; b += blockDim.x) {
      plan[2 + b] = prefix[b];
      plan[3 + B + b] = T_al ? s_wbase[b] : 0;
    }
    if (threadIdx.x == 0) {
      plan[0] = T_al;
      plan[1] = W;
    }
  }
  // logical warp ids run across CTAs first: a partition that leaves warps idle (pair-aligned
  // cuts use e.g. 1024 of 1184) spreads its busy warps over every SM instead of idling whole
  // SMs (measured: decode step 4.81 -> 4.78 ms at B=32 ctx 2k)
  const int w = warp * gridDim.x + blockIdx.x;
#ifdef STB_K3_TRACE
  K3T(1);
  if (w >= W) { k3_flush(); return; }
#else
  if (w >= W) return;
#endif
  int64_t u0, u1;
  if (T_al) {
    int lo = 0, hi = B - 1;  // sequence of warp w
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_wbase[mid] <= w) lo = mid; else hi = mid - 1;
    }
    const int ch = nchunks(s_ctx[lo]);
    const int k = (ch + T_al - 1) / T_al;
    const int r = w - s_wbase[lo], kh = r / k, part = r % k;
    const int64_t pbase = prefix[lo] + (int64_t)kh * ch;
    u0 = pbase + (int64_t)ch * part / k;
    u1 = pbase + (int64_t)ch * (part + 1) / k;
  } else {
    u0 = U * w / W;
    u1 = U * (w + 1) / W;
  }
  const int n = (int)(u1 - u0);
#ifdef STB_K3_TRACE
  if (n <= 0) { k3_flush(); return; }
#else
  if (n <= 0) return;
#endif

  // cursor over (b, kh, chunk) — located once by binary search, then incremented;
  // the pair's block-table row and length are cached when the cursor enters it
  struct Cur {
    int b, kh, c, chunks, ctx, c0;  // c counts from the sequence's first chunk c0 (sliding window)
    const int32_t* row;
  };
  auto enter = [&](Cur& r) {
    r.ctx = s_ctx[r.b];
    r.c0 = first_chunk(r.ctx);
    r.chunks = nchunks(r.ctx);
    r.row = table + (int64_t)s_slot[r.b] * max_bps;
  };
  auto locate = [&](int64_t u) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= u) lo = mid; else hi = mid - 1;
    }
    Cur r;
    r.b = lo;
    enter(r);
    const int rem = (int)(u - prefix[lo]);
    r.kh = rem / r.chunks;
    r.c = rem - r.kh * r.chunks;
    return r;
  };
  auto advance = [&](Cur& r) {
    if (++r.c < r.chunks) return;
    r.c = 0;
    if (++r.kh < n_kv) return;
    r.kh = 0;
    do {
      ++r.b;
      if (r.b < B) enter(r);
    } while (r.b < B && r.chunks == 0);
  };
  // K/V pages arrive by bulk copy (one lane, 4 KiB each) into a per-warp STAGES ring;
  // full[s] counts the bytes. Page ids are fetched one chunk ahead of their copy.
  const uint32_t wbase = smem_u32(smem) + warp * STAGES * STAGE;
  uint64_t* full = full_bars + warp * STAGES;
  int pid[NP];
  auto fetch = [&](const Cur& r) {
    const int npages = (r.ctx + 15) >> 4;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int page = (r.c0 + r.c) * NP + p;
      pid[p] = page < npages ? __ldg(r.row + page) : -1;
    }
  };
  auto issue = [&](const Cur& r, int i, const int* ids) {  // lane 0
    const uint32_t sb = wbase + (i % STAGES) * STAGE;
    uint32_t bytes = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) bytes += ids[p] >= 0 ? 2 * PAGE : 0;
    uint64_t* bar = full + (i % STAGES);
    mbar_expect_tx(bar, bytes);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (ids[p] >= 0) {
        const int64_t off = (((int64_t)ids[p] * n_kv + r.kh) * 16) * D;
        bulk_load(sb + p * 2 * PAGE, kpages + off, PAGE, bar);
        bulk_load(sb + p * 2 * PAGE + PAGE, vpages + off, PAGE, bar);
      }
    }
  };
  // Prologue before the dependency wait: every page except the one K1 writes in this
  // layer (the last page of each pair, inside the pair's last chunk) was final before
  // the preceding kernel started, so those copies overlap its tail; chunks holding a
  // pair's last page are issued after griddepcontrol.wait.
  Cur ld = locate(u0);
  Cur dcur[STAGES - 1];
  int dpid[STAGES - 1][NP];
  int deferred = 0;
  if (lane == 0) {
    fetch(ld);
#pragma unroll
    for (int s2 = 0; s2 < STAGES - 1; ++s2) {
      if (s2 < n) {
#ifndef STB_MQ_NODEFER
        if (QE > 1 || ld.c == ld.chunks - 1) {  // multi-query entries: a run's new rows span pages
#else
        if (ld.c == ld.chunks - 1) {
#endif
          deferred |= 1 << s2;
          dcur[s2] = ld;
#pragma unroll
          for (int p = 0; p < NP; ++p) dpid[s2][p] = pid[p];
        } else {
          issue(ld, s2, pid);
        }
        advance(ld);
        fetch(ld);
      }
    }
  }
  pdl_wait();  // q and this layer's newest K/V rows come from the preceding kernel
  if (lane == 0) {
#pragma unroll
    for (int s2 = 0; s2 < STAGES - 1; ++s2)
      if (deferred & (1 << s2)) issue(dcur[s2], s2, dpid[s2]);
  }
  Cur cu = locate(u0);
  // row r of pair (b, kh): query r / G of the entry (always 0 for decode entries), head r % G
  auto live = [&](int b, int r) { return QE > 1 ? (r < R && r / G < s_nq[b]) : r < G; };
  auto row_off = [&](int b, int kh, int r) -> int64_t {
    const int qrow = QE > 1 ? s_qrow[b] + r / G : b;
    return ((int64_t)qrow * n_q + kh * G + r % G) * D;
  };
  static_assert(QE == 1 || kChunkPages == 1, "multi-query entries need one page per chunk (warp-uniform limits)");
  uint32_t qf[D / 16][4];
  RowState<D> st;
  bool open = false;
  int seg_first = 0, seg_ctx = 0;
  int64_t seg_start = u0;
  for (int i = 0; i < n; ++i) {
    if (!open) {
      open = true;
      seg_first = cu.c;
      seg_ctx = cu.ctx;
      seg_start = u0 + i;
      const int r0 = lane >> 2, r1 = r0 + 8;
      load_q<D>(qf, live(cu.b, r0) ? q + row_off(cu.b, cu.kh, r0) : nullptr,
                live(cu.b, r1) ? q + row_off(cu.b, cu.kh, r1) : nullptr, qscale, lane);
      st.init();
    }
    mbar_wait(full + (i % STAGES), (uint32_t)(i / STAGES) & 1u);
#ifdef STB_K3_TRACE
    if (i == 0) K3T(2);
#endif
    const int kbase = (cu.c0 + cu.c) * 16 * NP;
    const int lim = seg_ctx - kbase;
    const int lo = window > 0 ? max(0, seg_ctx - window) - kbase : 0;
    int lim0 = lim, lim1 = lim;
    if constexpr (QE > 1) {  // query i of an n-query entry sees keys < ctx - (n - 1 - i)
      const int nq = s_nq[cu.b], r0 = lane >> 2, r1 = r0 + 8;
      if (r0 < R && r0 / G < nq) lim0 = lim - (nq - 1 - r0 / G);
      if (r1 < R && r1 / G < nq) lim1 = lim - (nq - 1 - r1 / G);
    }
    chunk_step<D, NP>(qf, wbase + (i % STAGES) * STAGE, lim0, lim1, st, lane, lo);
    __syncwarp();  // every lane's ldmatrix reads of the slot refilled below are done
    if (lane == 0 && i + STAGES - 1 < n) {
      fence_proxy_async_smem();
      issue(ld, i + STAGES - 1, pid);
      advance(ld);
      fetch(ld);
    }
    const bool pair_end = cu.c == cu.chunks - 1;
    if (pair_end || i == n - 1) {
      // close the segment of pair (cu.b, cu.kh)
      float l0 = st.l[0], l1 = st.l[1];
      l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
      l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      const int r0 = lane >> 2, r1 = r0 + 8;
      const int sb = cu.b, skh = cu.kh;
      const bool whole = seg_first == 0 && pair_end;
#ifdef STB_MQ_DEBUG
      if (QE > 1 && lane == 0 && cu.kh == 0)
        printf("close b=%d kh=%d w=%d whole=%d seg_first=%d chunks=%d c=%d i=%d n=%d T_al=%d W=%d\n", cu.b, cu.kh, w,
               (int)whole, seg_first, cu.chunks, cu.c, i, n, T_al, W);
#endif
      if (whole && sinks != nullptr) {  // the sink's exp(logit) joins the denominator (log2 domain)
        if (live(sb, r0)) l0 += fast_exp2(sinks[skh * G + r0 % G] * kLog2e - st.m[0]);
        if (live(sb, r1)) l1 += fast_exp2(sinks[skh * G + r1 % G] * kLog2e - st.m[1]);
      }
      const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
      if (whole) {
#pragma unroll
        for (int nd = 0; nd < D / 8; ++nd) {
          const int c = nd * 8 + (lane & 3) * 2;
          if (live(sb, r0))
            *reinterpret_cast<uint32_t*>(out + row_off(sb, skh, r0) + c) = pack_bf16(st.o[nd][0] * inv0, st.o[nd][1] * inv0);
          if (live(sb, r1))
            *reinterpret_cast<uint32_t*>(out + row_off(sb, skh, r1) + c) = pack_bf16(st.o[nd][2] * inv1, st.o[nd][3] * inv1);
        }
      } else {
        const int slot = w * 2 + (seg_start == u0 ? 0 : 1);
        float* op = o_part + (int64_t)slot * R * D;
#pragma unroll
        for (int nd = 0; nd < D / 8; ++nd) {
          const int c = nd * 8 + (lane & 3) * 2;
          if (r0 < R)
            __stcg(reinterpret_cast<float2*>(op + r0 * D + c), make_float2(st.o[nd][0] * inv0, st.o[nd][1] * inv0));
          if (r1 < R)
            __stcg(reinterpret_cast<float2*>(op + r1 * D + c), make_float2(st.o[nd][2] * inv1, st.o[nd][3] * inv1));
        }
        if ((lane & 3) == 0) {
          if (r0 < R) __stcg(lse_part + slot * R + r0, l0 > 0.f ? st.m[0] + log2f(l0) : -INFINITY);
          if (r1 < R) __stcg(lse_part + slot * R + r1, l1 > 0.f ? st.m[1] + log2f(l1) : -INFINITY);
        }
        __threadfence();
        __syncwarp();
        const int64_t pstart = prefix[sb] + (int64_t)skh * cu.chunks;
        int wf, wl;
        if (T_al) {  // the pair's k consecutive warps
          const int k = (cu.chunks + T_al - 1) / T_al;
          wf = s_wbase[sb] + skh * k;
          wl = wf + k - 1;
        } else {
          wf = warp_of(pstart, U, W);
          wl = warp_of(pstart + cu.chunks - 1, U, W);
        }
        int last = 0;
        if (lane == 0) last = atomicAdd(&tickets[sb * n_kv + skh], 1) == wl - wf;
        last = __shfl_sync(0xffffffffu, last, 0);
#ifdef STB_MQ_DEBUG
        if (QE > 1 && lane == 0 && skh == 0)
          printf("seg b=%d kh=%d w=%d wf=%d wl=%d ticket_last=%d qrow=%d nq=%d live0=%d off0=%lld\n", sb, skh, w, wf, wl,
                 last, s_qrow[sb], s_nq[sb], (int)live(sb, 0), (long long)row_off(sb, skh, 0));
#endif
        if (last) {
          __threadfence();
          // merge the nc partials of this pair: lanes own contributors for the LSE
          // reductions, then every lane accumulates D/32 dims of all G rows with the
          // contributor loop unrolled so the partial loads overlap
          const int nc = wl - wf + 1;
          auto part = [&](int c) {
            return c * 2 + ((!T_al && c == wf && (U * c / W) < pstart) ? 1 : 0);
          };
          // rows in groups of RG (a multi-query entry's 16 rows would not fit the registers at
          // once); groups whose first row is a dead query are skipped
          constexpr int RG = QE > 1 ? 4 : R;
#pragma unroll 1
          for (int rg = 0; rg < R; rg += RG) {
            if (QE > 1 && !live(sb, rg)) continue;
            float M[RG], L[RG], wt_l[RG];
#pragma unroll
            for (int r = 0; r < RG; ++r) M[r] = -INFINITY, L[r] = 0.f, wt_l[r] = 0.f;
            for (int j = lane; j < nc; j += 32) {
              const int sl = part(wf + j);
#pragma unroll
              for (int r = 0; r < RG; ++r) M[r] = fmaxf(M[r], __ldcg(lse_part + sl * R + rg + r));
            }
#pragma unroll
            for (int r = 0; r < RG; ++r)
#pragma unroll
              for (int o = 16; o; o >>= 1) M[r] = fmaxf(M[r], __shfl_xor_sync(0xffffffffu, M[r], o));
            for (int j = lane; j < nc; j += 32) {
              const int sl = part(wf + j);
#pragma unroll
              for (int r = 0; r < RG; ++r) {
                const float wt = M[r] == -INFINITY ? 0.f : exp2f(__ldcg(lse_part + sl * R + rg + r) - M[r]);
                L[r] += wt;
                if (j < 32) wt_l[r] = wt;
              }
            }
#pragma unroll
            for (int r = 0; r < RG; ++r)
#pragma unroll
              for (int o = 16; o; o >>= 1) L[r] += __shfl_xor_sync(0xffffffffu, L[r], o);
            if (sinks != nullptr) {
#pragma unroll
              for (int r = 0; r < RG; ++r) L[r] += exp2f(sinks[skh * G + (rg + r) % G] * kLog2e - M[r]);
            }
            float acc[RG][D / 32];
#pragma unroll
            for (int r = 0; r < RG; ++r)
#pragma unroll
              for (int j = 0; j < D / 32; ++j) acc[r][j] = 0.f;
#pragma unroll 4
            for (int c = 0; c < nc; ++c) {
              const int sl = part(wf + c);
#pragma unroll
              for (int r = 0; r < RG; ++r) {
                float wt = __shfl_sync(0xffffffffu, wt_l[r], c & 31);
                if (c >= 32) wt = M[r] == -INFINITY ? 0.f : exp2f(__ldcg(lse_part + sl * R + rg + r) - M[r]);
#pragma unroll
                for (int j = 0; j < D / 32; ++j)
                  acc[r][j] += wt * __ldcg(o_part + ((int64_t)sl * R + rg + r) * D + j * 32 + lane);
              }
            }
#pragma unroll
            for (int r = 0; r < RG; ++r) {
              if (!live(sb, rg + r)) continue;
#pragma unroll
              for (int j = 0; j < D / 32; ++j)
                out[row_off(sb, skh, rg + r) + j * 32 + lane] =
                    __float2bfloat16_rn(L[r] > 0.f ? acc[r][j] / L[r] : 0.f);
            }
          }
          if (lane == 0) tickets[sb * n_kv + skh] = 0;
        }
      }
      open = false;
    }
#ifdef STB_K3_TRACE
    if (i == n - 1) K3T(3);  // (after the last segment's close: its merge, if this warp merged)
#endif
    advance(cu);
  }
#ifdef STB_K3_TRACE
  k3_flush();
#endif
}

// ---------------------------------------------------------- short-run prefill
// grid: (q tiles, n_kv, S); 4 warps share each K/V page (CTA-wide cp.async), each
// warp owns 16 packed rows = 16/G queries x G heads. Rows are (query i, head g)
// with r = i*G + g. Causal: row's query at position qpos attends keys <= qpos.
template <int D, int G, int STAGES>
__global__ void __launch_bounds__(128) attn_prefill_kernel(
    const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ kpages,
    const __nv_bfloat16* __restrict__ vpages, const int32_t* __restrict__ table, int max_bps,
    const int32_t* __restrict__ slots, const int32_t* __restrict__ q_start, const int32_t* __restrict__ ctx_lens,
    int n_kv, float qscale) {
  pdl_wait();
  pdl_launch();
  constexpr int PAGE = 16 * D * 2;
  constexpr int QPW = 16 / G;  // queries per warp tile
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.z, kh = blockIdx.y;
  const int n_q = n_kv * G;
  const int t0 = q_start[s], n = q_start[s + 1] - t0;
  const int qbase = blockIdx.x * 4 * QPW;  // first query of this CTA
  if (qbase >= n) return;
  const int ctx = ctx_lens[s];
  const int pos0 = ctx - n;  // absolute position of query 0
  const int32_t* row = table + (int64_t)slots[s] * max_bps;

  const int wq0 = qbase + warp * QPW;  // first query of this warp
  uint32_t qf[D / 16][4];
  int qi_lo = wq0 + (lane >> 2) / G, qi_hi = wq0 + ((lane >> 2) + 8) / G;
  int g_lo = (lane >> 2) % G, g_hi = ((lane >> 2) + 8) % G;
  {
    const __nv_bfloat16* lo = qi_lo < n ? q + ((int64_t)(t0 + qi_lo) * n_q + kh * G + g_lo) * D : nullptr;
    const __nv_bfloat16* hi = qi_hi < n ? q + ((int64_t)(t0 + qi_hi) * n_q + kh * G + g_hi) * D : nullptr;
    load_q<D>(qf, lo, hi, qscale, lane);
  }
  RowState<D> st;
  st.init();
  // the CTA needs keys up to the last query it owns
  const int last_q = min(n, qbase + 4 * QPW) - 1;
  const int npages = (pos0 + last_q) / 16 + 1;
  const int lim_lo_abs = qi_lo < n ? pos0 + qi_lo + 1 : 0;  // keys < lim are visible
  const int lim_hi_abs = qi_hi < n ? pos0 + qi_hi + 1 : 0;
  const int warp_last = min(n - 1, wq0 + QPW - 1);
  const int warp_pages = wq0 < n ? (pos0 + warp_last) / 16 + 1 : 0;

  const uint32_t base = smem_u32(smem);
  auto issue = [&](int p, int stage) {
    // 128 threads copy one K page and one V page
    constexpr int CH = D / 8;
    const __nv_bfloat16* kp = kpages + (((int64_t)row[p] * n_kv + kh) * 16) * D;
    const __nv_bfloat16* vp = vpages + (((int64_t)row[p] * n_kv + kh) * 16) * D;
    uint32_t ks = base + stage * 2 * PAGE, vs = ks + PAGE;
    for (int idx = threadIdx.x; idx < 16 * CH; idx += 128) {
      int r = idx / CH, c = idx % CH;
      cp_async16(ks + (r * D / 8 + c) * 16, kp + r * D + c * 8);  // pre-swizzled pages: linear copy
      cp_async16(vs + (r * D / 8 + c) * 16, vp + r * D + c * 8);
    }
  };
#pragma unroll
  for (int st_i = 0; st_i < STAGES - 1; ++st_i) {
    if (st_i < npages) issue(st_i, st_i);
    cp_async_commit();
  }
  for (int p = 0; p < npages; ++p) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    int stage = p % STAGES;
    if (p < warp_pages) {
      int lo = lim_lo_abs - p * 16, hi = lim_hi_abs - p * 16;
      page_step<D>(qf, base + stage * 2 * PAGE, base + stage * 2 * PAGE + PAGE, lo, hi, st, lane);
    }
    __syncthreads();
    int nx = p + STAGES - 1;
    if (nx < npages) issue(nx, nx % STAGES);
    cp_async_commit();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    st.l[j] += __shfl_xor_sync(0xffffffffu, st.l[j], 1);
    st.l[j] += __shfl_xor_sync(0xffffffffu, st.l[j], 2);
  }
  float inv0 = st.l[0] > 0.f ? 1.f / st.l[0] : 0.f, inv1 = st.l[1] > 0.f ? 1.f / st.l[1] : 0.f;
#pragma unroll
  for (int nd = 0; nd < D / 8; ++nd) {
    int c = nd * 8 + (lane & 3) * 2;
    if (qi_lo < n) {
      __nv_bfloat16* o = out + ((int64_t)(t0 + qi_lo) * n_q + kh * G + g_lo) * D + c;
      *reinterpret_cast<uint32_t*>(o) = pack_bf16(st.o[nd][0] * inv0, st.o[nd][1] * inv0);
    }
    if (qi_hi < n) {
      __nv_bfloat16* o = out + ((int64_t)(t0 + qi_hi) * n_q + kh * G + g_hi) * D + c;
      *reinterpret_cast<uint32_t*>(o) = pack_bf16(st.o[nd][2] * inv1, st.o[nd][3] * inv1);
    }
  }
}

#ifndef STB_K3_STAGES
#define STB_K3_STAGES 3
#endif
constexpr int kDecodeStages = STB_K3_STAGES;
constexpr int kPrefillStages = 3;

// Per-device launch geometry of K3 (SM count, resident CTAs per SM), looked up once per
// (device, kernel instantiation) — never cached for the first device only.
constexpr int kMaxDevices = 64;
constexpr int kDecMaxPerSm = 2;

inline int decode_sms(int) { return device_sms(); }

// Caller workspace layout (stb_attn_decode_workspace): partial (o, lse) rows for every warp
// of the largest grid K3 can launch on this device, then the split-pair merge tickets
// (B * n_kv, after the stored partition; zeroed by the caller once; the merging warp resets its ticket, so the region
// is zero again after every launch). Nothing is allocated here: a CUDA graph captured for
// any B keeps pointing at the caller's buffer, whose growth the caller owns.
// Rows per partial slot are sized for the widest entry (16: a multi-query entry's full tile), so
// decode-only and multi-query launches share one workspace and one ticket offset.
constexpr int kPartRows = 16;
// the step's stored K3 partition (plan_mode 1 / 2) sits between the partials and the tickets, at
// an offset independent of B (the tickets region must stay zero for any later, larger B)
constexpr int kPlanInts = 2 * kMaxB + 8;
inline size_t decode_part_floats(int sms, int D) {
  return (size_t)kDecMaxPerSm * sms * kDecWarps * 2 * kPartRows * (D + 1);
}

template <int D, int G, int QE>
int launch_decode(const __nv_bfloat16* q, __nv_bfloat16* out, const __nv_bfloat16* kp, const __nv_bfloat16* vp,
                  const int32_t* table, int max_bps, const int32_t* slots, const int32_t* ctx, int B, int n_kv,
                  float qscale, int window, const float* sinks, const int32_t* q_rows, const int32_t* n_qs,
                  int plan_mode, void* work, cudaStream_t st) {
  if (B > kMaxB) return fail(STB_EINVAL, "attn_decode: at most %d sequences per step", kMaxB);
  if (!work) return fail(STB_EINVAL, "attn_decode: NULL workspace");
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = decode_sms(dev);
  constexpr size_t smem = (size_t)kDecWarps * kDecodeStages * kChunkPages * 2 * 16 * D * 2;
  auto kern = attn_decode_kernel<D, G, QE, kDecodeStages>;
  static int per_sm_of[kMaxDevices] = {};
  int& per_sm = per_sm_of[dev < kMaxDevices ? dev : 0];
  if (!per_sm) {
    smem_attr_once(kern, (int)smem);
    int n = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32 * kDecWarps, smem) != cudaSuccess || n < 1) n = 1;
    per_sm = std::min(n, kDecMaxPerSm);
  }
  smem_attr_once(kern, (int)smem);
  const int grid = per_sm * sms;
  const int W = grid * kDecWarps;
  constexpr int R = G * QE;
  float* o_part = (float*)work;
  float* lse_part = o_part + (size_t)W * 2 * R * D;
  int32_t* plan = (int32_t*)(o_part + decode_part_floats(sms, D));  // [T_al, W, prefix[B+1], wbase[B+1]]
  int* tickets = plan + kPlanInts;
  cudaError_t e = launch_k(kern, dim3(grid), dim3(32 * kDecWarps), smem, st, q, out, kp, vp, table, max_bps, slots, ctx,
                           B, n_kv, qscale, o_part, lse_part, tickets, window, sinks, q_rows, n_qs, plan, plan_mode);
  if (e != cudaSuccess) return fail(STB_ECUDA, "attn_decode launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

template <int D, int G>
int launch_prefill(const __nv_bfloat16* q, __nv_bfloat16* out, const __nv_bfloat16* kp, const __nv_bfloat16* vp,
                   const int32_t* table, int max_bps, const int32_t* slots, const int32_t* q_start, const int32_t* ctx,
                   int S, int n_kv, float qscale, int max_q, cudaStream_t st) {
  constexpr int QPC = 4 * (16 / G);  // queries per CTA
  size_t smem = (size_t)kPrefillStages * 2 * 16 * D * 2;
  auto kern = attn_prefill_kernel<D, G, kPrefillStages>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((max_q + QPC - 1) / QPC, n_kv, S);
  launch_k(kern, dim3(grid), dim3(128), smem, st, q, out, kp, vp, table, max_bps, slots, q_start, ctx, n_kv, qscale);
  STB_CHECK_LAUNCH("attn_prefill");
  return STB_OK;
}

}  // namespace

extern "C" {

int64_t stb_attn_decode_workspace(int B, int n_q, int n_kv, int d_head) {
  if (B < 0 || n_q <= 0 || n_kv <= 0 || n_q % n_kv || d_head <= 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t floats = decode_part_floats(decode_sms(dev), d_head);
  return (int64_t)(floats * 4 + (size_t)kPlanInts * 4 + (size_t)B * n_kv * 4 + 256);
}

int stb_attn_decode(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                    const int32_t* ctx_lens, int B, int n_q, float scale, int max_ctx, void* work, void* stream) {
  return stb_attn_decode_ex(pool, layer, q, out, slots, ctx_lens, B, n_q, scale, max_ctx, 0, nullptr, work, stream);
}

static int attn_decode_impl(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                            const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                            float scale, int max_ctx, int window, const float* sinks, int plan_mode, void* work,
                            void* stream);

int stb_attn_decode_ex(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                       const int32_t* ctx_lens, int B, int n_q, float scale, int max_ctx, int window,
                       const float* sinks, void* work, void* stream) {
  return attn_decode_impl(pool, layer, q, out, slots, ctx_lens, nullptr, nullptr, B, n_q, scale, max_ctx, window, sinks,
                          0, work, stream);
}

int stb_attn_decode_mq(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                       const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                       float scale, int max_ctx, void* work, void* stream) {
  if (!q_rows || !n_qs) return fail(STB_EINVAL, "attn_decode_mq: q_rows and n_qs are required");
  return attn_decode_impl(pool, layer, q, out, slots, ctx_lens, q_rows, n_qs, B, n_q, scale, max_ctx, 0, nullptr, 0,
                          work, stream);
}

int stb_attn_decode_planned(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                            const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                            float scale, int max_ctx, int plan_mode, void* work, void* stream) {
  if (plan_mode < 0 || plan_mode > 2) return fail(STB_EINVAL, "attn_decode_planned: plan_mode %d", plan_mode);
  if ((q_rows == nullptr) != (n_qs == nullptr))
    return fail(STB_EINVAL, "attn_decode_planned: q_rows and n_qs go together");
  return attn_decode_impl(pool, layer, q, out, slots, ctx_lens, q_rows, n_qs, B, n_q, scale, max_ctx, 0, nullptr,
                          plan_mode, work, stream);
}

static int attn_decode_impl(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                            const int32_t* ctx_lens, const int32_t* q_rows, const int32_t* n_qs, int B, int n_q,
                            float scale, int max_ctx, int window, const float* sinks, int plan_mode, void* work,
                            void* stream) {
  if (window < 0) return fail(STB_EINVAL, "attn_decode: window %d < 0", window);
  void *kp, *vp;
  if (int rc = stb_kv_layer_ptrs(pool, layer, &kp, &vp)) return rc;
  int32_t* table;
  int max_bps;
  stb_kv_block_table(pool, &table, &max_bps);
  if (B <= 0) return STB_OK;
  if (max_ctx > max_bps * 16)
    return fail(STB_EINVAL, "attn_decode: max_ctx %d exceeds the block table (%d rows)", max_ctx, max_bps * 16);
  int n_kv, d_head;
  stb_pool_geometry(pool, &n_kv, &d_head);
  if (n_q % n_kv) return fail(STB_EINVAL, "attn_decode: n_q %% n_kv != 0");
  int g = n_q / n_kv;
  float qs = scale * kLog2e;
  auto* qq = (const __nv_bfloat16*)q;
  auto* oo = (__nv_bfloat16*)out;
  auto* kk = (const __nv_bfloat16*)kp;
  auto* vv = (const __nv_bfloat16*)vp;
  cudaStream_t st = (cudaStream_t)stream;
#define ARGS qq, oo, kk, vv, table, max_bps, slots, ctx_lens, B, n_kv, qs, window, sinks, q_rows, n_qs, plan_mode, work, st
#ifdef STB_MQ_FORCE_QE1
  if (false) {
#else
  if (q_rows != nullptr) {  // multi-query entries: QE = 16 / G queries per 16-row tile
#endif
    if (d_head == 128 && g == 4) return launch_decode<128, 4, 4>(ARGS);
    if (d_head == 128 && g == 8) return launch_decode<128, 8, 2>(ARGS);
    if (d_head == 128 && g == 1) return launch_decode<128, 1, 16>(ARGS);
    if (d_head == 64 && g == 2) return launch_decode<64, 2, 8>(ARGS);
    if (d_head == 64 && g == 8) return launch_decode<64, 8, 2>(ARGS);
    if (d_head == 64 && g == 4) return launch_decode<64, 4, 4>(ARGS);
  } else {
    if (d_head == 128 && g == 4) return launch_decode<128, 4, 1>(ARGS);
    if (d_head == 128 && g == 8) return launch_decode<128, 8, 1>(ARGS);
    if (d_head == 128 && g == 1) return launch_decode<128, 1, 1>(ARGS);
    if (d_head == 64 && g == 2) return launch_decode<64, 2, 1>(ARGS);
    if (d_head == 64 && g == 8) return launch_decode<64, 8, 1>(ARGS);
    if (d_head == 64 && g == 4) return launch_decode<64, 4, 1>(ARGS);
  }
#undef ARGS
  return fail(STB_EINVAL, "attn_decode: unsupported (d_head=%d, group=%d)", d_head, g);
}

int stb_attn_prefill(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                     const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale, int max_q,
                     void* stream) {
  return stb_attn_prefill_split(pool, layer, q, out, slots, q_start, ctx_lens, S, T, n_q, scale, max_q, 0, stream);
}

int stb_attn_prefill_split(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                           const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale,
                           int max_q, int active_units, void* stream) {
  return stb_attn_prefill_ex(pool, layer, q, out, slots, q_start, ctx_lens, S, T, n_q, scale, max_q, active_units, 0,
                             nullptr, stream);
}

int stb_attn_prefill_ex(stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                        const int32_t* q_start, const int32_t* ctx_lens, int S, int T, int n_q, float scale,
                        int max_q, int active_units, int window, const float* sinks, void* stream) {
  if (window < 0) return fail(STB_EINVAL, "attn_prefill: window %d < 0", window);
  void *kp, *vp;
  if (int rc = stb_kv_layer_ptrs(pool, layer, &kp, &vp)) return rc;
  int32_t* table;
  int max_bps;
  stb_kv_block_table(pool, &table, &max_bps);
  if (S <= 0 || T <= 0) return STB_OK;
  // tcgen05/TMEM path unless explicitly pinned to the warp-MMA kernel (A/B checks)
  static int use_mma = -1;
  if (use_mma < 0) {
    const char* e = getenv("STB200_PREFILL");
    use_mma = (e && e[0] == 'm') ? 1 : 0;
  }
  if (!use_mma)
    return stb_attn_prefill_tc(pool, layer, q, out, slots, q_start, ctx_lens, S, T, n_q, scale, max_q, active_units,
                               window, sinks, stream);
  if (window > 0 || sinks != nullptr)
    return fail(STB_EINVAL, "attn_prefill: the mma.sync A/B kernel has no sliding window / sinks (unset STB200_PREFILL)");
  int n_kv, d_head;
  stb_pool_geometry(pool, &n_kv, &d_head);
  if (n_q % n_kv) return fail(STB_EINVAL, "attn_prefill: n_q %% n_kv != 0");
  int g = n_q / n_kv;
  float qs = scale * kLog2e;
  auto* qq = (const __nv_bfloat16*)q;
  auto* oo = (__nv_bfloat16*)out;
  auto* kk = (const __nv_bfloat16*)kp;
  auto* vv = (const __nv_bfloat16*)vp;
  cudaStream_t st = (cudaStream_t)stream;
#define ARGS qq, oo, kk, vv, table, max_bps, slots, q_start, ctx_lens, S, n_kv, qs, max_q, st
  if (d_head == 128 && g == 4) return launch_prefill<128, 4>(ARGS);
  if (d_head == 128 && g == 8) return launch_prefill<128, 8>(ARGS);
  if (d_head == 128 && g == 1) return launch_prefill<128, 1>(ARGS);
  if (d_head == 64 && g == 2) return launch_prefill<64, 2>(ARGS);
  if (d_head == 64 && g == 8) return launch_prefill<64, 8>(ARGS);
  if (d_head == 64 && g == 4) return launch_prefill<64, 4>(ARGS);
#undef ARGS
  return fail(STB_EINVAL, "attn_prefill: unsupported (d_head=%d, group=%d)", d_head, g);
}

}  // extern "C"

#ifdef STB_K3_TRACE
extern "C" int stb_debug_k3_trace(void* buf, int cap) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, g_k3t_n, sizeof(n));
  unsigned long long* p = (unsigned long long*)buf;
  unsigned int c = (unsigned int)cap, z = 0;
  cudaMemcpyToSymbol(g_k3t, &p, sizeof(p));
  cudaMemcpyToSymbol(g_k3t_cap, &c, sizeof(c));
  cudaMemcpyToSymbol(g_k3t_n, &z, sizeof(z));
  return (int)n;
}
#endif
