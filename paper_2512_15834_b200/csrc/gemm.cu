// K5 — bf16 projection / MLP GEMM on the 5th-gen tensor cores.
//
// C[M][N] (fp32) = X[M][K] (bf16 activations) * W[N][K]^T (bf16 weights).
// Replaces, with real FLOPs, every `rate x tokens` charge of the reference engine
// (`engine.py:251,270,296,358`): the QKV / O / gate-up / down / LM-head projections.
//
// Weight-stationary tiling: the 128-row UMMA "M" side is always 128 weight rows
// (output features) and the UMMA "N" side is BN tokens (16..256), so decode steps
// (M = resident batch, e.g. 32) run 128 x 32 UMMAs instead of padding the batch.
//
// Persistent, one CTA per SM, warp-specialised (192 threads):
//   warp 0      TMA producer: W [128 x 64] + X [BN x 64] per stage, 128B swizzle,
//               into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      MMA issuer: one elected thread, tcgen05.mma kind::f16 (fp32 accum
//               in TMEM); tcgen05.commit frees ring slots and publishes finished
//               accumulators; TMEM is double-buffered so the next tile's MMAs run
//               while the epilogue drains the previous one
//   warps 2..5  epilogue: tcgen05.ld of their 32-lane TMEM quarter, fp32 stores
//               (coalesced across the 32 features of a warp; stream-K partial
//               sums as red.global.add — TMA bulk reductions through an smem
//               stage measured no faster)
//
// Two schedules over the (tile, K-block) work space:
//   tiles  tile t -> CTA t mod G, whole K, plain stores (enough tiles to fill
//          the machine: prefill / ingest / LM head)
//   stream the tile-major unit range is cut into G equal contiguous pieces
//          (stream-K); a CTA's piece may end mid-tile, so tiles are reduced with
//          fp32 red.global.add. C is zeroed inside the kernel: after the
//          dependency wait every CTA clears a slice of C and arrives on a
//          self-resetting grid barrier that the epilogue passes before its first
//          reduction (the barrier completes long before the first tile's MMAs,
//          so it costs nothing and there is no separate memset node).
//          Decode-shaped GEMMs (M = 32) are HBM-bound on the weights: this keeps
//          every SM streaming weights for the whole kernel with no tail wave.
//
// Launched with programmatic dependent launch: the producer issues the weight
// loads of the first ring slots *before* griddepcontrol.wait (weights never
// depend on the previous kernel), so pipeline fill overlaps the previous
// kernel's tail; activations are loaded only after the wait.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/stb200.h"
#include "common.cuh"
#include "pool.cuh"
#include "rope.cuh"

using namespace stb;

namespace {

constexpr int BM = 128;  // weight rows per tile (UMMA M)
constexpr int BK = 64;   // K per stage: one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;
constexpr int EPI_CH = 16;        // tokens per fused-epilogue chunk
constexpr int EPI_LD = BM + 4;    // fp32 row stride of the QKV staging tile
constexpr int EPI_SMEM = 256 * 4 * 7 + EPI_CH * EPI_LD * 4;  // sizeof(EpiSmem)
constexpr int kMaxSsParts = 64;   // d_model <= 8192 (ss partials per row, a multiple of 4)

#ifndef STB_GEMM_RING_COUNTERS
#define STB_GEMM_RING_COUNTERS 1
#endif

template <int BN>
struct Cfg {
  static constexpr int W_BYTES = BM * BK * 2;
  static constexpr int X_BYTES = BN * BK * 2;
  static constexpr int STAGE = W_BYTES + X_BYTES;
#ifndef STB_GEMM_DECODE_RING_KB
#define STB_GEMM_DECODE_RING_KB 160
#endif
  // decode-shaped tiles (BN <= 64) use a smaller ring (STB_GEMM_DECODE_RING_KB): 160 KiB (8
  // stages of 20 KiB at BN = 32) measured 0.6-0.8% faster decode steps than 200 KiB (ctx 2k and
  // 4k, two repeats; 100 / 120 / 140 / 180 in between or worse); prefill tiles keep 200 KiB
  static constexpr int RING = (BN <= 64 ? STB_GEMM_DECODE_RING_KB : 200) * 1024;
  static constexpr int STAGES = (RING / STAGE) > 12 ? 12 : (RING / STAGE);
  static constexpr int TMEM_COLS = (2 * BN) < 32 ? 32 : 2 * BN;  // two accumulator buffers
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/ + EPI_SMEM;
};

struct Sched {
  int stream;        // 0: tile schedule, 1: stream-K
  int tiles_n;       // feature tiles (of BM rows)
  int tiles_m;       // token tiles (of bn rows)
  int tiles;         // tiles_n * tiles_m, ordered feature-major: the tiles_m token tiles
                     // that share a weight slice are adjacent, so they run concurrently and
                     // the slice is read from HBM once (L2 serves the others)
  int kb;            // K blocks per tile
  int64_t units;     // tiles * kb
  unsigned* bar;     // stream-K grid barrier {count, generation}, self-resetting
  int c_zeroed;      // stream-K: the caller guarantees C == 0 (no in-kernel zeroing, no barrier)
  int silu;          // tile schedule: fused SiLU-gate epilogue, C is bf16 act[M][N/2]
  int tag;           // launch sequence number (debug trace only)
  int load_debug;    // timing experiments (STB200_GEMM_LOAD_DEBUG): after the first ring fill
                     // 1 = skip X loads, 2 = skip W loads, 3 = skip both (results are garbage)
};

// Fused epilogue (stb_gemm_bf16_fused, include/stb200.h). kind 0 = the plain path above.
struct Epi {
  int kind;                       // 0 none, STB_EPI_SILU, STB_EPI_QKV, STB_EPI_RESID
  const float* ss_in;             // optional per-row RMSNorm statistics of the GEMM input:
  int ss_parts;                   //   ss_in[t][ss_parts] partial sums of squares (RESID: ss_out)
  float inv_dim, eps;
  __nv_bfloat16* out;             // SILU: act; RESID: bf16 copy of x; QKV: q
  int64_t ldo;
  float* x;                       // RESID: fp32 residual stream
  int64_t ldx;
  float* ss_out;                  // RESID: sum of squares of the new x rows (atomic)
  __nv_bfloat16* kpages;          // QKV: this layer's K / V pages (pre-swizzled, pool.cuh)
  __nv_bfloat16* vpages;
  const int32_t* table;
  int max_bps, n_kv, d_head, q_dim, kv_dim;
  const int32_t* slot_of;
  const int32_t* pos_of;
  const float* inv_freq;
  const __nv_bfloat16* q_norm;
  const __nv_bfloat16* k_norm;
  float qk_eps;
  unsigned* cnt;                  // stream-K tile tickets (self-resetting)
};


// Debug timeline (stb_debug_gemm_trace): per CTA {tag, t_last_epilogue, sm, t_entry,
// t_dep_wait, t_first_stage, t_last_mma_issue, t_exit} in %globaltimer ns. Off (null) in
// production; %globaltimer ticks at ~1 us here, so read medians over CTAs, not deltas.
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned int g_trace_n = 0;
__device__ unsigned int g_trace_cap = 0;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Segment iterator: (tile, kb_begin, kb_end) for this CTA, in order.
struct SegIter {
  Sched s;
  int cta, G;
  int u, u_end;  // stream mode cursor (32-bit: the launcher checks units * grid < 2^31)
  int t;         // tile mode cursor
  __device__ SegIter(const Sched& sc) : s(sc), cta(blockIdx.x), G(gridDim.x) {
    if (s.stream) {
      const int U = (int)s.units;
      u = U * cta / G;
      u_end = U * (cta + 1) / G;
    } else {
      t = cta;
    }
  }
  __device__ __forceinline__ bool next(int& tile, int& k0, int& k1) {
    if (s.stream) {
      if (u >= u_end) return false;
      tile = u / s.kb;
      const int base = tile * s.kb;
      k0 = u - base;
      const int e = min(base + s.kb, u_end);
      k1 = e - base;
      u = e;
      return true;
    }
    if (t >= s.tiles) return false;
    tile = t;
    k0 = 0;
    k1 = s.kb;
    t += G;
    return true;
  }
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Number of CTAs whose stream-K unit range [U*c/G, U*(c+1)/G) intersects tile t.
__device__ __forceinline__ int owner_of(int64_t u, int64_t U, int G) {
  int c = (int)((u * G) / U);
  while (c + 1 < G && (U * (c + 1)) / G <= u) ++c;
  return c;
}

// Per-tile token metadata of the fused epilogue, staged once per tile (the chunk loop then
// never waits on a global load): row scale, and for QKV the position and the pool block.
struct EpiSmem {
  float rs[256];
  int pos[256];
  int blk[256];
  float ssw[4][256];           // RESID: per-warp partial sums of squares
  float stage[EPI_CH][EPI_LD];  // QKV: the chunk, feature-major -> token-major
};

__device__ __forceinline__ void epi_tile_prologue(const Epi& ep, EpiSmem& sm, int t0, int ntok) {
  epi_bar();  // every epilogue thread is done with the previous tile's metadata
  const int i = threadIdx.x - 64;
  for (int t = i; t < ntok; t += 128) {
    float r = 1.f;
    if (ep.ss_in != nullptr) {
      // all partial loads issued before the first add (one L2 latency, not ss_parts of them)
      const float4* p = reinterpret_cast<const float4*>(ep.ss_in + (int64_t)(t0 + t) * ep.ss_parts);
      const int n4 = ep.ss_parts >> 2;
      float4 w[kMaxSsParts / 4];
#pragma unroll
      for (int j = 0; j < kMaxSsParts / 4; ++j) w[j] = j < n4 ? __ldcg(p + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < kMaxSsParts / 4; ++j) acc += (w[j].x + w[j].y) + (w[j].z + w[j].w);
      r = rsqrtf(acc * ep.inv_dim + ep.eps);
    }
    sm.rs[t] = r;
    if (ep.kind == STB_EPI_QKV) {
      const int pos = ep.pos_of[t0 + t];
      sm.pos[t] = pos;
      sm.blk[t] = ep.table[(int64_t)ep.slot_of[t0 + t] * ep.max_bps + (pos >> 4)];
    }
  }
  epi_bar();
}

// RESID: the tile's per-token partial sums of squares -> ss_out[t][tile_n] (plain stores:
// every (token, feature tile) slot is written exactly once per GEMM — no atomics)
__device__ __forceinline__ void epi_tile_finish(const Epi& ep, EpiSmem& sm, int t0, int ntok, int tile_n) {
  if (ep.kind != STB_EPI_RESID) return;
  epi_bar();
  const int i = threadIdx.x - 64;
  for (int t = i; t < ntok; t += 128)
    ep.ss_out[(int64_t)(t0 + t) * ep.ss_parts + tile_n] = (sm.ssw[0][t] + sm.ssw[1][t]) + (sm.ssw[2][t] + sm.ssw[3][t]);
}

// The fused epilogue for one chunk of EPI_CH tokens of a finished tile. Thread = weight row
// (feature fl = quarter * 32 + lane of the tile); v[q] = C[t0 + c + q][f0 + fl] (fp32 sum);
// xr[q] = x[t0 + c + q][f] for RESID (loaded a chunk ahead by the caller). All 128 epilogue
// threads call it together (QKV synchronises through smem).
__device__ __forceinline__ void epi_chunk(const Epi& ep, EpiSmem& sm, float* v, const float* xr, int f0, int fl,
                                          int t0, int c, int ntile, int N, int quarter, int lane) {
  const int ntok = min(EPI_CH, ntile - c);  // valid tokens of this chunk (>= 1)
  const int f = f0 + fl;
#pragma unroll
  for (int q = 0; q < EPI_CH; ++q) v[q] *= sm.rs[c + q];  // (rs of invalid tokens: unused)
  if (ep.kind == STB_EPI_SILU) {
    // (gate, up) of output feature f/2 sit in lanes (2i, 2i+1); the even lane emits the
    // first half of the chunk, the odd lane the second half
    const bool odd = lane & 1;
    __nv_bfloat16* __restrict__ out = ep.out;
#pragma unroll
    for (int q = 0; q < EPI_CH / 2; ++q) {
      const float mine = odd ? v[EPI_CH / 2 + q] : v[q];
      const float other = __shfl_xor_sync(0xffffffffu, odd ? v[q] : v[EPI_CH / 2 + q], 1);
      const int tok = odd ? EPI_CH / 2 + q : q;
      if (f < N && tok < ntok)
        out[(int64_t)(t0 + c + tok) * ep.ldo + (f >> 1)] =
            __float2bfloat16_rn(odd ? silu_gate(other, mine) : silu_gate(mine, other));
    }
  } else if (ep.kind == STB_EPI_RESID) {
    float* __restrict__ x = ep.x;
    __nv_bfloat16* __restrict__ out = ep.out;
#pragma unroll
    for (int q = 0; q < EPI_CH; ++q) {
      const float xn = xr[q] + v[q];
      float sq = 0.f;
      if (q < ntok && f < N) {
        const int64_t t = t0 + c + q;
        x[t * ep.ldx + f] = xn;
        out[t * ep.ldo + f] = __float2bfloat16_rn(xn);
        sq = xn * xn;
      }
      sq = warp_sum(sq);
      if (lane == 0) sm.ssw[quarter][c + q] = sq;
    }
  } else {  // STB_EPI_QKV: stage the chunk, then thread = (token, 8 rotation pairs)
#pragma unroll
    for (int q = 0; q < EPI_CH; ++q) sm.stage[q][fl] = v[q];
    epi_bar();
    const int i = threadIdx.x - 64;          // 0..127
    const int tt = i >> 3, sub = i & 7;      // token in chunk, pair group (8 pairs)
    const int d = ep.d_head, hp = d >> 1;    // rotation pairs per head
    const int p0 = sub * 8;                  // first pair (of the tile's 64)
    const int hl = p0 / hp, ip = p0 % hp;    // head in tile, pair index in head
    const int fa = hl * d + ip;              // local feature of the first element
    const int fh = f0 + hl * d;              // global first feature of the head
    float a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = sm.stage[tt][fa + j];
      b[j] = sm.stage[tt][fa + hp + j];
    }
    const int kind = fh < ep.q_dim ? 0 : (fh < ep.q_dim + ep.kv_dim ? 1 : 2);
    const int gpl = hp / 8;                  // lanes sharing one head (8, 4 or 2)
    if (kind < 2 && ep.q_norm != nullptr) {  // Qwen3 qk-norm over the head
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) ss = fmaf(a[j], a[j], fmaf(b[j], b[j], ss));
      for (int o = 1; o < gpl; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float r = rsqrtf(ss / (float)d + ep.qk_eps);
      const __nv_bfloat16* w = kind == 0 ? ep.q_norm : ep.k_norm;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] *= r * __bfloat162float(w[ip + j]);
        b[j] *= r * __bfloat162float(w[ip + hp + j]);
      }
    }
    const bool valid = tt < ntok;
    const int64_t t = t0 + c + tt;
    const int pos = sm.pos[c + tt];
    if (kind < 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float sn, cs;
        sincosf((float)pos * ep.inv_freq[ip + j], &sn, &cs);
        const float x1 = a[j], x2 = b[j];
        a[j] = x1 * cs - x2 * sn;
        b[j] = x2 * cs + x1 * sn;
      }
    }
    const uint4 lo = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
    const uint4 hi = make_uint4(pack_bf16(b[0], b[1]), pack_bf16(b[2], b[3]), pack_bf16(b[4], b[5]), pack_bf16(b[6], b[7]));
    if (valid) {
      if (kind == 0) {
        __nv_bfloat16* dst = ep.out + t * ep.ldo + fh + ip;
        *reinterpret_cast<uint4*>(dst) = lo;
        *reinterpret_cast<uint4*>(dst + hp) = hi;
      } else {
        const int kvh = (fh - ep.q_dim - (kind == 2 ? ep.kv_dim : 0)) / d;
        const int blk = sm.blk[c + tt];
        __nv_bfloat16* row = (kind == 1 ? ep.kpages : ep.vpages) + (((int64_t)blk * ep.n_kv + kvh) * 16 + (pos & 15)) * d;
        *reinterpret_cast<uint4*>(row + kv_phys_chunk(pos & 15, ip >> 3) * 8) = lo;
        *reinterpret_cast<uint4*>(row + kv_phys_chunk(pos & 15, (ip + hp) >> 3) * 8) = hi;
      }
    }
    epi_bar();  // staging reused by the next chunk
  }
}

// RESID: the residual values of chunk c (independent loads, issued a chunk ahead)
__device__ __forceinline__ void load_x(const Epi& ep, float* xr, int t0, int c, int ntile, int f, int N) {
#pragma unroll
  for (int q = 0; q < EPI_CH; ++q)
    xr[q] = (c + q < ntile && f < N) ? __ldcg(ep.x + (int64_t)(t0 + c + q) * ep.ldx + f) : 0.f;
}

// Epilogue warps of a fused-epilogue GEMM: whole tiles straight from TMEM; stream-K partial
// tiles are red.added into the zeroed workspace C, and the CTA that completes a tile
// (ticket) reads it back, runs the epilogue and clears it (C stays zero between calls).
template <int BN>
__device__ __forceinline__ void fused_epilogue(const Epi& ep, const Sched& sched, float* C, int64_t ldc, int M,
                                               int N, int bn, uint32_t tmem, uint64_t* acc_full, uint64_t* acc_empty,
                                               int* s_last, EpiSmem& sm, int quarter, int lane) {
  SegIter it(sched);
  int tile, k0, k1, j = 0;
  const int fl = quarter * 32 + lane;
  const bool resid = ep.kind == STB_EPI_RESID;
  while (it.next(tile, k0, k1)) {
    const int buf = j & 1;
    mbar_wait(&acc_full[buf], (j >> 1) & 1);
    tc_fence_after();
    const int tile_n = tile / sched.tiles_m;
    const int f0 = tile_n * BM;
    const int t0 = (tile % sched.tiles_m) * bn;
    const int f = f0 + fl;
    const int ntile = min(bn, M - t0);  // valid tokens of the tile
    const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN;
    const bool whole = k0 == 0 && k1 == sched.kb;
    if (whole) {
      epi_tile_prologue(ep, sm, t0, ntile);
      float xr[EPI_CH], xn[EPI_CH];
      if (resid) load_x(ep, xr, t0, 0, ntile, f, N);
      for (int c = 0; c < ntile; c += EPI_CH) {
        if (resid) load_x(ep, xn, t0, c + EPI_CH, ntile, f, N);
        uint32_t r[EPI_CH];
        tmem_ld16(base + c, r);
        tmem_ld_wait();
        float v[EPI_CH];
#pragma unroll
        for (int q = 0; q < EPI_CH; ++q) v[q] = __uint_as_float(r[q]);
        epi_chunk(ep, sm, v, xr, f0, fl, t0, c, ntile, N, quarter, lane);
#pragma unroll
        for (int q = 0; q < EPI_CH; ++q) xr[q] = xn[q];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      epi_tile_finish(ep, sm, t0, ntile, tile_n);
    } else {
      for (int c = 0; c < bn; c += EPI_CH) {
        uint32_t r[EPI_CH];
        tmem_ld16(base + c, r);
        tmem_ld_wait();
        if (f < N) {
#pragma unroll
          for (int q = 0; q < EPI_CH; ++q)
            if (c + q < ntile) atomicAdd(C + (int64_t)(t0 + c + q) * ldc + f, __uint_as_float(r[q]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      __threadfence();
      epi_bar();
      if (threadIdx.x == 64) {
        const int64_t kb = sched.kb, G = gridDim.x;
        const int first = owner_of((int64_t)tile * kb, sched.units, (int)G);
        const int last = owner_of((int64_t)(tile + 1) * kb - 1, sched.units, (int)G);
        *s_last = atomicAdd(ep.cnt + tile, 1u) == (unsigned)(last - first);
      }
      epi_bar();
      if (*s_last) {
        __threadfence();
        epi_tile_prologue(ep, sm, t0, ntile);
        auto load_c = [&](float* v, int c) {
#pragma unroll
          for (int q = 0; q < EPI_CH; ++q)
            v[q] = (f < N && c + q < ntile) ? __ldcg(C + (int64_t)(t0 + c + q) * ldc + f) : 0.f;
        };
        float v[EPI_CH], vn[EPI_CH], xr[EPI_CH], xn[EPI_CH];
        load_c(v, 0);
        if (resid) load_x(ep, xr, t0, 0, ntile, f, N);
        for (int c = 0; c < ntile; c += EPI_CH) {
          load_c(vn, c + EPI_CH);
          if (resid) load_x(ep, xn, t0, c + EPI_CH, ntile, f, N);
#pragma unroll
          for (int q = 0; q < EPI_CH; ++q)  // leave the workspace zeroed
            if (f < N && c + q < ntile) __stcg(C + (int64_t)(t0 + c + q) * ldc + f, 0.f);
          epi_chunk(ep, sm, v, xr, f0, fl, t0, c, ntile, N, quarter, lane);
#pragma unroll
          for (int q = 0; q < EPI_CH; ++q) v[q] = vn[q], xr[q] = xn[q];
        }
        epi_tile_finish(ep, sm, t0, ntile, tile_n);
        if (threadIdx.x == 64) ep.cnt[tile] = 0u;
      }
    }
    ++j;
  }
}

// FUSED selects the fused-epilogue instantiation (stb_gemm_bf16_fused): the plain kernel carries
// none of that code, so its instruction footprint (fetched cold at every launch) stays small.
template <int BN, bool FUSED>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_persistent(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                         float* __restrict__ C, int64_t ldc, int M, int N, Sched sched, int bn,
                         const __nv_bfloat16* __restrict__ w_tiled, const Epi ep) {
  // w_tiled != nullptr: W in the stb_weight_tile layout, one 16 KiB bulk copy per stage
  // bn: token-tile height actually used (<= BN, multiple of 16); BN sizes the smem ring
  using CF = Cfg<BN>;
  constexpr int STAGES = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  EpiSmem& esm = *reinterpret_cast<EpiSmem*>(smem + STAGES * CF::STAGE + 256);
  __shared__ unsigned long long tt[6];
  const bool tracing = g_trace != nullptr;
  if (tracing && threadIdx.x == 0) tt[0] = gtime();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    if (w_tiled == nullptr) tma_prefetch(&tm_w);
    tma_prefetch(&tm_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      auto load_w = [&](uint8_t* dst, int k, int f0, uint64_t* bar) {
        if (w_tiled != nullptr)
          bulk_load(smem_u32(dst), w_tiled + ((int64_t)(f0 / BM) * sched.kb + k) * (BM * BK), CF::W_BYTES, bar);
        else
          tma_load_2d(dst, &tm_w, bar, k * BK, f0);
      };
      // weights first: the ring's first slots fill before the dependency wait
#ifndef STB_GEMM_PREFETCH_STAGES
#define STB_GEMM_PREFETCH_STAGES 64  // (capped at the ring depth) A/B knob: weight stages issued before the wait
#endif
      constexpr int PRE = STB_GEMM_PREFETCH_STAGES < STAGES ? STB_GEMM_PREFETCH_STAGES : STAGES;
      SegIter pre(sched);
      int tile, k0, k1, i = 0;
      while (i < PRE && pre.next(tile, k0, k1)) {
        const int f0 = (tile / sched.tiles_m) * BM;
        for (int k = k0; k < k1 && i < PRE; ++k, ++i) {
          mbar_expect_tx(&full[i], CF::W_BYTES + bn * BK * 2);
          load_w(smem + i * CF::STAGE, k, f0, &full[i]);
        }
      }
      const int prefetched = i;
      if (tracing) tt[5] = gtime();
      pdl_wait();
      if (tracing) tt[1] = gtime();
      pdl_launch();
      SegIter it(sched);
      i = 0;
      while (it.next(tile, k0, k1)) {
        const int f0 = (tile / sched.tiles_m) * BM;
        const int t0 = (tile % sched.tiles_m) * bn;
        for (int k = k0; k < k1; ++k, ++i) {
          const int s = i % STAGES;
          uint8_t* sw = smem + s * CF::STAGE;
          if (i < prefetched) {
            tma_load_2d(sw + CF::W_BYTES, &tm_x, &full[s], k * BK, t0);
            continue;
          }
          mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
          if (sched.load_debug && i >= STAGES) {
            const bool lw = !(sched.load_debug & 2), lx = !(sched.load_debug & 1);
            const uint32_t b = (lw ? CF::W_BYTES : 0) + (lx ? bn * BK * 2 : 0);
            if (b) {
              mbar_expect_tx(&full[s], b);
              if (lw) load_w(sw, k, f0, &full[s]);
              if (lx) tma_load_2d(sw + CF::W_BYTES, &tm_x, &full[s], k * BK, t0);
            } else {
              mbar_arrive(&full[s]);
            }
            continue;
          }
          mbar_expect_tx(&full[s], CF::W_BYTES + bn * BK * 2);
          load_w(sw, k, f0, &full[s]);
          tma_load_2d(sw + CF::W_BYTES, &tm_x, &full[s], k * BK, t0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = umma_idesc_bf16(BM, bn, false, false);
      SegIter it(sched);
      int tile, k0, k1, i = 0, j = 0, rs = 0, rph = 0;
      const uint64_t wdesc0 = umma_desc_kmajor_sw128(smem_u32(smem), 1024);
      (void)rs, (void)rph, (void)wdesc0;
      while (it.next(tile, k0, k1)) {
        const int buf = j & 1;
        mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        for (int k = k0; k < k1; ++k, ++i) {
#if STB_GEMM_RING_COUNTERS
          const int s = rs;
          mbar_wait(&full[s], rph);
          if (++rs == STAGES) rs = 0, rph ^= 1;
          if (tracing && i == 0) tt[2] = gtime();
          const uint64_t adesc = wdesc0 + (uint64_t)((s * CF::STAGE) >> 4);
          const uint64_t bdesc = adesc + (CF::W_BYTES >> 4);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_f16_ss(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (k > k0 || kk > 0) ? 1u : 0u);
#else
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          if (tracing && i == 0) tt[2] = gtime();
          tc_fence_after();
          const uint32_t wa = smem_u32(smem + s * CF::STAGE);
          const uint32_t xa = wa + CF::W_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            umma_f16_ss(d, umma_desc_kmajor_sw128(wa + kk * 32, 1024), umma_desc_kmajor_sw128(xa + kk * 32, 1024),
                        idesc, (k > k0 || kk > 0) ? 1u : 0u);
          }
#endif
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
        ++j;
      }
      if (tracing) tt[3] = gtime();
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5 -> TMEM lane quarters 2,3,0,1
    pdl_wait();
    const int quarter = warp & 3;
    if constexpr (FUSED) {
      fused_epilogue<BN>(ep, sched, C, ldc, M, N, bn, tmem, acc_full, acc_empty, s_last, esm, quarter, lane);
    } else {
    const bool atomic = sched.stream != 0;
    const bool zero_here = atomic && !sched.c_zeroed;
    unsigned gen = 0;
    if (zero_here) {
      // clear this CTA's slice of C (rows split across CTAs, float4 when the row is aligned),
      // then arrive on the grid barrier
      const int G = gridDim.x;
      if (threadIdx.x == 64) gen = *(volatile unsigned*)(sched.bar + 1);
      const int et = threadIdx.x - 64;
      const bool vec = (N % 4 == 0) && (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
      const int per_row = vec ? N / 4 : N;
      const int total = M * per_row;
      const int lo = (int)((int64_t)total * blockIdx.x / G), hi = (int)((int64_t)total * (blockIdx.x + 1) / G);
      for (int e = lo + et; e < hi; e += 128) {
        const int r = e / per_row, cidx = e - r * per_row;
        if (vec)
          reinterpret_cast<float4*>(C + (int64_t)r * ldc)[cidx] = make_float4(0.f, 0.f, 0.f, 0.f);
        else
          C[(int64_t)r * ldc + cidx] = 0.f;
      }
      __threadfence();
      epi_bar();
      if (threadIdx.x == 64) {
        if (atomicAdd(sched.bar, 1u) == (unsigned)G - 1) {
          *(volatile unsigned*)sched.bar = 0u;
          __threadfence();
          atomicAdd(sched.bar + 1, 1u);
        }
      }
    }
    bool passed = !zero_here;
    SegIter it(sched);
    int tile, k0, k1, j = 0;
    while (it.next(tile, k0, k1)) {
      const int buf = j & 1;
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      if (tracing && threadIdx.x == 64) tt[4] = gtime();
      tc_fence_after();
      if (!passed) {  // every slice of C is zero before the first reduction lands
        if (threadIdx.x == 64)
          while (*(volatile unsigned*)(sched.bar + 1) == gen) __nanosleep(64);
        epi_bar();
        __threadfence();
        passed = true;
      }
      const int slab = (tile / sched.tiles_m) * BM + quarter * 32;  // this warp's 32 features
      const int feat = slab + lane;
      const int t0 = (tile % sched.tiles_m) * bn;
      const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN;
      // 32 tokens per TMEM load (one wait per 32), a 16-token load for the remainder; the
      // warp-collective loads run on every lane, stores only for features < N; full
      // in-range chunks store without per-token predicates
      const int ntok = min(bn, M - t0);
      const bool fok = feat < N;
      float* crow = C + (int64_t)t0 * ldc + feat;
      auto put = [&](int q, uint32_t v) {
        float* dst = crow + (int64_t)q * ldc;
        if (atomic) atomicAdd(dst, __uint_as_float(v));
        else *dst = __uint_as_float(v);
      };
      if (sched.silu) {
        // (gate, up) of output feature feat/2 sit in lanes (2i, 2i+1): one xor-shuffle
        // per token pair; the even lane emits the first half of each chunk, the odd lane
        // the second half
        __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)t0 * ldc + (feat >> 1);
        const bool odd = lane & 1;
        auto emit = [&](int tok, float g, float u) {
          if (fok && tok < ntok) act[(int64_t)tok * ldc] = __float2bfloat16_rn(silu_gate(g, u));
        };
        int c = 0;
#pragma unroll 1
        for (; c + 32 <= bn; c += 32) {
          uint32_t r[32];
          tmem_ld32(base + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float mine = __uint_as_float(odd ? r[16 + q] : r[q]);
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? r[q] : r[16 + q]), 1);
            if (odd) emit(c + 16 + q, other, mine);
            else emit(c + q, mine, other);
          }
        }
        if (c < bn) {
          uint32_t r[16];
          tmem_ld16(base + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float mine = __uint_as_float(odd ? r[8 + q] : r[q]);
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? r[q] : r[8 + q]), 1);
            if (odd) emit(c + 8 + q, other, mine);
            else emit(c + q, mine, other);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        ++j;
        continue;
      }
      int c = 0;
#pragma unroll 1
      for (; c + 32 <= bn; c += 32) {
        uint32_t r[32];
        tmem_ld32(base + c, r);
        tmem_ld_wait();
        if (fok) {
          if (c + 32 <= ntok) {
#pragma unroll
            for (int q = 0; q < 32; ++q) put(c + q, r[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (c + q < ntok) put(c + q, r[q]);
          }
        }
      }
      if (c < bn) {  // bn is a multiple of 16
        uint32_t r[16];
        tmem_ld16(base + c, r);
        tmem_ld_wait();
        if (fok) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c + q < ntok) put(c + q, r[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      ++j;
    }
    if (!passed && threadIdx.x == 64)  // no segment: still let the barrier complete before exiting
      while (*(volatile unsigned*)(sched.bar + 1) == gen) __nanosleep(64);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free(tmem, CF::TMEM_COLS);
  if (tracing && threadIdx.x == 64) {
    const unsigned slot = atomicAdd(&g_trace_n, 1u);
    if (slot < g_trace_cap) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      unsigned long long* r = g_trace + (size_t)slot * 8;
      r[0] = (unsigned long long)sched.tag;
      r[1] = tt[4];
      r[2] = tt[5];  // producer: ring pre-filled, about to wait on the previous grid
      (void)sm;
      r[3] = tt[0];
      r[4] = tt[1];
      r[5] = tt[2];
      r[6] = tt[3];
      r[7] = gtime();
    }
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

// 2-D bf16 row-major [rows][cols] (row stride ld elements), box [box_rows][64], 128B swizzle
int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return STB_OK;
}

struct MapKey {
  const void* p;
  int64_t rows, cols, ld;
  int box;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box;
  }
};
struct MapHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (k.rows * 1315423911u) ^ (k.cols << 7) ^ (k.ld << 17) ^ k.box;
  }
};

int cached_map(CUtensorMap* out, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapHash> cache;
  MapKey key{base, rows, cols, ld, box_rows};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STB_OK;
  }
  if (int rc = make_map(out, base, rows, cols, ld, box_rows)) return rc;
  if (cache.size() > 8192) cache.clear();
  cache.emplace(key, *out);
  return STB_OK;
}

// [rows][64] bf16 with 128-byte rows, box [128][64], no swizzle: one pre-swizzled weight tile
int cached_map_raw(CUtensorMap* out, const void* base, int64_t rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapHash> cache;
  MapKey key{base, rows, -1, 64, BM};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return STB_OK;
  }
  auto fn = encode_fn();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)BK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(BK * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "cuTensorMapEncodeTiled (tiled weights) failed (%d)", (int)r);
  if (cache.size() > 8192) cache.clear();
  cache.emplace(key, *out);
  return STB_OK;
}

int sm_count() { return device_sms(); }

// stream-K grid barrier state {arrivals, generation}: per (device, stream), zeroed once,
// self-resetting. Two stream-K GEMMs in flight on different streams never share a barrier.
unsigned* grid_barrier(cudaStream_t st) {
  return (unsigned*)stream_scratch(kScratchGridBar, st, 2 * sizeof(unsigned));
}

// stream-K tile tickets of the fused-epilogue path: per (device, stream), zeroed once, reset
// by each tile's finisher
constexpr int kMaxTickets = 1 << 14;
unsigned* tile_tickets(cudaStream_t st) {
  return (unsigned*)stream_scratch(kScratchTileTickets, st, kMaxTickets * sizeof(unsigned));
}

int bn_template(int M) { return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256; }

// Token-tile height and schedule for an M x N product.
//  M <= 128 (decode: HBM-bound on the weights): one token tile; tile schedule only when
//    the tiles fill the machine several times over, stream-K otherwise so every SM
//    streams weights for the whole kernel.
//  M > 128 (prefill / ingest: tensor-bound): pick the number of token tiles that
//    minimises waves x (bn + fixed per-tile cost) — wave quantisation dominates at a few
//    hundred tokens — and use whole tiles unless they would leave most SMs idle.
struct Plan {
  int bn, tiles_m, stream;
};
Plan plan(int M, int N, int sms) {
  const int BN = bn_template(M);
  const int tiles_n = (N + BM - 1) / BM;
  Plan p{BN, 1, 0};
  if (M <= 128) {
    p.stream = tiles_n >= 4 * sms ? 0 : 1;
    return p;
  }
#ifndef STB_GEMM_TILE_COST
#define STB_GEMM_TILE_COST 48
#endif
  constexpr int kTileCost = STB_GEMM_TILE_COST;  // per-tile fill/epilogue + smaller-tile inefficiency, in token columns
  long best = -1;
  for (int nt = (M + 255) / 256; nt <= (M + 63) / 64; ++nt) {
    const int bn = (((M + nt - 1) / nt + 15) / 16) * 16;
    if (bn > 256) continue;
    const int tm = (M + bn - 1) / bn;
    const long tiles = (long)tiles_n * tm;
    const long cost = ((tiles + sms - 1) / sms) * (long)(bn + kTileCost);
    if (best < 0 || cost < best) {
      best = cost;
      p.bn = bn;
      p.tiles_m = tm;
    }
  }
  const long tiles = (long)tiles_n * p.tiles_m;
  const long waves = (tiles + sms - 1) / sms;
  p.stream = 2 * tiles < waves * sms ? 1 : 0;  // whole tiles would leave most SMs idle
  return p;
}


// ============================================================================================
// K5 decode block (stb_gemm_block): a chain of decode-shaped GEMMs and the row ops between
// them in ONE persistent launch. A decode layer used to be nine dependent launches (QKV,
// RoPE+commit, attention, O, add+norm, gate-up, SiLU, down, add+norm): every boundary costs
// a CTA turnover, a prologue and an HBM first-byte latency, and the row ops sit on the
// critical path between weight streams. Here the chain between two attention launches —
// [O, norm, gate-up, SiLU, down, norm, QKV(next layer), RoPE+commit] — is one grid of one
// CTA per SM:
//   warp 0     producer: walks every GEMM's stream-K (tile, K-block) stages in order and
//              issues each stage's weight tile as soon as its ring slot is free — weights
//              never depend on the previous phase — and its activation tile once the phase
//              that produces those activations has completed grid-wide (a generation
//              counter it polls), so the ring is full of the next GEMM's weights while the
//              previous phase's reductions and row op finish
//   warp 1     MMA issuer (one thread), as gemm_bf16_persistent, across all GEMM phases
//   warps 2-5  epilogue: per GEMM phase, TMEM -> fp32 red.add into that phase's zeroed
//              accumulator; per row-op phase, the op on this CTA's slice of rows /
//              elements (the same arithmetic as stb_add_rmsnorm / stb_silu_mul /
//              rope_commit_elem); a grid barrier (arrive + generation) after every phase
// Co-residency: grid = SM count at one CTA per SM (the stream-K GEMMs already rely on it).
// ============================================================================================
constexpr int kBlkMaxGemm = 4;
constexpr int kBlkMaxGlue = 5;
constexpr int kBlkMaxOps = kBlkMaxGemm + kBlkMaxGlue;

struct alignas(64) BlkGemm {
  CUtensorMap tx;           // activations [M][K] bf16, box [bn][64], 128B swizzle
  const __nv_bfloat16* w;   // stb_weight_tile layout
  float* c;                 // fp32 accumulator, zero on entry
  int64_t ldc;
  int N;
  Sched s;                  // stream-K over the grid, one token tile
};

struct BlkGlue {
  int kind;                 // STB_OP_NORM / SILU / ROPE
  float* c;                 // NORM delta, SILU gate/up, ROPE qkv (all cleared)
  float* x;                 // NORM residual stream
  const __nv_bfloat16* w;   // NORM weight
  __nv_bfloat16* y;         // bf16 output (NORM: may be null -> residual add only)
  int n;                    // NORM d, SILU d_ff
  float eps;
  __nv_bfloat16* kpages;    // ROPE
  __nv_bfloat16* vpages;
  const int32_t* table;
  int max_bps, n_q, n_kv, d_head;
  const int32_t* slot_of;
  const int32_t* pos_of;
  const float* inv_freq;
  const __nv_bfloat16* q_norm;
  const __nv_bfloat16* k_norm;
};

struct BlkArgs {
  BlkGemm g[kBlkMaxGemm];
  BlkGlue u[kBlkMaxGlue];
  int n_ops, n_gemm, M, bn;
  int8_t kind[kBlkMaxOps];  // 0: GEMM, else the row op's STB_OP_* kind
  int8_t idx[kBlkMaxOps];   // index into g / u
  int8_t gneed[kBlkMaxGemm];  // GEMM j: barrier completions before its activations exist
  unsigned* bar;            // {arrivals, generation}: self-resetting grid barrier
  int tag;                  // launch sequence number (debug trace only)
};

// Debug timeline of decode-block launches (stb_debug_block_trace): per CTA 32 x u64 =
// {tag, cta, t_entry, t_dep_wait, then per op k: t_start (wait passed), t_done, t_arrived, ..., t_exit}
__device__ unsigned long long* g_btrace = nullptr;
__device__ unsigned int g_btrace_n = 0;
__device__ unsigned int g_btrace_cap = 0;

// grid barrier layout: the arrival counter and the generation word sit 4 KiB apart (different
// L2 lines and slices), so the pollers of the generation never queue behind the arrivals
constexpr int kGenOff = 1024;

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
// wait until k barrier completions past g0 have been published (one poller per CTA)
__device__ __forceinline__ void blk_wait_gen(const unsigned* bar, unsigned g0, int k) {
  if ((int)(ld_relaxed_gpu(bar + kGenOff) - g0) < k) {
    do {
      __nanosleep(100);
    } while ((int)(ld_relaxed_gpu(bar + kGenOff) - g0) < k);
  }
  fence_acq_rel_gpu();
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// every stream-K stage (GEMM j, tile, K block) of the chain, in issue order
struct BlkCursor {
  const BlkArgs* a;
  int j;
  SegIter it;
  int tile, k, k1;
  __device__ explicit BlkCursor(const BlkArgs& args) : a(&args), j(0), it(args.g[0].s), tile(0), k(0), k1(0) { seek(); }
  __device__ __forceinline__ void seek() {
    while (j < a->n_gemm) {
      if (it.next(tile, k, k1)) return;
      if (++j < a->n_gemm) it = SegIter(a->g[j].s);
    }
  }
  __device__ __forceinline__ bool done() const { return j >= a->n_gemm; }
  __device__ __forceinline__ void advance() {
    if (++k >= k1) seek();
  }
};

// NORM: row r of M on CTA r mod G; the 128 epilogue threads hold the row (float4 each per
// 512 columns, d <= 8192): x += delta (delta cleared), y = bf16(x * rsqrt(mean x^2 + eps) * w)
__device__ __forceinline__ void blk_norm(const BlkGlue& u, int M, float* red) {
  const int et = threadIdx.x - 64, we = et >> 5, lane = threadIdx.x & 31;
  const int d4 = u.n >> 2;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    float4* __restrict__ xr = reinterpret_cast<float4*>(u.x + (int64_t)r * u.n);
    float4* __restrict__ cr = u.c ? reinterpret_cast<float4*>(u.c + (int64_t)r * u.n) : nullptr;
    float4 v[16], e[16];
    // every load of the row first (one L2 latency, not one per float4), then the stores
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c4 = et + i * 128;
      v[i] = c4 < d4 ? __ldcg(xr + c4) : z;
      e[i] = (cr && c4 < d4) ? __ldcg(cr + c4) : z;
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c4 = et + i * 128;
      if (c4 >= d4) continue;
      if (cr) {
        v[i].x += e[i].x, v[i].y += e[i].y, v[i].z += e[i].z, v[i].w += e[i].w;
        __stcg(cr + c4, z);
        __stcg(xr + c4, v[i]);
      }
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
    ss = warp_sum(ss);
    if (lane == 0) red[we] = ss;
    epi_bar();
    const float tot = (red[0] + red[1]) + (red[2] + red[3]);
    epi_bar();  // red is reused by the next row
    if (u.y == nullptr) continue;
    const float inv = rsqrtf(tot / u.n + u.eps);
    __nv_bfloat16* yr = u.y + (int64_t)r * u.n;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c4 = et + i * 128;
      if (c4 >= d4) continue;
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(u.w + 4 * c4));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(u.w + 4 * c4 + 2));
      *reinterpret_cast<uint2*>(yr + 4 * c4) = make_uint2(pack_bf16(v[i].x * inv * w01.x, v[i].y * inv * w01.y),
                                                          pack_bf16(v[i].z * inv * w23.x, v[i].w * inv * w23.y));
    }
  }
}

// SILU: y[t][i] = silu(gu[t][2i]) * gu[t][2i+1] over every CTA's epilogue threads; gu cleared.
// Each thread's items are loaded in batches of 8 before any store (one L2 latency per batch).
__device__ __forceinline__ void blk_silu(const BlkGlue& u, int M) {
  const int et = threadIdx.x - 64;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t total4 = (int64_t)M * u.n / 4, step = (int64_t)gridDim.x * 128;
  constexpr int kBatch = 8;
  for (int64_t b0 = (int64_t)blockIdx.x * 128 + et; b0 < total4; b0 += kBatch * step) {
    float4 a[kBatch], b[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int64_t i4 = b0 + j * step;
      a[j] = b[j] = z;
      if (i4 < total4) {
        const int64_t i = i4 * 4, t = i / u.n, c = i - t * u.n;
        const float4* p = reinterpret_cast<const float4*>(u.c + t * 2 * u.n + 2 * c);
        a[j] = __ldcg(p);      // g0 u0 g1 u1
        b[j] = __ldcg(p + 1);  // g2 u2 g3 u3
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int64_t i4 = b0 + j * step;
      if (i4 >= total4) break;
      const int64_t i = i4 * 4, t = i / u.n, c = i - t * u.n;
      float4* p = reinterpret_cast<float4*>(u.c + t * 2 * u.n + 2 * c);
      __stcg(p, z);
      __stcg(p + 1, z);
      *reinterpret_cast<uint2*>(u.y + i) =
          make_uint2(pack_bf16(silu_gate(a[j].x, a[j].y), silu_gate(a[j].z, a[j].w)),
                     pack_bf16(silu_gate(b[j].x, b[j].y), silu_gate(b[j].z, b[j].w)));
    }
  }
}

// ROPE: rope_commit_elem over (token, head, rotation group) elements, a warp-aligned range
// per epilogue warp (the qk-norm shuffles need whole warps)
__device__ __forceinline__ void blk_rope(const BlkGlue& u, int M) {
  const int we = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
  const int64_t total = (int64_t)M * (u.n_q + 2 * u.n_kv) * (u.d_head / 16);
  for (int64_t base = ((int64_t)blockIdx.x * 4 + we) * 32; base < total; base += (int64_t)gridDim.x * 128)
    rope_commit_elem(base + lane, u.c, u.y, u.slot_of, u.pos_of, M, u.n_q, u.n_kv, u.d_head, u.inv_freq, u.table,
                     u.max_bps, u.kpages, u.vpages, M, u.q_norm, u.k_norm, u.eps, nullptr, 1.f);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_block_kernel(const __grid_constant__ BlkArgs a) {
  using CF = Cfg<BN>;
  constexpr int STAGES = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  __shared__ unsigned s_g0;
  __shared__ volatile int s_g0_set;
  __shared__ volatile int s_done;  // barrier completions the epilogue's poller has observed
  __shared__ float s_red[4];
  __shared__ unsigned long long bt[32];
  const bool btracing = g_btrace != nullptr;
  if (btracing && threadIdx.x == 0) bt[2] = gtime();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bn = a.bn, M = a.M;
  if (warp == 0 && lane == 0) {
    for (int j = 0; j < a.n_gemm; ++j) tma_prefetch(&a.g[j].tx);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
    s_g0_set = 0;
    s_done = 0;
  }
  if (warp == 1) tmem_alloc(tmem_slot, CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kStageTx = (uint32_t)CF::W_BYTES;

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t tx_bytes = kStageTx + (uint32_t)bn * BK * 2;
      BlkCursor cw(a), cx(a);
      int nw = 0, nx = 0;
      auto issue_w = [&]() {
        const int s = nw % STAGES;
        mbar_wait(&empty[s], ((nw / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], tx_bytes);
        const BlkGemm& g = a.g[cw.j];
        bulk_load(smem_u32(smem + s * CF::STAGE), g.w + ((int64_t)cw.tile * g.s.kb + cw.k) * (BM * BK), CF::W_BYTES,
                  &full[s]);
        cw.advance();
        ++nw;
      };
      // weights of the first ring slots before the dependency wait
      while (!cw.done() && nw < STAGES) issue_w();
      pdl_wait();
      const unsigned g0 = ld_acquire_gpu(a.bar + kGenOff);  // stable: the previous launch has completed
      if (btracing) bt[3] = gtime();
      s_g0 = g0;
      __threadfence_block();
      s_g0_set = 1;
      pdl_launch();
      int ready_j = -1;  // highest GEMM whose activations are known to exist
      while (!cx.done()) {
        if (nx < nw) {
          if (cx.j > ready_j) {
            // completions observed by this CTA's epilogue poller (no second global poller)
            const int need = a.gneed[cx.j];
            if (need == 0 || s_done >= need) {
              fence_acq_rel_gpu();
              fence_proxy_async_global();  // row-op outputs (generic stores) -> TMA reads
              ready_j = cx.j;
            }
          }
          if (cx.j <= ready_j) {
            const int s = nx % STAGES;
            tma_load_2d(smem + s * CF::STAGE + CF::W_BYTES, &a.g[cx.j].tx, &full[s], cx.k * BK, 0);
            cx.advance();
            ++nx;
            continue;
          }
        }
        if (!cw.done() && nw - nx < STAGES) {
          issue_w();
          continue;
        }
        __nanosleep(32);  // the next phase's activations are still being produced
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = umma_idesc_bf16(BM, bn, false, false);
      int i = 0, jj = 0;
      for (int j = 0; j < a.n_gemm; ++j) {
        SegIter it(a.g[j].s);
        int tile, k0, k1;
        while (it.next(tile, k0, k1)) {
          const int buf = jj & 1;
          mbar_wait(&acc_empty[buf], ((jj >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * BN;
          for (int k = k0; k < k1; ++k, ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            tc_fence_after();
            const uint32_t wa = smem_u32(smem + s * CF::STAGE);
            const uint32_t xa = wa + CF::W_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_f16_ss(d, umma_desc_kmajor_sw128(wa + kk * 32, 1024), umma_desc_kmajor_sw128(xa + kk * 32, 1024),
                          idesc, (k > k0 || kk > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          umma_commit(&acc_full[buf]);
          ++jj;
        }
      }
    }
    __syncwarp();
  } else {
    pdl_wait();
    if (threadIdx.x == 64)
      while (!s_g0_set) __nanosleep(32);
    epi_bar();
    const unsigned g0 = s_g0;
    const int quarter = warp & 3, G = gridDim.x;
    int jj = 0;
    for (int op = 0; op < a.n_ops; ++op) {
      const int kind = a.kind[op];
      // every phase before this one has completed grid-wide (op barriers so far). Waited for
      // by every CTA — also before a GEMM phase in which it owns no stream-K segment — so no
      // CTA arrives at barrier op+1 while barrier op is still counting arrivals
      if (threadIdx.x == 64 && op > 0) {
        blk_wait_gen(a.bar, g0, op);
        s_done = op;
      }
      if (btracing && threadIdx.x == 64) bt[4 + 3 * op] = gtime();
      if (kind == 0) {
        const BlkGemm& g = a.g[a.idx[op]];
        SegIter it(g.s);
        int tile, k0, k1;
        while (it.next(tile, k0, k1)) {
          const int buf = jj & 1;
          mbar_wait(&acc_full[buf], (jj >> 1) & 1);
          tc_fence_after();
          const int feat = tile * BM + quarter * 32 + lane;
          const bool fok = feat < g.N;
          float* crow = g.c + feat;
          const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN;
          int c = 0;
#pragma unroll 1
          for (; c + 32 <= bn; c += 32) {
            uint32_t r[32];
            tmem_ld32(base + c, r);
            tmem_ld_wait();
            if (fok) {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (c + q < M) atomicAdd(crow + (int64_t)(c + q) * g.ldc, __uint_as_float(r[q]));
            }
          }
          if (c < bn) {
            uint32_t r[16];
            tmem_ld16(base + c, r);
            tmem_ld_wait();
            if (fok) {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (c + q < M) atomicAdd(crow + (int64_t)(c + q) * g.ldc, __uint_as_float(r[q]));
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
          ++jj;
        }
      } else {
        epi_bar();
        const BlkGlue& u = a.u[a.idx[op]];
        if (kind == STB_OP_NORM) blk_norm(u, M, s_red);
        else if (kind == STB_OP_SILU) blk_silu(u, M);
        else blk_rope(u, M);
      }
      if (btracing && threadIdx.x == 64) bt[5 + 3 * op] = gtime();
      if (op + 1 < a.n_ops) {  // grid barrier: this phase's results are visible everywhere
        __threadfence();
        if (kind != 0) fence_proxy_async_global();
        epi_bar();
        if (threadIdx.x == 64) {
          __threadfence();
          if (atomicAdd(a.bar, 1u) == (unsigned)G - 1) {
            *(volatile unsigned*)a.bar = 0u;
            __threadfence();
            atomicAdd(a.bar + kGenOff, 1u);
          }
          if (btracing) bt[6 + 3 * op] = gtime();
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free(tmem, CF::TMEM_COLS);
  if (btracing && threadIdx.x == 64) {
    const unsigned slot = atomicAdd(&g_btrace_n, 1u);
    if (slot < g_btrace_cap) {
      bt[0] = ((unsigned long long)a.tag << 8) | (unsigned long long)a.n_ops;
      bt[1] = blockIdx.x;
      bt[31] = gtime();
      for (int i = 0; i < 32; ++i) g_btrace[(size_t)slot * 32 + i] = bt[i];
    }
  }
}

template <int BN>
int launch_block(const BlkArgs& a, int grid, cudaStream_t st) {
  auto kern = gemm_block_kernel<BN>;
  smem_attr_once(kern, Cfg<BN>::SMEM);
  cudaError_t e = launch_k(kern, dim3(grid), dim3(kThreads), Cfg<BN>::SMEM, st, a);
  if (e != cudaSuccess) return fail(STB_ECUDA, "gemm_block launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

// ============================================================================================
// K5 pair kernel: prefill-shaped GEMMs (whole tiles) on CTA pairs, tcgen05.mma.cta_group::2.
// A pair computes a 256-feature x bn-token tile: each CTA stages its own 128 weight rows and
// half of the bn token rows per pipeline stage; the leader issues UMMA M=256 x N=bn, which
// reads A from each CTA's smem and B from both halves, and accumulates each CTA's 128 rows in
// that CTA's TMEM. Per SM this halves the activation bytes staged per flop (the B operand is
// shared) and doubles the MMA work per issued instruction.
//   warp 0     producer (both CTAs): weight rows + token-row half per stage
//   warp 1     leader: MMA issuer (peer: idle)
//   warps 2-5  epilogue (both CTAs): this CTA's 128 rows from TMEM, plain stores / SiLU-gate
// Barriers: full[s] in the leader counts both CTAs' TMA bytes (cta_group::2 loads complete on
// the leader's barrier; the leader arms it for the pair), empty[s] and acc_full[b] in both CTAs
// (multicast tcgen05.commit), acc_empty[b] in the leader (4 local + 4 remote epilogue arrivals).
// An earlier version forwarded the peer's stage completion with a release-scoped remote arrive:
// that compiles to a GPU-wide membar per stage and ran at half the 1-CTA kernel's speed.
// ============================================================================================
constexpr int PAIR_BM = 2 * BM;  // features per pair tile

template <int BN>
struct PairCfg {
  static constexpr int W_BYTES = BM * BK * 2;
  static constexpr int X_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the token rows
  static constexpr int STAGE = W_BYTES + X_BYTES;
#ifndef STB_GEMM_PAIR_RING_KB
#define STB_GEMM_PAIR_RING_KB 224  // 7 stages of 32 KiB: down-proj (K = 14336) 4-5% faster than 6
#endif
  static constexpr int RING = STB_GEMM_PAIR_RING_KB * 1024;
  static constexpr int STAGES = (RING / STAGE) > 12 ? 12 : (RING / STAGE);
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 512;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_leader(const void* p) {  // same smem offset, CTA rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(0u));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void umma_f16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {  // arrive on bar in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::
                   "r"(smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

// TMA 2-D load into this CTA's smem whose completion is counted on the LEADER's mbarrier
// (cta_group::2: the pair's stage is complete when both CTAs' bytes have landed)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_pair(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                   float* __restrict__ C, int64_t ldc, int M, int N, int tiles_m, int tiles, int kb, int bn,
                   int silu, const __nv_bfloat16* __restrict__ w_tiled) {
  using CF = PairCfg<BN>;
  constexpr int STAGES = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int half = bn / 2;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_w);
    tma_prefetch(&tm_x);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // leader: 4 local + 4 peer epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated before any remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // W: rows of this CTA's half (tiled layout: a 2-D view of 128-row tiles, one box = one
      // pre-swizzled tile; row-major: the usual 128B-swizzled map); X: this CTA's token half.
      // Every load completes on the leader's full[s]; the leader arms it for both CTAs.
      auto load_w = [&](uint8_t* dst, int k, int f0, int st) {
        const int row0 = f0 + (int)rank * BM;
        const int y = w_tiled != nullptr ? ((row0 / BM) * kb + k) * BM : row0;
        tma_load_2d_pair(dst, &tm_w, mapa_leader(&full[st]), w_tiled != nullptr ? 0 : k * BK, y);
      };
      auto arm = [&](int st) {
        if (rank == 0) mbar_expect_tx(&full[st], 2 * (CF::W_BYTES + half * BK * 2));
      };
      int i = 0;
      for (int t = pair; t < tiles && i < STAGES; t += npairs) {  // weights before the dependency wait
        const int f0 = (t / tiles_m) * PAIR_BM;
        for (int k = 0; k < kb && i < STAGES; ++k, ++i) {
          arm(i);
          load_w(smem + i * CF::STAGE, k, f0, i);
        }
      }
      const int prefetched = i;
      pdl_wait();
      pdl_launch();
      i = 0;
      for (int t = pair; t < tiles; t += npairs) {
        const int f0 = (t / tiles_m) * PAIR_BM;
        const int x0 = (t % tiles_m) * bn + (int)rank * half;
        for (int k = 0; k < kb; ++k, ++i) {
          const int st = i % STAGES;
          uint8_t* sw = smem + st * CF::STAGE;
          if (i >= prefetched) {
            mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
            arm(st);
            load_w(sw, k, f0, st);
          }
          tma_load_2d_pair(sw + CF::W_BYTES, &tm_x, mapa_leader(&full[st]), k * BK, x0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {  // MMA issuer (leader)
      const uint32_t idesc = umma_idesc_bf16(PAIR_BM, bn, false, false);
      int i = 0, j = 0, rs = 0, rph = 0;
      const uint64_t wdesc0 = umma_desc_kmajor_sw128(smem_u32(smem), 1024);
      (void)rs, (void)rph, (void)wdesc0;
      for (int t = pair; t < tiles; t += npairs, ++j) {
        const int buf = j & 1;
        mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        for (int k = 0; k < kb; ++k, ++i) {
#if STB_GEMM_RING_COUNTERS
          // ring slot / phase as counters: a modulo by a stage count that is not a power of two
          // sits on the issuing thread's critical path every stage (the MoE GEMM measured it)
          const int st = rs;
          mbar_wait(&full[st], rph);
          if (++rs == STAGES) rs = 0, rph ^= 1;
          const uint64_t adesc = wdesc0 + (uint64_t)((st * CF::STAGE) >> 4);
          const uint64_t bdesc = adesc + (CF::W_BYTES >> 4);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_f16_ss_pair(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (k > 0 || kk > 0) ? 1u : 0u);
#else
          const int st = i % STAGES;
          mbar_wait(&full[st], (i / STAGES) & 1);
          tc_fence_after();
          const uint32_t wa = smem_u32(smem + st * CF::STAGE);
          const uint32_t xa = wa + CF::W_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_f16_ss_pair(d, umma_desc_kmajor_sw128(wa + kk * 32, 1024), umma_desc_kmajor_sw128(xa + kk * 32, 1024),
                             idesc, (k > 0 || kk > 0) ? 1u : 0u);
#endif
          umma_commit_pair(&empty[st]);
        }
        umma_commit_pair(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5 -> TMEM lane quarters 2,3,0,1 of this CTA's 128 rows
    pdl_wait();
    const int quarter = warp & 3;
    const uint32_t acc_empty_leader = mapa_leader(&acc_empty[0]);
    int j = 0;
    for (int t = pair; t < tiles; t += npairs, ++j) {
      const int buf = j & 1;
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      const int feat = (t / tiles_m) * PAIR_BM + (int)rank * BM + quarter * 32 + lane;
      const int t0 = (t % tiles_m) * bn;
      const int ntok = min(bn, M - t0);
      const bool fok = feat < N;
      const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN;
      if (silu) {
        __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)t0 * ldc + (feat >> 1);
        const bool odd = lane & 1;
        for (int c = 0; c < bn; c += 32) {
          uint32_t r[32];
          tmem_ld32(base + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float mine = __uint_as_float(odd ? r[16 + q] : r[q]);
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(odd ? r[q] : r[16 + q]), 1);
            const int tok = c + (odd ? 16 + q : q);
            if (fok && tok < ntok)
              act[(int64_t)tok * ldc] = __float2bfloat16_rn(odd ? silu_gate(other, mine) : silu_gate(mine, other));
          }
        }
      } else {
        float* crow = C + (int64_t)t0 * ldc + feat;
        for (int c = 0; c < bn; c += 32) {
          uint32_t r[32];
          tmem_ld32(base + c, r);
          tmem_ld_wait();
          if (fok) {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (c + q < ntok) crow[(int64_t)(c + q) * ldc] = __uint_as_float(r[q]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc_empty_leader + buf * 8);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's last MMA reads and TMEM writes are done before dealloc
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(CF::TMEM_COLS));
}

// token-tile height for the pair schedule: waves over sms/2 pairs x (bn + fixed cost)
struct PairPlan {
  int bn, tiles_m;
};
PairPlan pair_plan(int M, int N, int sms) {
  const int tiles_n = N / PAIR_BM;
  const int pairs = sms / 2;
#ifndef STB_PAIR_TILE_COST
#define STB_PAIR_TILE_COST 48
#endif
  constexpr int kTileCost = STB_PAIR_TILE_COST;
  PairPlan best{256, (M + 255) / 256};
  long best_cost = -1;
  for (int nt = (M + 255) / 256; nt <= (M + 31) / 32; ++nt) {
    const int bn = (((M + nt - 1) / nt + 31) / 32) * 32;  // bn/2 a multiple of 16
    if (bn > 256) continue;
    const int tm = (M + bn - 1) / bn;
    const long tl = (long)tiles_n * tm;
    const long cost = ((tl + pairs - 1) / pairs) * (long)(bn + kTileCost);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = PairPlan{bn, tm};
    }
  }
  return best;
}

template <int BN>
int launch_pair(const void* X, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M, int N, int K,
                int bn, int tiles_m, int flags, cudaStream_t st) {
  using CF = PairCfg<BN>;
  CUtensorMap tw, tx;
  const bool tiled = (flags & STB_GEMM_W_TILED) != 0;
  if (tiled) {  // the tiled buffer as [tiles * 128 rows][64] (128 B rows), unswizzled boxes of one tile
    if (int rc = cached_map_raw(&tw, W, (int64_t)((N + BM - 1) / BM) * ((K + BK - 1) / BK) * BM)) return rc;
  } else if (int rc = cached_map(&tw, W, N, K, ldw, BM)) {
    return rc;
  }
  if (int rc = cached_map(&tx, X, M, K, lda, bn / 2)) return rc;
  const int tiles = (N / PAIR_BM) * tiles_m;
  const int pairs = std::min(sm_count() / 2, tiles);
  auto kern = gemm_bf16_pair<BN>;
  smem_attr_once(kern, CF::SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = CF::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;  // cluster shape comes from __cluster_dims__
  count_launch();
  const int silu = (flags & STB_GEMM_SILU_MUL) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tw, tx, C, ldc, M, N, tiles_m, tiles, (K + BK - 1) / BK, bn, silu,
                                     tiled ? (const __nv_bfloat16*)W : (const __nv_bfloat16*)nullptr);
  if (e != cudaSuccess) return fail(STB_ECUDA, "gemm_bf16 pair launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

// The pair schedule serves whole-tile (prefill-shaped) products with N a multiple of 256 and no
// fused epilogue beyond SiLU; STB200_GEMM_PAIR=0 disables it (A/B).
bool pair_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STB200_GEMM_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
// STB200_GEMM_PAIR=3 (A/B only): the round-1 rule (pairs only for >= 2 waves of pair tiles or long K)
bool pair_legacy() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STB200_GEMM_PAIR");
    on = (e && e[0] == '3') ? 1 : 0;
  }
  return on == 1;
}
// STB200_GEMM_PAIR=2: every whole-tile product with N % 256 == 0 on the pair kernel (the default now)
bool pair_forced() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STB200_GEMM_PAIR");
    on = (e && e[0] == '2') ? 1 : 0;
  }
  return on == 1;
}

template <int BN>
int launch(const void* X, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M, int N, int K,
           int mode, int flags, cudaStream_t st, const Epi& ep) {
  using CF = Cfg<BN>;
  CUtensorMap tw, tx;
  const bool tiled = (flags & STB_GEMM_W_TILED) != 0;
  if (tiled) {
    memset(&tw, 0, sizeof(tw));  // unused: the producer bulk-copies whole tiles
  } else if (int rc = cached_map(&tw, W, N, K, ldw, BM)) {
    return rc;
  }
  const int sms = sm_count();
  const Plan pl = plan(M, N, sms);
  if (ep.kind == 0 && mode == 0 && !pl.stream && M > 128 && N % PAIR_BM == 0 && !(flags & STB_GEMM_C_ZEROED) &&
      pair_enabled()) {
    // pairs pay off once there are >= 2 waves of pair tiles or long K (measured: gate-up, down,
    // LM head at M = 608..2080 gain 7-17%; QKV / O at M = 608 — one partial wave — lose 5-13%)
    // (QKV / O-shaped products, N <= 8192 with K = 4096, measured from 0.56 to 0.79 on the pair
    // path across boxes vs a steady 0.77-0.80 on the 1-CTA kernel: they stay there)
    // Every whole-tile product with N a multiple of 256 runs on CTA pairs: measured in the decode
    // step with one prefill run packed in (tools/profile_step.py --mix, B = 32, ctx 2k, same box,
    // alternating runs) 8.41 -> 7.47 ms at 150 new tokens, 9.54 -> 9.41 at 300, 12.19 -> 12.18
    // at 576, 18.06 -> 17.80 at 1000 — the earlier rule (pairs only with >= 2 waves of pair
    // tiles or K >= 8192, from microbenchmarks of single products) kept QKV / O and the
    // one-wave gate-up of small runs on the 1-CTA kernel. STB200_GEMM_PAIR=3 restores that rule.
    const PairPlan pp = pair_plan(M, N, sms);
    const long pair_tiles = (long)(N / PAIR_BM) * pp.tiles_m;
    if (!pair_legacy() || (pair_tiles >= 2L * (sms / 2) && N > 8192) || K >= 8192 || pair_forced())
      return launch_pair<256>(X, lda, W, ldw, C, ldc, M, N, K, pp.bn, pp.tiles_m, flags, st);
  }
  const int bn = pl.bn;
  if (int rc = cached_map(&tx, X, M, K, lda, bn)) return rc;
  Sched s;
  s.tiles_n = (N + BM - 1) / BM;
  s.tiles_m = pl.tiles_m;
  s.tiles = s.tiles_n * s.tiles_m;
  s.kb = (K + BK - 1) / BK;
  s.units = (int64_t)s.tiles * s.kb;
  s.stream = mode == 1 ? 0 : (mode >= 2 ? 1 : pl.stream);
  int grid = s.stream ? sms : (s.tiles < sms ? s.tiles : sms);
  if (mode >= 2 && mode < grid) grid = mode;
  if (s.stream && s.units < grid) grid = (int)s.units;
  if (s.stream && s.units * (int64_t)(grid + 1) >= (int64_t)1 << 31)
    return fail(STB_EINVAL, "gemm_bf16: %lld stream-K units exceed the 32-bit schedule", (long long)s.units);
  s.c_zeroed = (flags & STB_GEMM_C_ZEROED) ? 1 : 0;
  s.silu = (flags & STB_GEMM_SILU_MUL) ? 1 : 0;
  if (s.silu && (s.stream || N % 2))
    return fail(STB_EINVAL, "gemm_bf16: the SiLU-gate epilogue needs the tile schedule and even N");
  static int launch_seq = 0;
  s.tag = launch_seq++;
  static const int load_debug = getenv("STB200_GEMM_LOAD_DEBUG") ? atoi(getenv("STB200_GEMM_LOAD_DEBUG")) : 0;
  s.load_debug = load_debug;
  s.bar = grid_barrier(st);
  if (!s.bar) return fail(STB_ENOMEM, "gemm_bf16: barrier state");
  auto kern = ep.kind != 0 ? gemm_bf16_persistent<BN, true> : gemm_bf16_persistent<BN, false>;
  smem_attr_once(kern, CF::SMEM);
  if (ep.kind != 0 && s.stream && (C == nullptr || ep.cnt == nullptr))
    return fail(STB_EINVAL, "gemm_bf16_fused: the stream-K schedule needs the zeroed fp32 workspace");
  if (ep.kind != 0 && s.stream && s.tiles > kMaxTickets)
    return fail(STB_EINVAL, "gemm_bf16_fused: %d stream-K tiles exceed the ticket array", s.tiles);
  cudaError_t e = launch_k(kern, dim3(grid), dim3(kThreads), CF::SMEM, st, tw, tx, C, ldc, M, N, s, bn,
                           tiled ? (const __nv_bfloat16*)W : (const __nv_bfloat16*)nullptr, ep);
  if (e != cudaSuccess) return fail(STB_ECUDA, "gemm_bf16 launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

int dispatch(const void* A, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M, int N, int K,
             int split_k, int flags, cudaStream_t st, const Epi& ep) {
  if (M <= 16) return launch<16>(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, ep);
  if (M <= 32) return launch<32>(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, ep);
  if (M <= 64) return launch<64>(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, ep);
  if (M <= 128) return launch<128>(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, ep);
  return launch<256>(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, ep);
}

}  // namespace

namespace {
// one thread per 16-byte chunk of the tiled layout: gathers 8 bf16 of W (zero padding)
__global__ void weight_tile_kernel(const __nv_bfloat16* __restrict__ W, int64_t ldw, int N, int K, int kbs,
                                   int64_t chunks, uint4* __restrict__ out) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    const int pc = (int)(i & 7);              // physical chunk within the 128-byte row
    const int r = (int)((i >> 3) & (BM - 1));  // row within the tile
    const int64_t t = i >> 10;                // tile index = n_tile * kbs + k_tile
    const int c = pc ^ (r & 7);               // logical chunk stored at pc
    const int64_t row = (t / kbs) * BM + r;
    const int64_t col = (t % kbs) * BK + c * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < N) {
      const __nv_bfloat16* src = W + row * ldw + col;
      if (col + 8 <= K) {
        v = *reinterpret_cast<const uint4*>(src);
      } else if (col < K) {
        __nv_bfloat16 e[8];
        for (int j = 0; j < 8; ++j) e[j] = col + j < K ? src[j] : __float2bfloat16(0.f);
        v = *reinterpret_cast<const uint4*>(e);
      }
    }
    out[i] = v;
  }
}
}  // namespace

extern "C" int64_t stb_weight_tiled_elems(int N, int K) {
  if (N <= 0 || K <= 0) return 0;
  return (int64_t)((N + BM - 1) / BM) * ((K + BK - 1) / BK) * BM * BK;
}

extern "C" int stb_weight_tile(const void* W, int64_t ldw, int N, int K, void* out, void* stream) {
  if (N <= 0 || K <= 0) return STB_OK;
  if (ldw < K || ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(out)) & 15) || ldw % 8)
    return fail(STB_EINVAL, "weight_tile: W must be 16-byte aligned with ldw >= K, ldw %% 8 == 0");
  const int64_t chunks = stb_weight_tiled_elems(N, K) / 8;
  const int kbs = (K + BK - 1) / BK;
  const int grid = (int)std::min<int64_t>((chunks + 255) / 256, 148 * 16);
  launch_k(weight_tile_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)W, ldw, N, K,
           kbs, chunks, (uint4*)out);
  STB_CHECK_LAUNCH("weight_tile");
  return STB_OK;
}

// 1 when stb_gemm_bf16(split_k = 0) would run this shape stream-K (reductions into C)
extern "C" int stb_gemm_is_stream(int M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  return plan(M, N, sm_count()).stream;
}

// split_k: 0 = automatic schedule, 1 = tile schedule (no reductions), >= 2 = stream-K over
// min(split_k, SMs) CTAs (tests use it to force mid-tile splits).
// Debug only (not part of include/stb200.h): record per-CTA GEMM timelines into
// buf[cap][8] (device memory) — buf = NULL turns tracing off. Returns records written.
extern "C" int stb_debug_gemm_trace(void* buf, int cap) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n));
  unsigned long long* p = (unsigned long long*)buf;
  unsigned int c = (unsigned int)cap, z = 0;
  cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
  cudaMemcpyToSymbol(g_trace_cap, &c, sizeof(c));
  cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z));
  return (int)n;
}

extern "C" int stb_gemm_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M,
                             int N, int K, int split_k, int flags, void* stream) {
  if (M <= 0 || N <= 0) return STB_OK;
  if (K <= 0 || K % 8 != 0) return fail(STB_EINVAL, "gemm_bf16: K must be a positive multiple of 8");
  if (lda % 8 != 0 || (ldw % 8 != 0 && !(flags & STB_GEMM_W_TILED)))
    return fail(STB_EINVAL, "gemm_bf16: row strides must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15)
    return fail(STB_EINVAL, "gemm_bf16: operands must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  Epi none;
  memset(&none, 0, sizeof(none));
  return dispatch(A, lda, W, ldw, C, ldc, M, N, K, split_k, flags, st, none);
}

extern "C" int stb_debug_block_trace(void* buf, int cap) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, g_btrace_n, sizeof(n));
  unsigned long long* p = (unsigned long long*)buf;
  unsigned int c = (unsigned int)cap, z = 0;
  cudaMemcpyToSymbol(g_btrace, &p, sizeof(p));
  cudaMemcpyToSymbol(g_btrace_cap, &c, sizeof(c));
  cudaMemcpyToSymbol(g_btrace_n, &z, sizeof(z));
  return (int)n;
}

extern "C" int stb_gemm_block(const stb_block_op* ops, int n_ops, int M, void* stream) {
  if (!ops || n_ops < 1 || n_ops > kBlkMaxOps) return fail(STB_EINVAL, "gemm_block: 1..%d ops", kBlkMaxOps);
  if (M < 1 || M > 64) return fail(STB_EINVAL, "gemm_block: M = %d outside 1..64 (decode batches)", M);
  cudaStream_t st = (cudaStream_t)stream;
  BlkArgs a;
  memset(&a, 0, sizeof(a));
  a.n_ops = n_ops;
  a.M = M;
  a.bn = (M + 15) / 16 * 16;
  const int grid = sm_count();
  int ng = 0, nu = 0;
  for (int i = 0; i < n_ops; ++i) {
    const stb_block_op& o = ops[i];
    if (o.kind == STB_OP_GEMM) {
      if (ng >= kBlkMaxGemm) return fail(STB_EINVAL, "gemm_block: at most %d GEMMs", kBlkMaxGemm);
      if (!o.x || !o.w || !o.c || o.n <= 0 || o.k <= 0 || o.k % 8 || o.ldx % 8 || o.ldx < o.k || o.ldc < o.n)
        return fail(STB_EINVAL, "gemm_block: GEMM %d: bad operands", i);
      if ((reinterpret_cast<uintptr_t>(o.x) | reinterpret_cast<uintptr_t>(o.w)) & 15)
        return fail(STB_EINVAL, "gemm_block: GEMM %d: operands must be 16-byte aligned", i);
      BlkGemm& g = a.g[ng];
      if (int rc = cached_map(&g.tx, o.x, M, o.k, o.ldx, a.bn)) return rc;
      g.w = (const __nv_bfloat16*)o.w;
      g.c = o.c;
      g.ldc = o.ldc;
      g.N = o.n;
      Sched& s = g.s;
      s.stream = 1;
      s.tiles_n = (o.n + BM - 1) / BM;
      s.tiles_m = 1;
      s.tiles = s.tiles_n;
      s.kb = (o.k + BK - 1) / BK;
      s.units = (int64_t)s.tiles * s.kb;
      s.c_zeroed = 1;
      if (s.units * (int64_t)(grid + 1) >= (int64_t)1 << 31)
        return fail(STB_EINVAL, "gemm_block: GEMM %d has too many stream-K units", i);
      a.kind[i] = 0;
      a.idx[i] = (int8_t)ng;
      a.gneed[ng] = (int8_t)i;  // a barrier follows every op: op i starts after i completions
      ++ng;
      continue;
    }
    if (nu >= kBlkMaxGlue) return fail(STB_EINVAL, "gemm_block: at most %d row ops", kBlkMaxGlue);
    BlkGlue& u = a.u[nu];
    u.kind = o.kind;
    u.c = o.c;
    u.y = (__nv_bfloat16*)o.y;
    u.n = o.n;
    u.eps = o.eps;
    if (o.kind == STB_OP_NORM) {
      if (!o.x_res || o.n <= 0 || o.n % 4 || o.n > 8192 || (o.y && !o.w))
        return fail(STB_EINVAL, "gemm_block: NORM %d: needs x_res, d a multiple of 4 up to 8192, w with y", i);
      u.x = o.x_res;
      u.w = (const __nv_bfloat16*)o.w;
    } else if (o.kind == STB_OP_SILU) {
      if (!o.c || !o.y || o.n <= 0 || o.n % 4) return fail(STB_EINVAL, "gemm_block: SILU %d: bad operands", i);
    } else if (o.kind == STB_OP_ROPE) {
      stb_kv_pool* p = o.pool;
      if (!p || o.layer < 0 || o.layer >= p->layers || !o.c || !o.y || !o.slot_of || !o.pos_of || o.n_q <= 0 ||
          o.n_q % p->n_kv || p->d_head % 16 || (o.q_norm == nullptr) != (o.k_norm == nullptr))
        return fail(STB_EINVAL, "gemm_block: ROPE %d: bad operands", i);
      void *kp, *vp;
      stb_kv_layer_ptrs(p, o.layer, &kp, &vp);
      u.kpages = (__nv_bfloat16*)kp;
      u.vpages = (__nv_bfloat16*)vp;
      u.table = p->dev_table;
      u.max_bps = p->max_bps;
      u.n_q = o.n_q;
      u.n_kv = p->n_kv;
      u.d_head = p->d_head;
      u.slot_of = o.slot_of;
      u.pos_of = o.pos_of;
      u.inv_freq = stb_rope_inv_freq(o.rope_theta, p->d_head);
      if (!u.inv_freq) return fail(STB_ENOMEM, "gemm_block: inv_freq");
      u.q_norm = (const __nv_bfloat16*)o.q_norm;
      u.k_norm = (const __nv_bfloat16*)o.k_norm;
    } else {
      return fail(STB_EINVAL, "gemm_block: op %d has unknown kind %d", i, o.kind);
    }
    a.kind[i] = (int8_t)o.kind;
    a.idx[i] = (int8_t)nu;
    ++nu;
  }
  if (ng == 0) return fail(STB_EINVAL, "gemm_block: no GEMM in the chain");
  a.n_gemm = ng;
  a.bar = (unsigned*)stream_scratch(kScratchBlockBar, st, (kGenOff + 32) * sizeof(unsigned));
  if (!a.bar) return fail(STB_ENOMEM, "gemm_block: barrier state");
  static int launch_seq = 0;
  a.tag = launch_seq++;
  const int BNt = bn_template(M);
  if (BNt == 16) return launch_block<16>(a, grid, st);
  if (BNt == 32) return launch_block<32>(a, grid, st);
  return launch_block<64>(a, grid, st);
}

extern "C" int stb_gemm_bf16_fused(const void* A, int64_t lda, const void* W, int64_t ldw, float* work,
                                   int64_t ldwork, int M, int N, int K, int flags, const stb_gemm_epi* e,
                                   void* stream) {
  if (M <= 0 || N <= 0) return STB_OK;
  if (!e || e->kind < STB_EPI_SILU || e->kind > STB_EPI_RESID) return fail(STB_EINVAL, "gemm_bf16_fused: bad epilogue");
  if (K <= 0 || K % 8 != 0) return fail(STB_EINVAL, "gemm_bf16: K must be a positive multiple of 8");
  if (lda % 8 != 0 || (ldw % 8 != 0 && !(flags & STB_GEMM_W_TILED)))
    return fail(STB_EINVAL, "gemm_bf16: row strides must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15)
    return fail(STB_EINVAL, "gemm_bf16: operands must be 16-byte aligned");
  Epi ep;
  memset(&ep, 0, sizeof(ep));
  ep.kind = e->kind;
  ep.ss_in = e->ss_in;
  ep.ss_parts = e->ss_parts;
  ep.inv_dim = e->inv_dim;
  ep.eps = e->eps;
  ep.out = (__nv_bfloat16*)e->out;
  ep.ldo = e->ldo;
  ep.cnt = tile_tickets((cudaStream_t)stream);
  if (!ep.cnt) return fail(STB_ENOMEM, "gemm_bf16_fused: tickets");
  if (e->kind == STB_EPI_SILU && N % 2) return fail(STB_EINVAL, "gemm_bf16_fused: SiLU-gate needs even N");
  if (e->ss_in && (e->ss_parts <= 0 || e->ss_parts % 4 || e->ss_parts > kMaxSsParts ||
                   (reinterpret_cast<uintptr_t>(e->ss_in) & 15)))
    return fail(STB_EINVAL, "gemm_bf16_fused: ss_in needs 16-byte rows of ss_parts (multiple of 4, <= %d)",
                kMaxSsParts);
  if (e->kind == STB_EPI_RESID) {
    if (!e->x || !e->out || !e->ss_out) return fail(STB_EINVAL, "gemm_bf16_fused: RESID needs x, out, ss_out");
    if (e->ss_parts < (N + BM - 1) / BM || e->ss_parts % 4)
      return fail(STB_EINVAL, "gemm_bf16_fused: RESID needs ss_parts >= ceil(N/128), a multiple of 4");
    ep.x = e->x;
    ep.ldx = e->ldx;
    ep.ss_out = e->ss_out;
  }
  if (e->kind == STB_EPI_QKV) {
    stb_kv_pool* p = e->pool;
    if (!p || e->layer < 0 || e->layer >= p->layers) return fail(STB_EINVAL, "gemm_bf16_fused: QKV needs a pool layer");
    if ((e->q_norm == nullptr) != (e->k_norm == nullptr)) return fail(STB_EINVAL, "gemm_bf16_fused: q_norm/k_norm");
    ep.d_head = p->d_head;
    ep.n_kv = p->n_kv;
    ep.q_dim = e->n_q * p->d_head;
    ep.kv_dim = p->n_kv * p->d_head;
    if (ep.d_head % 32 || ep.d_head > 128 || ep.q_dim % BM || ep.kv_dim % BM || N != ep.q_dim + 2 * ep.kv_dim)
      return fail(STB_EINVAL, "gemm_bf16_fused: QKV needs d_head in {32,64,128} and 128-aligned q/kv widths");
    void *kp, *vp;
    stb_kv_layer_ptrs(p, e->layer, &kp, &vp);
    ep.kpages = (__nv_bfloat16*)kp;
    ep.vpages = (__nv_bfloat16*)vp;
    ep.table = p->dev_table;
    ep.max_bps = p->max_bps;
    ep.slot_of = e->slot_of;
    ep.pos_of = e->pos_of;
    ep.inv_freq = stb_rope_inv_freq(e->rope_theta, p->d_head);
    if (!ep.inv_freq) return fail(STB_ENOMEM, "gemm_bf16_fused: inv_freq");
    ep.q_norm = (const __nv_bfloat16*)e->q_norm;
    ep.k_norm = (const __nv_bfloat16*)e->k_norm;
    ep.qk_eps = e->qk_eps;
  }
  return dispatch(A, lda, W, ldw, work, ldwork, M, N, K, 0, flags | STB_GEMM_C_ZEROED, (cudaStream_t)stream, ep);
}
