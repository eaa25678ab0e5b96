// K2 — append-prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the prefill / verify / ingest charges of the reference engine
// (`engine.py:251,296,358`): n new query tokens of a resident sequence attend
// causally to its whole paged context (the new rows already committed by K1).
//
// One CTA per (two tiles of 128 packed query rows, kv head, sequence). GQA
// packing: row r = (query r / G, head r % G), so the G heads sharing a kv head
// share every K/V tile, and both query tiles share it too. Warp roles (320 thr):
//   warp 8     TMA producer: Q tiles A and B once (4-D map over [T][n_kv][G][D]),
//              then per KV tile of 128 keys the 8 K and 8 V pages through the
//              block table (2-D maps over the page pool, 16 x 64 boxes; pages are
//              stored pre-swizzled, so the boxes land in the 128B-swizzle layout
//              with no tensor-map swizzle) into a 2-stage ring
//   warp 9     MMA issuer (one thread), ping-pong over the two tiles:
//              S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
//              S = Q K^T into TMEM (M=128, N=128 keys, K=D); O += P V with P read
//              from TMEM (A operand) and V an MN-major B operand from smem
//   warps 0-3  softmax of tile A, warps 4-7 softmax of tile B: thread = row; one
//              pass over its S row (128 TMEM columns -> registers), exp2, row sum,
//              P packed to bf16 and stored back over S; O (in TMEM) is rescaled
//              only when a warp's running max moved. While one warpgroup does its
//              softmax the tensor core runs the other tile's MMAs. The softmax is
//              the pacing resource (16 MUFU ex2/clk/SM vs 1024 MMA clocks per tile):
//              scale/subtract and the row sum are packed f32x2 (FFMA2/FADD2), ex2
//              is the ftz SFU form, and 2 of every 8 column pairs are exponentiated
//              on the FMA pipe (exp2_emu2) on unmasked tiles.
// CTAs are issued longest-first (causal work grows with the query-tile index).
// TMEM (512 columns): S/P_A | S/P_B | O_A | O_B.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include "../../include/stb200.h"
#include "common.cuh"
#include "pool.cuh"

using namespace stb;

namespace {

constexpr int ROWS = 128;   // packed query rows per tile (UMMA M)
constexpr int KT = 128;     // keys per KV tile (UMMA N of S, K of P V)
constexpr int KV_STAGES = 2;
#ifndef STB_K2_HALVES
#define STB_K2_HALVES 1
#endif
// softmax threads per S row. 2 = each row split over two warps of the same TMEM lane quarter
// (64 columns each; only the row max is exchanged per KV tile), 16 softmax warps in all:
// measured slower (C5 ingest 1.01 -> 1.06 ms) — 576 threads cap registers at 96 and the
// row state spills; 1 (the default) keeps one thread per row at 168 registers
constexpr int kHalves = STB_K2_HALVES;
constexpr int kSoftWarps = 8 * kHalves;  // two Q tiles x 4 lane quarters x halves
constexpr int kThreads = 32 * (kSoftWarps + 2);
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxSplits = 18;     // KV splits per (query-tile pair, kv head, run) work unit (8 units x 18 = 144 CTAs)
#ifndef STB_K2_MIN_SPLIT_TILES
#define STB_K2_MIN_SPLIT_TILES 1
#endif
constexpr int kMinSplitTiles = STB_K2_MIN_SPLIT_TILES;  // fewest KV tiles a split CTA streams
template <int D>
constexpr int kPartFloats = 2 * ROWS * (D + 1);  // one split's partial rows: O/l of both tiles + lse

// KV splits of a unit whose query tiles need n_tiles KV tiles (identical in K2 and the merge)
__host__ __device__ __forceinline__ int unit_splits(int n_tiles, int max_splits) {
  return max(1, min(max_splits, n_tiles / kMinSplitTiles));
}

template <int D>
struct TcCfg {
  static constexpr int HALVES = D / 64;              // 64-column swizzle atoms along d
  static constexpr int Q_BYTES = ROWS * D * 2;       // per tile: [half][128 rows][64]
  static constexpr int KV_BYTES = KT * D * 2;        // one of K or V: [half][128 keys][64]
  static constexpr int STAGE = 2 * KV_BYTES;
  static constexpr int SMEM = 2 * Q_BYTES + KV_STAGES * STAGE + 1024 + 256;
  static constexpr int TMEM_COLS = 512;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// 2^x for a pair of x in [-126, 8] on the FMA pipe (FA4-style offload from the MUFU unit,
// which otherwise paces the softmax: 16 ex2/clk/SM against 8192 bf16 flop/clk/SM of MMA).
// Round-to-nearest split x = k + f with the 1.5*2^23 shifter (f in [-0.5, 0.5]), a cubic
// minimax for 2^f (max relative error 7.5e-5, far below the 3.9e-3 of the bf16 P it feeds),
// and k added straight into the exponent field: the shifter's low mantissa bits hold k, so
// bits(j) << 23 == k << 23 (mod 2^32).
__device__ __forceinline__ float2 exp2_emu2(float2 x) {
  const float2 shift = make_float2(12582912.f, 12582912.f);
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 j = __fadd2_rn(x, shift);
  const float2 f = __fadd2_rn(x, __fadd2_rn(shift, make_float2(-j.x, -j.y)));
  float2 p = __ffma2_rn(make_float2(0.0551716117f, 0.0551716117f), f, make_float2(0.24261117f, 0.24261117f));
  p = __ffma2_rn(p, f, make_float2(0.693261001f, 0.693261001f));
  p = __ffma2_rn(p, f, make_float2(0.999928071f, 0.999928071f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

#ifndef STB_EXP_EMU
#define STB_EXP_EMU 2  // column pairs in every 8 exponentiated on the FMA pipe (unmasked tiles)
#endif
constexpr float kRescaleSlack = 8.f;  // lazy rescale: keep the stale max until the row max grows by > 2^8

// One S row (KT fp32 scores in registers, already masked) -> bf16 P pairs + row sum.
// Scale-and-subtract and the row sum run as packed f32x2 (FFMA2 / FADD2); exponentials
// on MUFU (ex2.approx.ftz) except STB_EXP_EMU of every 8 pairs when EMU.
template <bool EMU, int NC>
__device__ __forceinline__ float exp_row(const uint32_t* v, uint32_t* pk, float qscale, float ref) {
  const float2 sc = make_float2(qscale, qscale), nr = make_float2(-ref, -ref);
  float2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    const float2 x = __ffma2_rn(make_float2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), sc, nr);
    float2 e;
    if (EMU && ((c / 2) % 8) < STB_EXP_EMU) {
      e = exp2_emu2(x);
    } else {
      e.x = fast_exp2(x.x);
      e.y = fast_exp2(x.y);
    }
    acc[(c / 2) % 4] = __fadd2_rn(acc[(c / 2) % 4], e);
    pk[c / 2] = pack_bf16(e.x, e.y);
  }
  const float2 a = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return a.x + a.y;
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ out,
                           const int32_t* __restrict__ table, int max_bps, const int32_t* __restrict__ slots,
                           const int32_t* __restrict__ q_start, const int32_t* __restrict__ ctx_lens, int n_kv,
                           float qscale, int max_splits, float* __restrict__ part, int window,
                           const float* __restrict__ sinks) {
  using CF = TcCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;  // tile A, then tile B
  uint8_t* sKV = sQ + 2 * CF::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + KV_STAGES * CF::STAGE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;              // [KV_STAGES]
  uint64_t* kv_empty = kv_full + KV_STAGES;  // [KV_STAGES]
  uint64_t* s_full = kv_empty + KV_STAGES;   // [2] per tile
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* o_done = p_full + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // longest-first order: the causal work of a CTA grows with its query-tile index, so the
  // linear launch order walks query tiles from the last down (all heads and runs of one
  // index before the next) and the short diagonal CTAs fill the tail of the last wave
  const int nyz = gridDim.y * gridDim.z;
  const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int bx = gridDim.x - 1 - lin / nyz;
  const int kh = (lin % nyz) % gridDim.y, zz = (lin % nyz) / gridDim.y;
  const int s = zz / max_splits, sp = zz % max_splits;  // run, KV split
  constexpr int QPT = ROWS / G;  // queries per tile
  // the run metadata and the block table are host-uploaded (not written by the preceding kernel),
  // so everything up to the first Q / K / V copy overlaps the preceding kernel's tail
  const int t0 = q_start[s], n = q_start[s + 1] - t0;
  const int qi0 = bx * 2 * QPT;
  if (qi0 >= n) return;
  const bool has_b = qi0 + QPT < n;
  const int ctx = ctx_lens[s];
  const int pos0 = ctx - n;  // absolute position of query 0
  const int q_last = min(n, qi0 + 2 * QPT) - 1;
  const int n_tiles = (pos0 + q_last) / KT + 1;  // KV tiles the query tiles need (causal)
  // sliding window (gpt-oss): the first query's window starts in tile j_lo; earlier tiles are
  // never loaded
  const int j_lo = window > 0 ? max(0, pos0 + qi0 - window + 1) / KT : 0;
  // KV split (launches with few work units, e.g. one verify pass): this CTA streams tiles
  // [j0, j0 + nt) and writes partial rows; attn_prefill_merge_kernel combines them
  const int nsplit = unit_splits(n_tiles - j_lo, max_splits);
  if (sp >= nsplit) return;
  const int j0 = j_lo + (n_tiles - j_lo) * sp / nsplit, nt = j_lo + (n_tiles - j_lo) * (sp + 1) / nsplit - j0;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128 * kHalves);
      mbar_init(&o_done[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == kSoftWarps + 1) tmem_alloc(tmem_slot, CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // q and this step's new K / V rows come from the preceding kernels
  pdl_launch();
  const uint32_t tmem = *tmem_slot;
  // column map: S/P of tile t at t*KT, O of tile t at 2*KT + t*D
  auto tS = [&](int t) { return tmem + t * KT; };
  auto tO = [&](int t) { return tmem + 2 * KT + t * D; };

  if (warp == kSoftWarps) {
    // ---------------- TMA producer
    const int32_t* row = table + (int64_t)slots[s] * max_bps;
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(q_full, 2 * CF::Q_BYTES);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < CF::HALVES; ++h)
          tma_load_4d(sQ + t * CF::Q_BYTES + h * ROWS * 128, &tm_q, q_full, h * 64, 0, kh, t0 + qi0 + t * QPT);
      // page ids one KV tile ahead: the block-table loads of tile jj + 1 are in flight while the
      // producer waits for tile jj's ring slot (they used to sit between the wait and the copies)
      // (pages past the context are still fetched: finite pool rows, masked to -inf)
      int pid[KT / 16];
      auto load_pids = [&](int j, int* dst) {
#pragma unroll
        for (int p = 0; p < KT / 16; ++p) dst[p] = __ldg(row + min(j * (KT / 16) + p, max_bps - 1));
      };
      load_pids(j0, pid);
      for (int jj = 0; jj < nt; ++jj) {
        const int st = jj % KV_STAGES;
        int nxt[KT / 16];
        if (jj + 1 < nt) load_pids(j0 + jj + 1, nxt);
        mbar_wait(&kv_empty[st], ((jj / KV_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], CF::STAGE);
        uint8_t* sk = sKV + st * CF::STAGE;
        uint8_t* sv = sk + CF::KV_BYTES;
#pragma unroll
        for (int p = 0; p < KT / 16; ++p) {
          const int prow = (pid[p] * n_kv + kh) * 16;
#pragma unroll
          for (int h = 0; h < CF::HALVES; ++h) {
            tma_load_2d(sk + h * KT * 128 + p * 16 * 128, &tm_k, &kv_full[st], h * 64, prow);
            tma_load_2d(sv + h * KT * 128 + p * 16 * 128, &tm_v, &kv_full[st], h * 64, prow);
          }
        }
        if (jj + 1 < nt) {
#pragma unroll
          for (int p = 0; p < KT / 16; ++p) pid[p] = nxt[p];
        }
      }
    }
    __syncwarp();
  } else if (warp == kSoftWarps + 1) {
    // ---------------- MMA issuer (ping-pong)
    if (elect_one()) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(ROWS, KT, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(ROWS, D, false, true);
      const int ntile_q = has_b ? 2 : 1;
      mbar_wait(q_full, 0);
      auto issue_s = [&](int t, int j) {
        const uint32_t ka = smem_u32(sKV + (j % KV_STAGES) * CF::STAGE);
        const uint32_t qa = smem_u32(sQ + t * CF::Q_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * ROWS * 128 + (kk % 4) * 32;
          umma_f16_ss(tS(t), umma_desc_kmajor_sw128(qa + off, 1024),
                      umma_desc_kmajor_sw128(ka + (kk / 4) * KT * 128 + (kk % 4) * 32, 1024), idesc_s, kk > 0);
        }
        umma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t va = smem_u32(sKV + (j % KV_STAGES) * CF::STAGE) + CF::KV_BYTES;
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk)  // P: 16 keys = 8 packed bf16x2 columns per k-step
          umma_f16_ts(tO(t), tS(t) + kk * 8, umma_desc_mnmajor_sw128(va + kk * 16 * 128, KT * 128, 1024), idesc_o,
                      (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&o_done[t]);
      };
      mbar_wait(&kv_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      if (ntile_q > 1) issue_s(1, 0);
      for (int j = 0; j < nt; ++j) {  // local tile index: ring slots and barrier phases
        const bool more = j + 1 < nt;
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, j);
        if (more) {
          mbar_wait(&kv_full[(j + 1) % KV_STAGES], ((j + 1) / KV_STAGES) & 1);
          tc_fence_after();
          issue_s(0, j + 1);
        }
        if (ntile_q > 1) {
          mbar_wait(&p_full[1], j & 1);
          tc_fence_after();
          issue_pv(1, j);
          if (more) issue_s(1, j + 1);
        }
        umma_commit(&kv_empty[j % KV_STAGES]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax: warps [0, 4H) tile A, [4H, 8H) tile B; thread = (row, column half)
    constexpr int NC = KT / kHalves;  // S columns per thread
    constexpr int OC = D / kHalves;   // O columns per thread (rescale, output)
    const int t = warp / (4 * kHalves);
    const int wt = warp % (4 * kHalves);
    const int quarter = wt & 3, hf = wt >> 2;
    const int r = quarter * 32 + lane;
    const bool tile_live = t == 0 || has_b;
    const int qi = qi0 + t * QPT + r / G;
    const int g = r % G;
    const bool live = tile_live && qi < n;
    const int qpos = pos0 + qi;                               // keys <= qpos are visible
    const int full_tiles = (pos0 + qi0 + t * QPT + 1) / KT;   // tiles visible to every row of this tile
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    __shared__ float xmax[2][2][kHalves][ROWS];  // [parity][tile][half][row]: partial row maxima
    auto tile_bar = [&]() {  // the tile's softmax threads
      if (kHalves > 1) asm volatile("bar.sync %0, %1;\n" ::"r"(1 + t), "r"(128 * kHalves) : "memory");
    };
    float m = -INFINITY, l = 0.f;
    // the softmax variant depends on the KV tile only, never on the row: a run whose query
    // count is not a multiple of 32 rows leaves a warp of the last tile partly live, and a
    // per-row choice ran both exp variants back to back on every KV tile of the longest CTA
    // (+80% at n=996). Dead rows of such a warp exponentiate finite scores (keys below the
    // first row's position, Q rows of the next run or TMA zero fill) and are never stored;
    // a split writes lse = -inf for them, so the merge weighs them 0. Warps with no live row
    // write zero P and skip the exponentials
    const bool warp_dead = !__any_sync(0xffffffffu, live);
    if (tile_live) {
      for (int jj = 0; jj < nt; ++jj) {
        const int j = j0 + jj;  // absolute KV tile (masking); jj: barrier phases
        mbar_wait(&s_full[t], jj & 1);
        tc_fence_after();
        if (warp_dead) {
          if (kHalves > 1) {
            xmax[jj & 1][t][hf][r] = -INFINITY;
            tile_bar();
          }
          uint32_t pk[NC / 2];
#pragma unroll
          for (int c = 0; c < NC / 2; ++c) pk[c] = 0u;
#pragma unroll
          for (int c = 0; c < NC / 2; c += 32) tmem_st32(tS(t) + lane_base + hf * (NC / 2) + c, pk + c);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&p_full[t]);
          continue;
        }
        uint32_t v[NC];
#pragma unroll
        for (int c = 0; c < NC; c += 32) tmem_ld32(tS(t) + lane_base + hf * NC + c, v + c);
        tmem_ld_wait();
        const int kbase = j * KT + hf * NC;
        const bool masked = j >= full_tiles || window > 0;
        if (masked) {
          const int klo = window > 0 ? qpos - window : -1;  // keys <= klo are outside the window
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (!live || kbase + c > qpos || kbase + c <= klo) v[c] = __float_as_uint(-INFINITY);
        }
        // tree-reduced row max (8 independent chains), then across the row's halves
        float mx8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = __uint_as_float(v[q]);
#pragma unroll
        for (int c = 8; c < NC; c += 8)
#pragma unroll
          for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], __uint_as_float(v[c + q]));
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if (kHalves > 1) {
          xmax[jj & 1][t][hf][r] = mx;
          tile_bar();
#pragma unroll
          for (int h2 = 0; h2 < kHalves; ++h2) mx = fmaxf(mx, xmax[jj & 1][t][h2][r]);
        }
        mx *= qscale;
        // lazy rescale (FA4): exponentiate against a stale reference while the row max stays
        // within 2^8 of it; exact because O and l always share the reference (both halves of
        // a row see the same maxima, so they keep the same reference)
        float alpha = 1.f;
        if (mx > m + kRescaleSlack || m == -INFINITY) {
          const float mn = fmaxf(m, mx);
          // a row that saw only masked keys has P = 0, so O = 0 and l = 0: no rescale (alpha 1
          // keeps dead rows off the O rescale path below)
          alpha = m == -INFINITY ? 1.f : exp2f(m - mn);
          m = mn;
        }
        const float ref = m == -INFINITY ? 0.f : m;
        uint32_t pk[NC / 2];
        const float rs = masked ? exp_row<false, NC>(v, pk, qscale, ref) : exp_row<true, NC>(v, pk, qscale, ref);
        l = l * alpha + rs;  // this half's share of the row sum (combined at the end)
        // P (bf16 pairs) over the S columns just read: the A operand of P V
#pragma unroll
        for (int c = 0; c < NC / 2; c += 32) tmem_st32(tS(t) + lane_base + hf * (NC / 2) + c, pk + c);
        // rescale this thread's O columns when the running max moved and O holds earlier tiles
        if (jj > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // rare with the lazy reference
          mbar_wait(&o_done[t], (jj - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < OC; c += 32) {
            uint32_t o[32];
            tmem_ld32(tO(t) + lane_base + hf * OC + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
            tmem_st32(tO(t) + lane_base + hf * OC + c, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      if (kHalves > 1) {  // the row sum: both halves' shares (parity buffer nt & 1 is free)
        xmax[nt & 1][t][hf][r] = l;
        tile_bar();
        l = 0.f;
#pragma unroll
        for (int h2 = 0; h2 < kHalves; ++h2) l += xmax[nt & 1][t][h2][r];
      }
      // final: O / l
      mbar_wait(&o_done[t], (nt - 1) & 1);
      tc_fence_after();
      if (sinks != nullptr && nsplit == 1 && m != -INFINITY)  // sink logit joins the denominator
        l += fast_exp2(sinks[kh * G + g] * kLog2e - m);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* dst = out + ((int64_t)(t0 + qi) * (n_kv * G) + kh * G + g) * D + hf * OC;
      float* prow = nullptr;  // split: this row's partial slot
      if (nsplit > 1) {
        float* po = part + ((((int64_t)s * n_kv + kh) * gridDim.x + bx) * max_splits + sp) * kPartFloats<D>;
        prow = po + (t * ROWS + r) * D + hf * OC;
        if (hf == 0) po[2 * ROWS * D + t * ROWS + r] = (live && l > 0.f) ? m + log2f(l) : -INFINITY;
      }
#pragma unroll
      for (int c = 0; c < OC; c += 32) {
        uint32_t o[32];
        tmem_ld32(tO(t) + lane_base + hf * OC + c, o);
        tmem_ld_wait();
        if (prow != nullptr) {
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            __stcg(reinterpret_cast<float4*>(prow + c + q),
                   make_float4(__uint_as_float(o[q]) * inv, __uint_as_float(o[q + 1]) * inv,
                               __uint_as_float(o[q + 2]) * inv, __uint_as_float(o[q + 3]) * inv));
        } else if (live) {
#pragma unroll
          for (int q = 0; q < 32; q += 8)
            *reinterpret_cast<uint4*>(dst + c + q) = make_uint4(
                pack_bf16(__uint_as_float(o[q]) * inv, __uint_as_float(o[q + 1]) * inv),
                pack_bf16(__uint_as_float(o[q + 2]) * inv, __uint_as_float(o[q + 3]) * inv),
                pack_bf16(__uint_as_float(o[q + 4]) * inv, __uint_as_float(o[q + 5]) * inv),
                pack_bf16(__uint_as_float(o[q + 6]) * inv, __uint_as_float(o[q + 7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kSoftWarps + 1) tmem_free(tmem, CF::TMEM_COLS);
}

// Combine the KV-split partial rows of K2: one warp per (tile, packed row) of a work unit,
// lane = 4 of the D columns (one float4 per split: all split loads in flight at once);
// out = sum_k 2^(lse_k - M) (O/l)_k / sum_k 2^(lse_k - M).
template <int D, int G>
__global__ void __launch_bounds__(256) attn_prefill_merge_kernel(__nv_bfloat16* __restrict__ out,
                                                                 const float* __restrict__ part,
                                                                 const int32_t* __restrict__ q_start,
                                                                 const int32_t* __restrict__ ctx_lens, int n_kv,
                                                                 int max_splits, int gx, int window,
                                                                 const float* __restrict__ sinks) {
  pdl_wait();
  pdl_launch();
  constexpr int QPT = ROWS / G;
  const int unit = blockIdx.x / (2 * ROWS / 8);              // 8 rows (warps) per block
  const int row = (blockIdx.x % (2 * ROWS / 8)) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int bx = unit % gx, kh = blockIdx.y, s = blockIdx.z;
  const int t0 = q_start[s], n = q_start[s + 1] - t0;
  const int qi0 = bx * 2 * QPT;
  if (qi0 >= n) return;
  const int pos0 = ctx_lens[s] - n;
  const int j_lo = window > 0 ? max(0, pos0 + qi0 - window + 1) / KT : 0;
  const int nsplit = unit_splits((pos0 + min(n, qi0 + 2 * QPT) - 1) / KT + 1 - j_lo, max_splits);
  if (nsplit == 1) return;  // K2 wrote this unit's rows directly
  const int t = row / ROWS, r = row % ROWS;
  const int qi = qi0 + t * QPT + r / G, g = r % G;
  if (qi >= n) return;
  const float* base = part + (((int64_t)s * n_kv + kh) * gx + bx) * max_splits * kPartFloats<D>;
  float w[kMaxSplits];
  float4 v[kMaxSplits];
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < kMaxSplits; ++k) {
    w[k] = -INFINITY;
    v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < nsplit) {
      const float* pk = base + k * kPartFloats<D>;
      w[k] = __ldcg(pk + 2 * ROWS * D + t * ROWS + r);
      if (lane < D / 4) v[k] = __ldcg(reinterpret_cast<const float4*>(pk + (t * ROWS + r) * D) + lane);
    }
    mx = fmaxf(mx, w[k]);
  }
  float wsum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kMaxSplits; ++k) {
    const float e = (k < nsplit && w[k] != -INFINITY) ? exp2f(w[k] - mx) : 0.f;
    wsum += e;
    acc.x += e * v[k].x, acc.y += e * v[k].y, acc.z += e * v[k].z, acc.w += e * v[k].w;
  }
  if (sinks != nullptr && mx != -INFINITY) wsum += exp2f(sinks[kh * G + g] * kLog2e - mx);
  const float winv = wsum > 0.f ? 1.f / wsum : 0.f;
  if (lane < D / 4) {
    __nv_bfloat16* dst = out + ((int64_t)(t0 + qi) * (n_kv * G) + kh * G + g) * D + lane * 4;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(acc.x * winv, acc.y * winv), pack_bf16(acc.z * winv, acc.w * winv));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
           const cuuint32_t* box, CUtensorMapSwizzle swizzle) {
  auto fn = encode_tiled();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "attn_prefill_tc: tensor map encode failed (%d)", (int)r);
  return STB_OK;
}

struct Maps {
  CUtensorMap q, k, v;
};

// Tensor maps of one launch geometry: everything the encoded maps depend on is in the key
// (a freed pool re-allocated at the same address with another num_blocks, or another layer
// geometry, must never hit a stale map: out-of-bounds boxes would silently zero-fill).
struct MapKey {
  const void* q;
  int64_t T;
  const void* kp;
  const void* vp;
  int64_t num_blocks;
  int n_kv, G, D, dev;
  bool operator<(const MapKey& o) const {
    return std::tie(q, T, kp, vp, num_blocks, n_kv, G, D, dev) <
           std::tie(o.q, o.T, o.kp, o.vp, o.num_blocks, o.n_kv, o.G, o.D, o.dev);
  }
};

template <int D, int G>
int launch_tc(const stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots, const int32_t* q_start,
              const int32_t* ctx, int S, int T, int n_kv, float qscale, int max_q, int active_hint, int window,
              const float* sinks, cudaStream_t st) {
  using CF = TcCfg<D>;
  // tensor maps: Q over [T][n_kv][G][D] (box 64 x G x 1 x 128/G), K / V pages of the layer as
  // [num_blocks * n_kv * 16 rows][D] (box 64 x 16); cached per (q base, T, layer pointers)
  static std::mutex mu;
  static std::map<MapKey, Maps> cache;
  void *kp, *vp;
  stb_kv_layer_ptrs(pool, layer, &kp, &vp);
  int dev = 0;
  cudaGetDevice(&dev);
  const MapKey key{q, (int64_t)T, kp, vp, (int64_t)pool->num_blocks, n_kv, G, D, dev};
  Maps mp;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      mp = it->second;
    } else {
      cuuint64_t qd[4] = {(cuuint64_t)D, (cuuint64_t)G, (cuuint64_t)n_kv, (cuuint64_t)T};
      cuuint64_t qs[3] = {(cuuint64_t)D * 2, (cuuint64_t)G * D * 2, (cuuint64_t)n_kv * G * D * 2};
      cuuint32_t qb[4] = {64, (cuuint32_t)G, 1, (cuuint32_t)(ROWS / G)};
      if (int rc = encode(&mp.q, q, 4, qd, qs, qb, CU_TENSOR_MAP_SWIZZLE_128B)) return rc;
      const cuuint64_t rows = (cuuint64_t)pool->num_blocks * n_kv * 16;
      cuuint64_t kd[2] = {(cuuint64_t)D, rows};
      cuuint64_t ks[1] = {(cuuint64_t)D * 2};
      cuuint32_t kb[2] = {64, 16};
      if (int rc = encode(&mp.k, kp, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return rc;
      if (int rc = encode(&mp.v, vp, 2, kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_NONE)) return rc;
      if (cache.size() > 4096) cache.clear();
      cache.emplace(key, mp);
    }
  }
  auto kern = attn_prefill_tc_kernel<D, G>;
  smem_attr_once(kern, CF::SMEM);
  const int gx = (max_q + 2 * ROWS / G - 1) / (2 * ROWS / G);
  // KV split only for launches far from filling the machine (a verify pass is 8 work units
  // on 148 SMs); `active_hint` = units that hold queries (0: the full grid)
  const int sms = device_sms();
  const int64_t units = (int64_t)gx * n_kv * S;
  const int64_t active = active_hint > 0 ? active_hint : units;
  static const int split_env = getenv("STB200_K2_SPLIT") ? atoi(getenv("STB200_K2_SPLIT")) : -1;  // A/B only
  int splits = 1;
  if (2 * active <= sms) splits = (int)std::min<int64_t>(kMaxSplits, sms / active);
  if (split_env >= 1) splits = std::min(split_env, kMaxSplits);
  // partials: fixed per-(device, stream) scratch for sms/2 units x kMaxSplits (a split is only
  // chosen for launches with fewer active units than half the SMs); a ragged grid whose
  // units x splits would not fit gets fewer splits, never a reallocation under a graph
  const size_t cap_units = (size_t)(sms / 2) * kMaxSplits;
  float* part = nullptr;
  if (splits > 1) {
    if ((size_t)units * splits > cap_units) splits = (int)(cap_units / (size_t)units);
    if (splits > 1) {
      part = (float*)stream_scratch(kScratchK2Split, st, cap_units * kPartFloats<D> * sizeof(float));
      if (!part) return fail(STB_ENOMEM, "attn_prefill split scratch");
    } else {
      splits = 1;
    }
  }
  dim3 grid(gx, n_kv, S * splits);
  cudaError_t e = launch_k(kern, grid, dim3(kThreads), CF::SMEM, st, mp.q, mp.k, mp.v, (__nv_bfloat16*)out,
                           pool->dev_table, pool->max_bps, slots, q_start, ctx, n_kv, qscale, splits, part, window,
                           sinks);
  if (e != cudaSuccess) return fail(STB_ECUDA, "attn_prefill_tc launch: %s", cudaGetErrorString(e));
  if (splits > 1) {
    e = launch_k(attn_prefill_merge_kernel<D, G>, dim3(gx * (2 * ROWS / 8), n_kv, S), dim3(256), 0, st,
                 (__nv_bfloat16*)out, (const float*)part, q_start, ctx, n_kv, splits, gx, window, sinks);
    if (e != cudaSuccess) return fail(STB_ECUDA, "attn_prefill merge launch: %s", cudaGetErrorString(e));
  }
  return STB_OK;
}

}  // namespace

// internal entry used by stb_attn_prefill (attention.cu) for tensor-core-sized runs
int stb_attn_prefill_tc(const stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                        const int32_t* q_start, const int32_t* ctx, int S, int T, int n_q, float scale, int max_q,
                        int active_hint, int window, const float* sinks, void* stream) {
  int n_kv = pool->n_kv, d = pool->d_head;
  int g = n_q / n_kv;
  float qs = scale * kLog2e;
  cudaStream_t st = (cudaStream_t)stream;
#define ARGS pool, layer, q, out, slots, q_start, ctx, S, T, n_kv, qs, max_q, active_hint, window, sinks, st
  if (d == 128 && g == 4) return launch_tc<128, 4>(ARGS);
  if (d == 128 && g == 8) return launch_tc<128, 8>(ARGS);
  if (d == 128 && g == 1) return launch_tc<128, 1>(ARGS);
  if (d == 64 && g == 2) return launch_tc<64, 2>(ARGS);
  if (d == 64 && g == 8) return launch_tc<64, 8>(ARGS);
  if (d == 64 && g == 4) return launch_tc<64, 4>(ARGS);
#undef ARGS
  return fail(STB_EINVAL, "attn_prefill_tc: unsupported (d_head=%d, group=%d)", d, g);
}
