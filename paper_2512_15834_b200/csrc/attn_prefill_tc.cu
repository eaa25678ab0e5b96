// K2 — append-prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the prefill / verify / ingest charges of the reference engine
// (`engine.py:251,296,358`): n new query tokens of a resident sequence attend
// causally to its whole paged context (the new rows already committed by K1).
//
// One CTA per (tile of 128 packed query rows, kv head, sequence). GQA packing:
// row r = (query r / G, head r % G) so the G heads sharing a kv head share every
// K/V tile. Warp roles (192 threads):
//   warp 4  TMA producer: Q once (4-D map over [T][n_kv][G][D]), then per KV tile
//           of 128 keys the 8 K pages and 8 V pages through the block table
//           (2-D maps over the page pool, 16 x 64 boxes, 128B swizzle) into a
//           2-stage ring
//   warp 5  MMA issuer: S = Q K^T (M=128, N=128 keys, K=D) into TMEM; after the
//           softmax wrote P, O_tile = P V (M=128, N=D, K=128 keys; V is an
//           MN-major B operand) into a second TMEM region
//   warps 0-3  softmax: thread = row (TMEM lane), two passes over its S row
//           (max, then exp2 / sum / bf16 pack into the swizzled P tile), then
//           O = O * alpha + O_tile in registers; final O / l to global
// TMEM: 128 columns S + D columns O_tile.
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "../../include/stb200.h"
#include "common.cuh"
#include "pool.cuh"

using namespace stb;

namespace {

constexpr int ROWS = 128;   // packed query rows per CTA (UMMA M)
constexpr int KT = 128;     // keys per KV tile (UMMA N of S, K of P V)
constexpr int KV_STAGES = 2;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct TcCfg {
  static constexpr int HALVES = D / 64;              // 64-column swizzle atoms along d
  static constexpr int Q_BYTES = ROWS * D * 2;       // [half][128 rows][64]
  static constexpr int KV_BYTES = KT * D * 2;        // one of K or V: [half][128 keys][64]
  static constexpr int P_BYTES = ROWS * KT * 2;      // [key half][128 rows][64 keys]
  static constexpr int STAGE = 2 * KV_BYTES;
  static constexpr int SMEM = Q_BYTES + KV_STAGES * STAGE + P_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = (KT + D) <= 256 ? 256 : 512;
};

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ out,
                           const int32_t* __restrict__ table, int max_bps, const int32_t* __restrict__ slots,
                           const int32_t* __restrict__ q_start, const int32_t* __restrict__ ctx_lens, int n_kv,
                           float qscale) {
  using CF = TcCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + CF::Q_BYTES;
  uint8_t* sP = sKV + KV_STAGES * CF::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + CF::P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;             // [KV_STAGES]
  uint64_t* kv_empty = kv_full + KV_STAGES; // [KV_STAGES]
  uint64_t* s_full = kv_empty + KV_STAGES;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;
  uint64_t* pv_full = p_full + 1;
  uint64_t* pv_free = pv_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.z, kh = blockIdx.y;
  constexpr int QPT = ROWS / G;  // queries per tile
  pdl_wait();
  pdl_launch();
  const int t0 = q_start[s], n = q_start[s + 1] - t0;
  const int qi0 = blockIdx.x * QPT;
  if (qi0 >= n) return;
  const int ctx = ctx_lens[s];
  const int pos0 = ctx - n;                            // absolute position of query 0
  const int q_last = min(n, qi0 + QPT) - 1;            // last query of this tile
  const int n_tiles = (pos0 + q_last) / KT + 1;        // KV tiles the tile needs (causal)
  const int full_tiles = (pos0 + qi0 + 1) / KT;        // tiles visible to every row of the tile

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 128);
    mbar_init(p_full, 128);
    mbar_init(pv_full, 1);
    mbar_init(pv_free, 128);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + KT;

  if (warp == 4) {
    // ---------------- TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(q_full, CF::Q_BYTES);
#pragma unroll
      for (int h = 0; h < CF::HALVES; ++h)
        tma_load_4d(sQ + h * ROWS * 128, &tm_q, q_full, h * 64, 0, kh, t0 + qi0);
      const int32_t* row = table + (int64_t)slots[s] * max_bps;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KV_STAGES;
        mbar_wait(&kv_empty[st], ((j / KV_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], CF::STAGE);
        uint8_t* sk = sKV + st * CF::STAGE;
        uint8_t* sv = sk + CF::KV_BYTES;
#pragma unroll
        for (int p = 0; p < KT / 16; ++p) {
          // pages past the context are still fetched (finite pool rows; masked to -inf)
          const int page = min(j * (KT / 16) + p, max_bps - 1);
          const int prow = (row[page] * n_kv + kh) * 16;
#pragma unroll
          for (int h = 0; h < CF::HALVES; ++h) {
            tma_load_2d(sk + h * KT * 128 + p * 16 * 128, &tm_k, &kv_full[st], h * 64, prow);
            tma_load_2d(sv + h * KT * 128 + p * 16 * 128, &tm_v, &kv_full[st], h * 64, prow);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(ROWS, KT, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(ROWS, D, false, true);
      mbar_wait(q_full, 0);
      const uint32_t qa = smem_u32(sQ);
      const uint32_t pa = smem_u32(sP);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KV_STAGES;
        const uint32_t ka = smem_u32(sKV + st * CF::STAGE);
        const uint32_t va = ka + CF::KV_BYTES;
        mbar_wait(&kv_full[st], (j / KV_STAGES) & 1);
        mbar_wait(s_free, (j & 1) ^ 1);  // softmax finished reading S of tile j-1
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * ROWS * 128 + (kk % 4) * 32;
          umma_f16_ss(tS, umma_desc_kmajor_sw128(qa + off, 1024),
                      umma_desc_kmajor_sw128(ka + (kk / 4) * KT * 128 + (kk % 4) * 32, 1024), idesc_s, kk > 0);
        }
        umma_commit(s_full);
        mbar_wait(p_full, j & 1);         // P of tile j is in smem
        mbar_wait(pv_free, (j & 1) ^ 1);  // O_tile of tile j-1 consumed
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk) {
          // A = P (K-major over keys), B = V (MN-major: rows = keys, 64-wide d halves LBO apart)
          umma_f16_ss(tO, umma_desc_kmajor_sw128(pa + (kk / 4) * ROWS * 128 + (kk % 4) * 32, 1024),
                      umma_desc_mnmajor_sw128(va + kk * 16 * 128, KT * 128, 1024), idesc_o, kk > 0);
        }
        umma_commit(pv_full);
        umma_commit(&kv_empty[st]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax / output warps: thread = row
    const int r = warp * 32 + lane;
    const int qi = qi0 + r / G;
    const int g = r % G;
    const bool live = qi < n;
    const int qpos = pos0 + qi;  // keys <= qpos are visible
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float o[D];
#pragma unroll
    for (int c = 0; c < D; ++c) o[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int kbase = j * KT;
      const bool full = j < full_tiles;
      // pass 1: row max
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KT; c += 16) {
        uint32_t v[16];
        tmem_ld16(tS + lane_base + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float x = __uint_as_float(v[q]) * qscale;
          if (!full && (kbase + c + q > qpos || !live)) x = -INFINITY;
          mx = fmaxf(mx, x);
        }
      }
      const float mn = fmaxf(m, mx);
      const float ref = mn == -INFINITY ? 0.f : mn;
      const float alpha = exp2f(m - ref);
      m = mn;
      // pass 2: p = exp2(s - m), row sum, bf16 P tile (wait until P V of tile j-1 read P)
      if (j > 0) mbar_wait(pv_full, (j - 1) & 1);
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < KT; c += 16) {
        uint32_t v[16];
        tmem_ld16(tS + lane_base + c, v);
        tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          float x0 = __uint_as_float(v[q]) * qscale, x1 = __uint_as_float(v[q + 1]) * qscale;
          if (!full && (kbase + c + q > qpos || !live)) x0 = -INFINITY;
          if (!full && (kbase + c + q + 1 > qpos || !live)) x1 = -INFINITY;
          const float e0 = exp2f(x0 - ref), e1 = exp2f(x1 - ref);
          rs += e0 + e1;
          pk[q / 2] = pack_bf16(e0, e1);
        }
        // 32 bytes of row r, keys c..c+15 -> two swizzled 16B chunks of the K-major P tile
        const int half = c / 64, ch = (c % 64) / 8;
        uint8_t* prow = sP + half * ROWS * 128 + r * 128;
        *reinterpret_cast<uint4*>(prow + ((ch ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(prow + (((ch + 1) ^ (r & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      l = l * alpha + rs;
      tc_fence_before();
      mbar_arrive(s_free);   // S region may be overwritten by the next tile's QK^T
      fence_async_smem();    // make the P stores visible to the tensor core (async proxy)
      mbar_arrive(p_full);
      // O = O * alpha + P V
      mbar_wait(pv_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D; c += 16) {
        uint32_t v[16];
        tmem_ld16(tO + lane_base + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) o[c + q] = o[c + q] * alpha + __uint_as_float(v[q]);
      }
      tc_fence_before();
      mbar_arrive(pv_free);
    }
    if (live) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* dst = out + ((int64_t)(t0 + qi) * (n_kv * G) + kh * G + g) * D;
#pragma unroll
      for (int c = 0; c < D; c += 8) {
        *reinterpret_cast<uint4*>(dst + c) =
            make_uint4(pack_bf16(o[c] * inv, o[c + 1] * inv), pack_bf16(o[c + 2] * inv, o[c + 3] * inv),
                       pack_bf16(o[c + 4] * inv, o[c + 5] * inv), pack_bf16(o[c + 6] * inv, o[c + 7] * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_free(tmem, CF::TMEM_COLS);
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
           const cuuint32_t* box) {
  auto fn = encode_tiled();
  if (!fn) return fail(STB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STB_ECUDA, "attn_prefill_tc: tensor map encode failed (%d)", (int)r);
  return STB_OK;
}

struct Maps {
  CUtensorMap q, k, v;
};

template <int D, int G>
int launch_tc(const stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots, const int32_t* q_start,
              const int32_t* ctx, int S, int T, int n_kv, float qscale, int max_q, cudaStream_t st) {
  using CF = TcCfg<D>;
  // tensor maps: Q over [T][n_kv][G][D] (box 64 x G x 1 x 128/G), K / V pages of the layer as
  // [num_blocks * n_kv * 16 rows][D] (box 64 x 16); cached per (q base, T, layer pointers)
  static std::mutex mu;
  static std::unordered_map<uint64_t, Maps> cache;
  void *kp, *vp;
  stb_kv_layer_ptrs(pool, layer, &kp, &vp);
  const uint64_t key = reinterpret_cast<uint64_t>(q) * 1000003ull ^ (uint64_t)T * 7919ull ^ reinterpret_cast<uint64_t>(kp);
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
      if (int rc = encode(&mp.q, q, 4, qd, qs, qb)) return rc;
      const cuuint64_t rows = (cuuint64_t)pool->num_blocks * n_kv * 16;
      cuuint64_t kd[2] = {(cuuint64_t)D, rows};
      cuuint64_t ks[1] = {(cuuint64_t)D * 2};
      cuuint32_t kb[2] = {64, 16};
      if (int rc = encode(&mp.k, kp, 2, kd, ks, kb)) return rc;
      if (int rc = encode(&mp.v, vp, 2, kd, ks, kb)) return rc;
      if (cache.size() > 4096) cache.clear();
      cache.emplace(key, mp);
    }
  }
  auto kern = attn_prefill_tc_kernel<D, G>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    attr = true;
  }
  dim3 grid((max_q + ROWS / G - 1) / (ROWS / G), n_kv, S);
  cudaError_t e = launch_k(kern, grid, dim3(kThreads), CF::SMEM, st, mp.q, mp.k, mp.v, (__nv_bfloat16*)out,
                           pool->dev_table, pool->max_bps, slots, q_start, ctx, n_kv, qscale);
  if (e != cudaSuccess) return fail(STB_ECUDA, "attn_prefill_tc launch: %s", cudaGetErrorString(e));
  return STB_OK;
}

}  // namespace

// internal entry used by stb_attn_prefill (attention.cu) for tensor-core-sized runs
int stb_attn_prefill_tc(const stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                        const int32_t* q_start, const int32_t* ctx, int S, int T, int n_q, float scale, int max_q,
                        void* stream) {
  int n_kv = pool->n_kv, d = pool->d_head;
  int g = n_q / n_kv;
  float qs = scale * kLog2e;
  cudaStream_t st = (cudaStream_t)stream;
#define ARGS pool, layer, q, out, slots, q_start, ctx, S, T, n_kv, qs, max_q, st
  if (d == 128 && g == 4) return launch_tc<128, 4>(ARGS);
  if (d == 128 && g == 8) return launch_tc<128, 8>(ARGS);
  if (d == 128 && g == 1) return launch_tc<128, 1>(ARGS);
  if (d == 64 && g == 2) return launch_tc<64, 2>(ARGS);
  if (d == 64 && g == 8) return launch_tc<64, 8>(ARGS);
  if (d == 64 && g == 4) return launch_tc<64, 4>(ARGS);
#undef ARGS
  return fail(STB_EINVAL, "attn_prefill_tc: unsupported (d_head=%d, group=%d)", d, g);
}
