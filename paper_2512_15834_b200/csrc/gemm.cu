// K5 — bf16 projection / MLP GEMM on the 5th-gen tensor cores.
//
// C[M][N] (fp32) = X[M][K] (bf16 activations) * W[N][K]^T (bf16 weights).
// Replaces, with real FLOPs, every `rate x tokens` charge of the reference engine
// (`engine.py:251,270,296,358`): the QKV / O / gate-up / down / LM-head projections.
//
// Weight-stationary tiling: the 128-row MMA "M" side is always 128 weight rows
// (output features) and the MMA "N" side is BN tokens (16..256). Decode steps
// (M = batch = 32) then run 128 x 32 UMMAs instead of padding the batch to 128,
// and prefill/ingest (M = thousands of tokens) run 128 x 256. Operands are
// K-major and arrive by TMA with 128-byte swizzle into a STAGES-deep smem ring;
// one elected thread issues tcgen05.mma (kind::f16, fp32 accumulate in TMEM);
// tcgen05.commit releases ring slots back to the TMA producer; after the last
// K block all four warps drain their 32 TMEM lanes with tcgen05.ld and store
// fp32 rows (coalesced across the 32 features a warp owns). When the tile grid
// is smaller than the SM count the K loop is split and partial tiles are
// reduced with fp32 red.global.add into a zeroed C (decode-shaped GEMMs are
// HBM-bound on the weights: the split keeps all 148 SMs streaming).
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "../../include/stb200.h"
#include "common.cuh"

using namespace stb;

namespace {

constexpr int BM = 128;  // weight rows per tile (UMMA M)
constexpr int BK = 64;   // K per stage: one 128-byte swizzle atom of bf16

template <int BN>
struct Cfg {
  static constexpr int W_BYTES = BM * BK * 2;
  static constexpr int X_BYTES = BN * BK * 2;
  static constexpr int STAGE = W_BYTES + X_BYTES;
  static constexpr int STAGES = (196 * 1024 / STAGE) > 8 ? 8 : (196 * 1024 / STAGE);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                        float* __restrict__ C, int64_t ldc, int M, int N, int kb_per_split, int kb_total) {
  using CF = Cfg<BN>;
  constexpr int STAGES = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f0 = blockIdx.x * BM;
  const int t0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(kb_total, kb0 + kb_per_split);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_w);
    tma_prefetch(&tm_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // TMA producer
      for (int i = 0; i < nkb; ++i) {
        int s = i % STAGES;
        uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sw = smem + s * CF::STAGE;
        mbar_expect_tx(&full[s], CF::STAGE);
        int kx = (kb0 + i) * BK;
        tma_load_2d(sw, &tm_w, &full[s], kx, f0);
        tma_load_2d(sw + CF::W_BYTES, &tm_x, &full[s], kx, t0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // MMA issuer: D[128 x BN] += W[128 x 64] * X[BN x 64]^T per stage, 4 UMMA_K=16 steps
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, false, false);
      for (int i = 0; i < nkb; ++i) {
        int s = i % STAGES;
        uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        uint32_t wa = smem_u32(smem + s * CF::STAGE);
        uint32_t xa = wa + CF::W_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          uint64_t da = umma_desc_kmajor_sw128(wa + k * 32, 1024);
          uint64_t db = umma_desc_kmajor_sw128(xa + k * 32, 1024);
          umma_f16_ss(tmem, da, db, idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
  }

  // epilogue: every warp drains its 32 TMEM lanes (= 32 weight rows / output features)
  if (nkb > 0) {
    mbar_wait(done, 0);
    tc_fence_after();
    const int feat = f0 + warp * 32 + lane;
    const bool split = gridDim.z > 1;
#pragma unroll 1
    for (int c = 0; c < BN / 16; ++c) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c * 16, r);
      tmem_ld_wait();
      if (feat < N) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          int tok = t0 + c * 16 + j;
          if (tok < M) {
            float v = __uint_as_float(r[j]);
            float* dst = C + (int64_t)tok * ldc + feat;
            if (split)
              atomicAdd(dst, v);
            else
              *dst = v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free(tmem, CF::TMEM_COLS);
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
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return STB_OK;
}

template <int BN>
int launch(const void* X, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M, int N, int K,
           int split_k, cudaStream_t st) {
  using CF = Cfg<BN>;
  CUtensorMap tw, tx;
  if (int rc = cached_map(&tw, W, N, K, ldw, BM)) return rc;
  if (int rc = cached_map(&tx, X, M, K, lda, BN)) return rc;
  int kb_total = (K + BK - 1) / BK;
  int tiles = ((N + BM - 1) / BM) * ((M + BN - 1) / BN);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int splits = split_k;
  if (splits <= 0) {
    splits = 1;
    if (tiles < sms) splits = (2 * sms + tiles - 1) / tiles;  // ~2 waves of K slices
    int max_s = kb_total / 4 > 0 ? kb_total / 4 : 1;          // keep >= 4 K blocks per slice
    if (splits > max_s) splits = max_s;
  }
  if (splits > kb_total) splits = kb_total;
  int kbps = (kb_total + splits - 1) / splits;
  splits = (kb_total + kbps - 1) / kbps;
  if (splits > 1) cudaMemsetAsync(C, 0, sizeof(float) * ((size_t)(M - 1) * ldc + N), st);
  auto kern = gemm_bf16_tn_kernel<BN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
  dim3 grid((N + BM - 1) / BM, (M + BN - 1) / BN, splits);
  kern<<<grid, 128, CF::SMEM, st>>>(tw, tx, C, ldc, M, N, kbps, kb_total);
  count_launch();
  STB_CHECK_LAUNCH("gemm_bf16");
  return STB_OK;
}

}  // namespace

extern "C" int stb_gemm_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, float* C, int64_t ldc, int M,
                             int N, int K, int split_k, void* stream) {
  if (M <= 0 || N <= 0) return STB_OK;
  if (K <= 0 || K % 8 != 0) return fail(STB_EINVAL, "gemm_bf16: K must be a positive multiple of 8");
  if (lda % 8 != 0 || ldw % 8 != 0) return fail(STB_EINVAL, "gemm_bf16: row strides must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15)
    return fail(STB_EINVAL, "gemm_bf16: operands must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (M <= 16) return launch<16>(A, lda, W, ldw, C, ldc, M, N, K, split_k, st);
  if (M <= 32) return launch<32>(A, lda, W, ldw, C, ldc, M, N, K, split_k, st);
  if (M <= 64) return launch<64>(A, lda, W, ldw, C, ldc, M, N, K, split_k, st);
  if (M <= 128) return launch<128>(A, lda, W, ldw, C, ldc, M, N, K, split_k, st);
  return launch<256>(A, lda, W, ldw, C, ldc, M, N, K, split_k, st);
}
