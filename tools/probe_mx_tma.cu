// Probe (not product code): the hardware-unpacking operand path for the block-scaled MXFP4 GEMM.
// (a) packed e2m1 codes [128 rows][64 B] loaded by TMA with CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B
//     (3-D map over stages of 8704 B: 8192 B of codes + 512 B of scale words), 128-byte swizzle;
// (b) the weight scale words staged [lane l][column j] = row 32 j + l (512 B) and moved to TMEM by
//     tcgen05.cp.32x128b.warpx4 issued by the MMA thread; (c) the token scale words likewise.
// Checked against a host double product, as tools/probe_mxf8f6f4.cu.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe_mx_tma.cu -o tools/probe_mx_tma.bin -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2512_15834_b200/csrc/common.cuh"

using namespace stb;

constexpr int M = 128, K = 128, STAGE = 8704;

__device__ __forceinline__ void umma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                        uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void tc_cp_32x128b_x4(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n" ::"r"(taddr), "l"(desc));
}
// bounded wait: returns false after ~2^22 polls (so a wrong transaction count reports instead of hanging)
__device__ __forceinline__ bool mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (int it = 0; it < (1 << 22); ++it) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    if (ok) return true;
  }
  return false;
}
__device__ __forceinline__ uint64_t plain_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // no swizzle
}

// w: stage 0 of [stages][8704]; sfa_perm: 512 B [l][j]; b: [N][128] e4m3; sfb_perm: [l][c] words (c < 4)
__global__ void probe(const __grid_constant__ CUtensorMap tm, const uint8_t* w, const uint8_t* b,
                      const uint32_t* sfb_perm, float* out, int N, int mode, int lbo, int sbo) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                // 128 rows x 128 B (unpacked by TMA)
  uint8_t* sb = sm + 16384;        // N rows x 128 B
  uint8_t* ssfa = sb + 256 * 128;  // 512 B
  uint8_t* ssfb = ssfa + 512;      // 512 B
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar, (mode & 2 ? 8192 : 16384) + 512);
    tma_load_3d(sa, &tm, &bar, 0, 0, 0);
    bulk_load(smem_u32(ssfa), w + 8192, 512, &bar);
  }
  for (int n = tid; n < N; n += 128)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(sb + n * 128 + ((c ^ (n & 7)) * 16)) = *reinterpret_cast<const uint4*>(b + n * 128 + c * 16);
  reinterpret_cast<uint32_t*>(ssfb)[tid] = sfb_perm[tid];
  if (warp == 0) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t SFA_COL = 256, SFB_COL = 272;
  __shared__ int s_ok;
  if (tid == 0) {
    s_ok = mbar_wait_bounded(&bar, 0);
    if (!s_ok) out[M * N + 63] = -1.f;
  }
  __syncthreads();
  if (!s_ok) {
    if (warp == 0) tmem_free(tmem, 512);
    return;
  }
  if (tid == 0) {
    tc_fence_after();
    tc_cp_32x128b_x4(tmem + SFA_COL, plain_desc(smem_u32(ssfa), lbo, sbo));
    tc_cp_32x128b_x4(tmem + SFB_COL, plain_desc(smem_u32(ssfb), lbo, sbo));
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t idesc = (5u << 7) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
      idesc |= ((uint32_t)kk << 29) | ((uint32_t)kk << 4);
      const uint64_t ad = umma_desc_kmajor_sw128(smem_u32(sa), 1024) + 2 * kk;
      const uint64_t bd = umma_desc_kmajor_sw128(smem_u32(sb), 1024) + 2 * kk;
      umma_mx(tmem, ad, bd, idesc, (tmem + SFA_COL) | ((uint32_t)kk << 30), (tmem + SFB_COL) | ((uint32_t)kk << 30),
              kk > 0 ? 1u : 0u);
    }
    umma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  if (mode == 1 && tid == 0) {  // dump the unpacked smem row 0 / 1 for inspection
    for (int j = 0; j < 64; ++j) out[M * N + j] = sa[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

static double e2m1(int c) {
  static const double v[8] = {0, 0.5, 1, 1.5, 2, 3, 4, 6};
  return (c & 8 ? -1 : 1) * v[c & 7];
}
static double e4m3(int c) {
  const int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
  const double mag = e == 0 ? std::ldexp(m / 8.0, -6) : std::ldexp(1 + m / 8.0, e - 7);
  return s ? -mag : mag;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  srand(4321);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int N : {32, 64}) {
    std::vector<uint8_t> w(2 * STAGE), bb(N * 128);
    std::vector<uint32_t> sfb_perm(128, 0x7f7f7f7fu);
    std::vector<uint8_t> sfa(M * 4), sfb(N * 4);
    for (auto& x : w) x = rand() & 255;
    for (auto& x : sfa) x = 124 + rand() % 7;
    for (auto& x : sfb) x = 124 + rand() % 7;
    for (int l = 0; l < 32; ++l)
      for (int j = 0; j < 4; ++j) {
        const int r = 32 * j + l;
        uint32_t word = 0;
        for (int t = 0; t < 4; ++t) word |= (uint32_t)sfa[r * 4 + t] << (8 * t);
        reinterpret_cast<uint32_t*>(w.data() + 8192)[l * 4 + j] = word;
        if (r < N) {
          uint32_t wb = 0;
          for (int t = 0; t < 4; ++t) wb |= (uint32_t)sfb[r * 4 + t] << (8 * t);
          sfb_perm[l * 4 + j] = wb;
        }
      }
    for (auto& x : bb) {
      do x = rand() & 255; while ((x & 0x7f) == 0x7f);
    }
    std::vector<double> ref(M * N);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) {
          const int code = (w[m * 64 + k / 2] >> (4 * (k & 1))) & 15;
          s += e2m1(code) * std::ldexp(1.0, sfa[m * 4 + k / 32] - 127) * e4m3(bb[n * 128 + k]) *
               std::ldexp(1.0, sfb[n * 4 + k / 32] - 127);
        }
        ref[m * N + n] = s;
      }
    uint8_t *dw, *db;
    uint32_t* dsfb;
    float* dout;
    cudaMalloc(&dw, w.size());
    cudaMalloc(&db, bb.size());
    cudaMalloc(&dsfb, 512);
    cudaMalloc(&dout, (M * N + 64) * 4);
    cudaMemcpy(dw, w.data(), w.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, bb.data(), bb.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsfb, sfb_perm.data(), 512, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[3] = {128, 128, 2};
    cuuint64_t strides[2] = {64, STAGE};
    cuuint32_t box[3] = {128, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 3, dw, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("N=%d encode 16U4_ALIGN16B 3-D: %d\n", N, (int)r);
    if (r != CUDA_SUCCESS) return 1;
    const int smem = 1024 + 16384 + 256 * 128 + 1024 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int combos[][2] = {{16, 128}, {0, 128}, {128, 16}, {512, 128}};
    for (int tx = 0; tx < 2; ++tx)
    for (auto& cb : combos) {
      cudaMemset(dout, 0, (M * N + 64) * 4);
      probe<<<1, 128, smem>>>(tm, dw, db, dsfb, dout, N, 1 | (tx << 1), cb[0], cb[1]);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("N=%d lbo=%d sbo=%d: CUDA error %s\n", N, cb[0], cb[1], cudaGetErrorString(e));
        return 1;
      }
      std::vector<float> o(M * N + 64);
      cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0;
      int bad = 0;
      for (int i = 0; i < M * N; ++i) {
        const double d = std::fabs(o[i] - ref[i]);
        maxerr = std::max(maxerr, d);
        maxref = std::max(maxref, std::fabs(ref[i]));
        if (d > 1e-4 * (1 + std::fabs(ref[i]))) ++bad;
      }
      if (o[M * N + 63] == -1.f) {
        printf("N=%d tx=%s: TMA transaction count never completed\n", N, tx ? "8192" : "16384");
        break;
      }
      printf("tx=%s N=%d lbo=%d sbo=%d: max|err| %.3g (max|ref| %.3g) bad %d/%d  smem row0:", tx ? "8192" : "16384", N, cb[0], cb[1], maxerr,
             maxref, bad, M * N);
      for (int j = 0; j < 32; ++j) printf(" %02x", (int)o[M * N + j]);
      printf("  (global row0: %02x %02x %02x %02x)\n", w[0], w[1], w[2], w[3]);
    }
    cudaFree(dw);
    cudaFree(db);
    cudaFree(dsfb);
    cudaFree(dout);
  }
  return 0;
}
