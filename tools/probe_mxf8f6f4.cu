// Probe (not product code): tcgen05.mma kind::mxf8f6f4.block_scale with A = e2m1 weights
// (one ue8m0 scale per 32 along K, the MXFP4 checkpoint format) and B = e4m3 token rows,
// one 128 x N x 128 tile, against a host double-precision product. Settles the operand
// formats the MXFP4 grouped GEMM needs before it is written: the padded 4-bit shared-memory
// layout, the scale-factor TMEM layout and the instruction descriptor.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe_mxf8f6f4.cu -o /tmp/probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2512_15834_b200/csrc/common.cuh"

using namespace stb;

constexpr int M = 128, K = 128;

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]));
}

__device__ __forceinline__ void umma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                        uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}

// pad: 0 = data in the low 8 bytes of each 16-byte chunk, 1 = high 8 bytes, 2 = both
// sfmode: 0 = replicated (lane l of every quarter, column j = row 32 j + l), 1 = lane r, column r / 32 only
__global__ void probe(const uint8_t* acodes, const uint8_t* sfa, const uint8_t* b, const uint8_t* sfb, float* out,
                      int N, int pad, int sfmode, int idmode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;            // 128 rows x 128 B
  uint8_t* sb = sm + M * 128;  // N rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const int r = tid;  // A row
    for (int c = 0; c < 8; ++c) {
      uint2 d = *reinterpret_cast<const uint2*>(acodes + r * 64 + c * 8);
      uint4 v;
      if (pad == 0) v = make_uint4(d.x, d.y, 0u, 0u);
      else if (pad == 1) v = make_uint4(0u, 0u, d.x, d.y);
      else v = make_uint4(d.x, d.y, d.x, d.y);
      *reinterpret_cast<uint4*>(sa + r * 128 + ((c ^ (r & 7)) * 16)) = v;
    }
    for (int n = tid; n < N; n += 128)
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sb + n * 128 + ((c ^ (n & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(b + n * 128 + c * 16);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t SFA_COL = 256, SFB_COL = 272;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {
    uint32_t w[8];
    if (sfmode == 0) {
      for (int j = 0; j < 4; ++j) w[j] = *reinterpret_cast<const uint32_t*>(sfa + (32 * j + lane) * 4);
    } else {
      for (int j = 0; j < 4; ++j) w[j] = 0x7f7f7f7fu;
      w[warp] = *reinterpret_cast<const uint32_t*>(sfa + (32 * warp + lane) * 4);
    }
    tmem_st4(tmem + lane_base + SFA_COL, w);
    for (int j = 0; j < 8; ++j) w[j] = 0x7f7f7f7fu;
    for (int j = 0; j < N / 32; ++j) {
      const int n = 32 * j + lane;
      w[j] = *reinterpret_cast<const uint32_t*>(sfb + n * 4);
    }
    tmem_st4(tmem + lane_base + SFB_COL, w);
    tmem_st4(tmem + lane_base + SFB_COL + 4, w + 4);
    tmem_st_wait();
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t idesc = (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
      idesc |= 5u << 7;  // A = e2m1
      uint32_t sfa_a = tmem + SFA_COL, sfb_a = tmem + SFB_COL;
      if (idmode == 0 || idmode == 1) idesc |= ((uint32_t)kk << 29) | ((uint32_t)kk << 4);
      if (idmode == 0 || idmode == 2) sfa_a |= (uint32_t)kk << 30, sfb_a |= (uint32_t)kk << 30;
      const uint64_t ad = umma_desc_kmajor_sw128(smem_u32(sa), 1024) + 2 * kk;
      const uint64_t bd = umma_desc_kmajor_sw128(smem_u32(sb), 1024) + 2 * kk;
      umma_mx(tmem, ad, bd, idesc, sfa_a, sfb_a, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + lane_base + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
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
  srand(1234);
  for (int N : {16, 32, 64, 256}) {
    std::vector<uint8_t> ac(M * 64), sfa(M * 4), bb(N * 128), sfb(N * 4);
    for (auto& x : ac) x = rand() & 255;
    for (auto& x : sfa) x = 124 + rand() % 7;
    for (auto& x : bb) {
      do x = rand() & 255; while ((x & 0x7f) == 0x7f);
    }
    for (auto& x : sfb) x = 124 + rand() % 7;
    std::vector<double> ref(M * N);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) {
          const int code = (ac[m * 64 + k / 2] >> (4 * (k & 1))) & 15;
          s += e2m1(code) * std::ldexp(1.0, sfa[m * 4 + k / 32] - 127) * e4m3(bb[n * 128 + k]) *
               std::ldexp(1.0, sfb[n * 4 + k / 32] - 127);
        }
        ref[m * N + n] = s;
      }
    uint8_t *dac, *dsfa, *db, *dsfb;
    float* dout;
    cudaMalloc(&dac, ac.size());
    cudaMalloc(&dsfa, sfa.size());
    cudaMalloc(&db, bb.size());
    cudaMalloc(&dsfb, sfb.size());
    cudaMalloc(&dout, M * N * 4);
    cudaMemcpy(dac, ac.data(), ac.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsfa, sfa.data(), sfa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, bb.data(), bb.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsfb, sfb.data(), sfb.size(), cudaMemcpyHostToDevice);
    const int smem = 1024 + M * 128 + 256 * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int pad = 0; pad < 3; ++pad)
      for (int sfmode = 0; sfmode < 2; ++sfmode)
        for (int idmode = 0; idmode < 3; ++idmode) {
          if ((pad != 2 && (sfmode || idmode)) || (sfmode && idmode)) continue;
          cudaMemset(dout, 0, M * N * 4);
          probe<<<1, 128, smem>>>(dac, dsfa, db, dsfb, dout, N, pad, sfmode, idmode);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("N=%d pad=%d sfmode=%d idmode=%d: CUDA error %s\n", N, pad, sfmode, idmode, cudaGetErrorString(e));
            return 1;
          }
          std::vector<float> o(M * N);
          cudaMemcpy(o.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
          double maxerr = 0, maxref = 0;
          int bad = 0;
          for (int i = 0; i < M * N; ++i) {
            const double d = std::fabs(o[i] - ref[i]);
            maxerr = std::max(maxerr, d);
            maxref = std::max(maxref, std::fabs(ref[i]));
            if (d > 1e-4 * (1 + std::fabs(ref[i]))) ++bad;
          }
          printf("N=%3d pad=%d sfmode=%d idmode=%d: max|err| %.3g (max|ref| %.3g), bad %d / %d  [o0=%g ref0=%g]\n", N,
                 pad, sfmode, idmode, maxerr, maxref, bad, M * N, o[0], ref[0]);
        }
    cudaFree(dac);
    cudaFree(dsfa);
    cudaFree(db);
    cudaFree(dsfb);
    cudaFree(dout);
  }
  return 0;
}
