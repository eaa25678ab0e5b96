// Probe (not product code): issue-to-completion cycles of back-to-back tcgen05.mma on one SM, per
// kind and N, to see what paces the MXFP4 grouped GEMM (values are garbage; only time matters).
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/probe_mma_rate.cu -o tools/probe_mma_rate.bin
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2512_15834_b200/csrc/common.cuh"

using namespace stb;

__device__ __forceinline__ void umma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                        uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void tc_cp_sf(uint32_t taddr, uint32_t saddr) {
  const uint64_t desc = (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n" ::"r"(taddr), "l"(desc));
}
__device__ __forceinline__ void umma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ bool i0_init(uint64_t* b) {
  mbar_init(&b[0], 1u << 20);  // never completes: commits only arrive
  mbar_init(&b[1], 1u << 20);
  fence_mbar_init();
  return true;
}

// kind: 0 = f16 (bf16 SS), 1 = mxf8f6f4 block-scaled (e2m1 x e4m3), 2 = f8f6f4 (e4m3 x e4m3, no scales)
__global__ void rate(long long* out, int kind, int N, int iters, int naccs) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x11111111u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint64_t ad = umma_desc_kmajor_sw128(smem_u32(sm), 1024);
    const uint64_t bd = umma_desc_kmajor_sw128(smem_u32(sm + 16384), 1024);
    uint32_t idesc;
    if (kind == 0) idesc = umma_idesc_bf16(128, N, false, false);
    else if (kind == 1) idesc = (5u << 7) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | (8u << 24);
    else idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);  // f32 accumulate, e4m3 x e4m3
    const long long t0 = clock64();
    if (naccs >= 4) {  // one MX pipeline stage: [cp SFA, cp SFB,] 4 MMAs, [2 commits]; per-MMA figure
      __shared__ uint64_t dummy[2];
      if (i0_init(dummy)) {}
      for (int i = 0; i < iters; i += 4) {
        if (naccs & 1) {
          tc_cp_sf(tmem + 480 + (i & 4), smem_u32(sm));
          tc_cp_sf(tmem + 488 + (i & 4), smem_u32(sm + 512));
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_mx(tmem, ad + 2 * kk, bd + 2 * kk, idesc | ((uint32_t)kk << 29) | ((uint32_t)kk << 4),
                  (tmem + 480) | ((uint32_t)kk << 30), (tmem + 488) | ((uint32_t)kk << 30), 1u);
        if (naccs & 2) {
          umma_commit(&dummy[0]);
          umma_commit(&dummy[1]);
        }
      }
    } else if (naccs == 3) {  // 4 MMAs per iteration, compile-time offsets, one accumulator
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kind == 0) umma_f16_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
          else if (kind == 1)
            umma_mx(tmem, ad + 2 * kk, bd + 2 * kk, idesc | ((uint32_t)kk << 29) | ((uint32_t)kk << 4),
                    (tmem + 480) | ((uint32_t)kk << 30), (tmem + 488) | ((uint32_t)kk << 30), 1u);
          else umma_f8(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
        }
      }
    } else
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (i % naccs) * N;
      const int kk = i & 3;
      if (kind == 0) umma_f16_ss(d, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
      else if (kind == 1)
        umma_mx(d, ad + 2 * kk, bd + 2 * kk, idesc | ((uint32_t)kk << 29) | ((uint32_t)kk << 4),
                (tmem + 480) | ((uint32_t)kk << 30), (tmem + 488) | ((uint32_t)kk << 30), 1u);
      else umma_f8(d, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
    }
    const long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = 1024 + 16384 + 32768;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"f16 SS", "mxf8f6f4 SS", "f8f6f4 SS"};
  for (int kind = 0; kind < 3; ++kind)
    for (int N : {32, 64, 128, 256})
      for (int naccs : {3, 5, 6, 7}) {
        if (naccs > 3 && kind != 1) continue;
        const int iters = 1024;
        rate<<<1, 128, smem>>>(d, kind, N, iters, naccs);
        long long h[2];
        if (cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost) != cudaSuccess) {
          printf("%s N=%d: error %s\n", names[kind], N, cudaGetErrorString(cudaGetLastError()));
          return 1;
        }
        printf("%-12s M=128 N=%3d mode=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor 128*N/256 = %d)\n",
               names[kind], N, naccs, (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256);
      }
  return 0;
}
