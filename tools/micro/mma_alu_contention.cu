// Does decode-style ALU/FMA work on the other warps of the SM slow the
// tcgen05 MMA issuer?  Warp 0 lane 0 issues 1024 K blocks of 4 TS-form MMAs
// (M=128, N=64, K=16), A/B either fixed or cycling through 12 slots like the
// GEMM's rings; NW other warps run a PRMT/IMAD.HI/LOP3/HFMA2 loop until the
// issuer is done.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2507_07145_b200/csrc/tcgen05.cuh"
using namespace ccqb;

template <int N>
__global__ void bench(unsigned long long* out, int iters, int cyc, int nalu) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    done = 0;
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t b = smem_addr(smem);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int sl = cyc ? i % 12 : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_f16_ts(tm, tm + 64 + sl * 32 + k * 8, smem_desc(b + sl * 8192 + k * 32, 16, 1024, 2), idesc, (i | k) != 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
    done = 1;
  } else if (warp >= 1 && warp <= nalu) {
    uint32_t x = threadIdx.x * 2654435761u, acc = 0;
    const uint32_t M = 0x9E3779B1u | threadIdx.x;
    __half2 h = __floats2half2_rn(1.f, 2.f), sc = __floats2half2_rn(0.5f, 0.25f);
    while (!done) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t q = __byte_perm(x, 0, 0x4440 + j % 4);
        const uint32_t hi = __umulhi(q, M);
        const uint32_t w2 = __byte_perm(hi, 0, 0x2121);
        const uint32_t w3 = w2 >> 6;
        uint32_t l0, l1;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(l0) : "r"(w2), "r"(0x01F8003Fu), "r"(0x64006400u));
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(l1) : "r"(w3), "r"(0x01F8003Fu), "r"(0x64006400u));
        h = __hfma2(*reinterpret_cast<__half2*>(&l0), sc, h);
        h = __hfma2(*reinterpret_cast<__half2*>(&l1), sc, h);
        x += hi;
      }
      acc ^= *reinterpret_cast<uint32_t*>(&h);
    }
    if (acc == 0x12345u) out[1] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  auto k = bench<64>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 8192 + 1024);
  for (int cyc = 0; cyc < 2; ++cyc)
    for (int nalu : {0, 4, 8, 12, 15}) {
      k<<<1, 512, 12 * 8192 + 1024>>>(d, 1024, cyc, nalu);
      cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("N=64 cycling=%d alu_warps=%2d: %.1f cycles per K block (4 MMA)  %s\n", cyc, nalu, h / 1024.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  // full-chip: 148 CTAs
  for (int nalu : {0, 12}) {
    k<<<148, 512, 12 * 8192 + 1024>>>(d, 1024, 1, nalu);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("148 CTAs cycling=1 alu_warps=%2d: %.1f cycles per K block (4 MMA)\n", nalu, h / 1024.0);
  }
}
