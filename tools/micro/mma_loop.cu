// Cost per K block of the GEMM's MMA-issuer sequence at N=64 (TS form):
//  v0: 4 MMA
//  v1: 4 MMA + commit
//  v2: mbar wait (already complete) + fence + 4 MMA + commit
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_07145_b200/csrc/tcgen05.cuh"
using namespace ccqb;

template <int V, int N = 64>
__global__ void bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cbar[16];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    mbar_arrive(&bar);  // complete phase 0 of `bar`
    const uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t b = smem_addr(smem);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (V >= 2) { mbar_wait(&bar, 0); tc_fence_after(); }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_f16_ts(tm, tm + 256 + k * 8, smem_desc(b + k * 32, 16, 1024, 2), idesc, (i | k) != 0);
      if (V >= 1) mma_commit(&cbar[i & 15]);
    }
    mma_commit(&bar);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int V, int N = 64>
void run(unsigned long long* d) {
  auto k = bench<V, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 128, 100000>>>(d, 1024);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("variant %d N=%3d: %.1f cycles per K block (4 MMA)  %s\n", V, N, h / 1024.0, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<0>(d); run<1>(d); run<2>(d);
  run<2, 16>(d); run<2, 32>(d); run<2, 128>(d); run<2, 256>(d);
  run<0, 16>(d); run<0, 32>(d); run<0, 256>(d);
}
