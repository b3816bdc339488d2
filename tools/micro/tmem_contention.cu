// Does tcgen05.st traffic from other warps slow tcgen05.mma (TS form, N=64)?
// Thread 0 issues back-to-back 4-MMA K blocks; warps 4..7 (TMEM lane
// quadrants 0..3) optionally stream tcgen05.st 32x32b.x32 into other columns.
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_07145_b200/csrc/tcgen05.cuh"
using namespace ccqb;

template <bool STORES, int N>
__global__ void bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { stop = 0; mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t b = smem_addr(smem);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_f16_ts(tm, tm + 128 + k * 8, smem_desc(b + k * 32, 16, 1024, 2), idesc, (i | k) != 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
    stop = 1;
  } else if (STORES && warp >= 4 && warp < 8) {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = 0x3c003c00u + lane;
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    int n = 0;
    while (!stop) {
      tmem_st32(tm + lane_base + 256 + (n & 7) * 32, r);
      tmem_st_wait();
      ++n;
    }
    if (lane == 0) out[1 + (warp - 4)] = n;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <bool S, int N>
void run(unsigned long long* d) {
  auto k = bench<S, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 256, 100000>>>(d, 2048);
  cudaDeviceSynchronize();
  unsigned long long h[5];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("stores=%d N=%3d: %.1f cycles per 4 MMA (K block); store loops per warp %llu  %s\n", S, N, h[0] / 2048.0,
         S ? h[1] : 0ull, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  run<false, 64>(d); run<true, 64>(d); run<false, 256>(d); run<true, 256>(d);
}
