// Microbenchmark: cycles per tcgen05.mma.kind::f16 (M=128, K=16) issued back
// to back by one thread, for N in {64,128,256}, A from SMEM (SS) or TMEM (TS).
// Operand contents are irrelevant (zeros).  nvcc -arch=sm_100a -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_07145_b200/csrc/tcgen05.cuh"
using namespace ccqb;

template <int N, bool TS, int M = 128, int ND = 1>
__global__ void bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16_f32(M, N);
    const uint32_t a = smem_addr(smem), b = smem_addr(smem + 16384);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t db = smem_desc(b, 16, 1024, 2);
      const uint32_t d = tm + (i % ND) * N;
      if (TS) mma_f16_ts(d, tm + 256, db, idesc, i >= ND);
      else mma_f16(d, smem_desc(a, 128, 1024, 0), db, idesc, i > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int N, bool TS, int M = 128, int ND = 1>
void run(unsigned long long* d) {
  auto k = bench<N, TS, M, ND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 128, 100000>>>(d, 4096);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("ND=%d M=%3d N=%3d %s: %.1f cycles per MMA (ideal %d)  err=%s\n", ND, M, N, TS ? "TS" : "SS", h / 4096.0,
         M * N / 256, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<64, true>(d); run<64, true, 128, 2>(d); run<64, true, 128, 4>(d);
  run<16, true>(d); run<16, true, 128, 2>(d); run<16, true, 128, 4>(d); run<16, true, 128, 8>(d);
  run<32, true, 128, 4>(d); run<32, true, 128, 8>(d);
  run<16, false, 128, 8>(d); run<8, false, 64, 8>(d); run<16, false, 64, 8>(d);
  run<128, true, 128, 2>(d);
  return 0;
}
