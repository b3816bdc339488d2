// Throughput of legacy warp-level mma.sync.m16n8k16 (f16 in, f32 accumulate)
// on sm_100a: cycles per HMMA per SMSP with 16 warps/SM and 4 independent
// accumulator chains per warp.   nvcc -gencode arch=compute_100a,code=sm_100a -o hmma_rate hmma_rate.cu
#include <cstdio>

#define ITERS 2048
__global__ void __launch_bounds__(512) k(float* out, unsigned long long* cyc, unsigned seed) {
  unsigned a0 = seed * threadIdx.x, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a0 * 3, b0 = seed, b1 = seed ^ 5;
  float d[4][4] = {};
  __syncthreads();
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  unsigned long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Latency: one warp per SM, one dependent accumulator chain.
__global__ void lat(float* out, unsigned long long* cyc, unsigned seed) {
  unsigned a0 = seed * threadIdx.x, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a0 * 3, b0 = seed, b1 = seed ^ 5;
  float d[4] = {};
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  unsigned long long t1 = clock64();
  out[blockIdx.x * 32 + threadIdx.x] = d[0] + d[1] + d[2] + d[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* o; unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  for (int rep = 0; rep < 2; ++rep) k<<<148, 512>>>(o, c, 12345);
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double per_smsp = 4.0 * ITERS * 4;  // 4 warps per SMSP x ITERS x 4 chains
  const double cyc_per = double(h[0]) / per_smsp;
  // one m16n8k16 = 2*16*8*16 = 4096 flop
  printf("HMMA m16n8k16 f16->f32: %.2f cycles per warp-mma per SMSP; %.1f TFLOP/s at 1.9 GHz x 148 SM\n",
         cyc_per, 4096.0 * 4 / cyc_per * 1.9e9 * 148 / 1e12);
  lat<<<148, 32>>>(o, c, 12345);
  lat<<<148, 32>>>(o, c, 12345);
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("HMMA m16n8k16 dependent-chain latency: %.1f cycles\n", double(h[0]) / ITERS);
  return 0;
}
