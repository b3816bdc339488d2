// Epilogue store-throughput probe: 148 CTAs x 384 threads, each thread
// stores 96 floats in the GEMM epilogue pattern (lane = row, 32 tokens per
// slice, token stride ld floats).  Variants: 0 plain STG (stride ld),
// 1 contiguous [slice][token][row] (stride 128 rows), 2 __stcg contiguous,
// 3 float4 stores of 4 consecutive rows per lane (row-quad layout).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384) k(float* y, long ld, int variant) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, quad = warp & 3, par = warp >> 2;
  const long row = long(blockIdx.x) * 128 + quad * 32 + lane;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = float(i + lane);
  for (int cc = par * 32; cc < 256; cc += 96) {
    if (variant == 5) continue;
    if (variant == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) y[(cc + i) * ld + row] = v[i];
    } else if (variant == 1) {
      float* p = y + long(blockIdx.x) * 256 * 128 + (quad * 32 + lane);
#pragma unroll
      for (int i = 0; i < 32; ++i) p[(cc + i) * 128] = v[i];
    } else if (variant == 2) {
      float* p = y + long(blockIdx.x) * 256 * 128 + (quad * 32 + lane);
#pragma unroll
      for (int i = 0; i < 32; ++i) __stcg(p + (cc + i) * 128, v[i]);
    } else if (variant == 4) {
      // smem staging [32 tokens][32 rows] per warp + one 4 KB bulk store
      extern __shared__ float sm[];
      float* w = sm + warp * 1024;
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i * 32 + lane] = v[i];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        float* dst = y + long(blockIdx.x) * 256 * 128 + long(cc / 32) * 4096 + quad * 1024;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(dst),
                     "r"(unsigned(__cvta_generic_to_shared(w))) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    } else {
      float4* p = reinterpret_cast<float4*>(y + long(blockIdx.x) * 256 * 128) + (quad * 32 + lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) p[(cc / 4 + i) * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
}
int main() {
  const long ld = 14336;
  float* y;
  cudaMalloc(&y, size_t(256) * ld * 4 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int variant = 0; variant < 6; ++variant) {
    for (int w = 0; w < 3; ++w) k<<<112, 384, 48 * 1024>>>(y, ld, variant);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k<<<112, 384, 48 * 1024>>>(y, ld, variant);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 20;
    printf("variant %d: %.2f us per launch, %.1f GB/s total (112 CTAs x 128 KB)\n", variant, us,
           112.0 * 128 * 1024 / us / 1e3);
  }
  return 0;
}
