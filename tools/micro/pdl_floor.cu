// Per-launch floor of a chain of PDL kernels captured in a CUDA graph
// (148 CTAs, the GEMV launch shape): how much of a 2-15 us GEMV launch is
// fixed launch/drain cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_floor pdl_floor.cu
#include <cstdio>

__global__ void null_k(float* y, int work) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float v = threadIdx.x;
  for (int i = 0; i < work; ++i) v = v * 1.0001f + 0.5f;
  if (threadIdx.x == 0) y[blockIdx.x] = v;
}

__global__ void plain_k(float* y, int work) {
  float v = threadIdx.x;
  for (int i = 0; i < work; ++i) v = v * 1.0001f + 0.5f;
  if (threadIdx.x == 0) y[blockIdx.x] = v;
}

int main() {
  float* y;
  cudaMalloc(&y, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaFuncSetAttribute(null_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(plain_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int variant = 0; variant < 6; ++variant) {
    const bool pdl = variant % 2 == 0;
    const int threads = 512;
    const size_t smem = variant < 2 ? 0 : (variant < 4 ? 100 * 1024 : 200 * 1024);
    const int work = 0;
    const int n = 50;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl ? 1 : 0;
      if (pdl) cudaLaunchKernelEx(&cfg, null_k, y, work);
      else cudaLaunchKernelEx(&cfg, plain_k, y, work);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s smem %3zu KB: %.2f us per launch (%s)\n", pdl ? "PDL  " : "plain", smem / 1024, ms * 1000 / (10 * n),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
