// Issue-rate micro-benchmark for the decode instruction mix (sm_100a):
// per-SMSP cycles per warp instruction for LOP3, PRMT, IMAD.HI, IMAD.SHL,
// FFMA2, HFMA2, and mixes.  16 warps/SM, 8 independent chains per thread.
#include <cstdio>
#include <cuda_fp16.h>

#define ITERS 4096
template <int OP>
__global__ void __launch_bounds__(512) k(unsigned* out, unsigned long long* cyc, unsigned seed) {
  unsigned v[8];
  float2 f[8];
  for (int i = 0; i < 8; ++i) { v[i] = seed * (threadIdx.x + i); f[i] = make_float2(v[i] * 1e-9f, 1.f); }
  const unsigned m = seed | 1, one = 0x3f800000u, m64 = seed & 64u;
  const unsigned long long c64 = (unsigned long long)seed << 20;
  __syncthreads();
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
      if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(m), "r"(one));
      if (OP == 2) { unsigned long long r = (unsigned long long)v[i] * m + c64; v[i] = unsigned(r >> 32); }
      if (OP == 3) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(m64));
      if (OP == 4) f[i] = __ffma2_rn(f[i], make_float2(1.0001f, 0.9999f), make_float2(1e-7f, 2e-7f));
      if (OP == 5) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(m), "r"(one));
      if (OP == 6) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f33800000;" : "+f"(f[i].x));
      if (OP == 7) {  // mix: 1 LOP3 + 1 FFMA2
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        f[i] = __ffma2_rn(f[i], make_float2(1.0001f, 0.9999f), make_float2(1e-7f, 2e-7f));
      }
      if (OP == 8) {  // mix: 1 LOP3 + 1 IMAD.SHL
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v[(i + 1) & 7]) : "r"(m64));
      }
      if (OP == 9) asm volatile("shf.r.wrap.b32 %0, %0, %1, 6;" : "+r"(v[i]) : "r"(m));
      if (OP == 10) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(m));
      if (OP == 11) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(m));
    }
  }
  unsigned long long t1 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i] ^ __float_as_uint(f[i].x) ^ __float_as_uint(f[i].y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_iter_instr) {
  unsigned* o; unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  k<OP><<<148, 512>>>(o, c, 12345);
  k<OP><<<148, 512>>>(o, c, 12345);
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  // 16 warps per SM = 4 per SMSP; instructions per SMSP = 4 * ITERS * 8 * per_iter
  const double instr = 4.0 * ITERS * 8 * per_iter_instr;
  printf("%-22s %.2f cycles per warp-instr per SMSP\n", name, double(h[0]) / instr);
  cudaFree(o); cudaFree(c);
}

int main() {
  run<0>("LOP3", 1); run<1>("PRMT", 1); run<2>("IMAD.HI(64b add)", 1); run<3>("IMAD.SHL", 1);
  run<4>("FFMA2", 1); run<5>("HFMA2", 1); run<6>("FFMA imm", 1); run<7>("LOP3+FFMA2", 2);
  run<8>("LOP3+IMAD.SHL", 2); run<9>("SHF", 1); run<10>("IMAD.HI", 1); run<11>("IADD", 1);
  return 0;
}
