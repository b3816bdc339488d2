// Issue-rate micro-benchmark, round 2: the FP64 pipe and instruction mixes
// for the 2.06 decode (sm_100a).  16 warps/SM, 8 independent chains per
// thread; reports SM cycles per warp-instruction per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rate2 pipe_rate2.cu
#include <cstdio>

#define ITERS 2048
template <int OP>
__global__ void __launch_bounds__(512) k(unsigned* out, unsigned long long* cyc, unsigned seed) {
  unsigned v[8];
  double d[8];
  float f[8];
  for (int i = 0; i < 8; ++i) {
    v[i] = seed * (threadIdx.x + i);
    d[i] = 1.0 + v[i] * 1e-12;
    f[i] = v[i] * 1e-9f;
  }
  const unsigned m = seed | 1, one = 0x3f800000u;
  const double A = 1.0000001, B = 1e-9;
  unsigned b0 = seed ^ 0x3c003c00u, b1 = seed ^ 0x3c013c00u;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  __syncthreads();
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(A), "d"(B));
      if (OP == 1) asm volatile("add.rm.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(B));
      if (OP == 2) {  // DFMA + LOP3
        asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(A), "d"(B));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
      }
      if (OP == 3) {  // DFMA + LOP3 + IMAD
        asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(A), "d"(B));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[(i + 3) & 7]) : "r"(m), "r"(one));
      }
      if (OP == 4) {  // decode mix per byte: PRMT, DFMA, DADD, 2 LOP3, 0.5 IMAD, 0.5 SHF
        unsigned hw;
        asm volatile("prmt.b32 %0, %1, %2, 0x7640;" : "=r"(hw) : "r"(v[i]), "r"(one));
        double x = __hiloint2double(int(hw), 0);
        asm volatile("fma.rm.f64 %0, %1, %2, %3;" : "=d"(x) : "d"(x), "d"(A), "d"(B));
        asm volatile("add.rm.f64 %0, %0, %1;" : "+d"(x) : "d"(B));
        unsigned c = unsigned(__double2loint(x));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(c) : "r"(m), "r"(one));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(c) : "r"(m), "r"(one));
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c) : "r"(m), "r"(one));
        else asm volatile("shr.u32 %0, %0, 6;" : "+r"(c));
        v[i] ^= c;
      }
      if (OP == 5) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(A));
      if (OP == 6) {  // HMMA alone (one per 2 chains)
        if (i & 1)
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};"
              : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
              : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(b0), "r"(b1));
      }
      if (OP == 7) {  // 4 LOP3 + 1 HMMA per 2 chains
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[(i + 4) & 7]) : "r"(m), "r"(one));
        if (i & 1)
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
              "{%0,%1,%2,%3};"
              : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
              : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(b0), "r"(b1));
      }
      if (OP == 8) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
      if (OP == 9) {  // LOP3 + PRMT alternating (both ALU)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(v[(i + 4) & 7]) : "r"(m), "r"(one));
      }
      if (OP == 10) {  // F2F-free FP32 widen: FFMA.RM + FADD.RM
        asm volatile("fma.rm.f32 %0, %0, 0f3F800001, 0f33800000;" : "+f"(f[i]));
        asm volatile("add.rm.f32 %0, %0, 0f4B000000;" : "+f"(f[(i + 4) & 7]));
      }
      if (OP == 11) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
      if (OP == 12) {  // LOP3 + FFMA(3 reg)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
      }
      if (OP == 13) {  // LOP3 + DFMA + FFMA
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(m), "r"(one));
        asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(A), "d"(B));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
      }
    }
  }
  unsigned long long t1 = clock64();
  unsigned a = 0;
  for (int i = 0; i < 8; ++i) a ^= v[i] ^ unsigned(__double2loint(d[i])) ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ __float_as_uint(acc[0] + acc[1] + acc[2] + acc[3]);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, double per_iter_instr) {
  unsigned* o;
  unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4);
  cudaMalloc(&c, 148 * 8);
  k<OP><<<148, 512>>>(o, c, 12345);
  k<OP><<<148, 512>>>(o, c, 12345);
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double instr = 4.0 * ITERS * 8 * per_iter_instr;  // per SMSP
  printf("%-34s %.2f cycles per warp-instr per SMSP (%s)\n", name, double(h[0]) / instr,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<0>("DFMA", 1);
  run<1>("DADD.RM", 1);
  run<5>("DMUL", 1);
  run<2>("DFMA+LOP3", 2);
  run<3>("DFMA+LOP3+IMAD", 3);
  run<4>("decode mix (7 instr/byte)", 7);
  run<6>("HMMA 16816 (per mma)", 0.5);
  run<7>("4 LOP3 + HMMA (per LOP3)", 2);
  run<8>("LOP3", 1);
  run<9>("LOP3+PRMT", 2);
  run<10>("FFMA.RM imm + FADD.RM imm", 2);
  run<11>("FFMA 3-reg", 1);
  run<12>("LOP3 + FFMA 3-reg", 2);
  run<13>("LOP3 + DFMA + FFMA", 3);
  return 0;
}
