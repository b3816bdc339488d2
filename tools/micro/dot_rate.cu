// Throughput of 2.06 group-decode variants (16 packed bytes -> 64 weights
// dotted with 64 f32 activations held in registers), data in shared memory.
// Reports SM cycles per warp-byte per SMSP (lower is better).
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d;
}
template <uint32_t MASK>
__device__ __forceinline__ float fm(uint32_t v, uint32_t one) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "n"(MASK), "r"(one));
  return __uint_as_float(d);
}

template <int V>
__device__ __forceinline__ float dot(uint4 c, const float4 (&x)[16], uint64_t C, uint32_t M,
                                     const uint32_t (&sel)[4], uint32_t one) {
  float2 a0 = make_float2(0.f, 0.f), a1 = a0;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const uint32_t word = wi == 0 ? c.x : wi == 1 ? c.y : wi == 2 ? c.z : c.w;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t qb = prmt(word, 0u, sel[b]);
      uint32_t hi;
      if (V == 3) {  // 32-bit IMAD (lo) widening + SHF to move code to [8,23)
        uint32_t lo = qb * M + uint32_t(C);
        asm("shf.r.wrap.b32 %0, %1, %1, 9;" : "=r"(hi) : "r"(lo));
      } else {
        hi = uint32_t((uint64_t(qb) * M + C) >> 32);
      }
      uint32_t h2;
      if (V == 1) h2 = hi << 6;
      else asm("shf.l.wrap.b32 %0, %1, %1, 6;" : "=r"(h2) : "r"(hi));
      const float4 xx = x[4 * wi + b];
      if (V == 2) {
        s0 = fmaf(fm<0x007E0000u>(hi, one), xx.x, s0);
        s1 = fmaf(fm<0x000FC000u>(hi, one), xx.y, s1);
        s2 = fmaf(fm<0x007E0000u>(h2, one), xx.z, s2);
        s3 = fmaf(fm<0x000FC000u>(h2, one), xx.w, s3);
      } else {
        const float2 f01 = make_float2(fm<0x007E0000u>(hi, one), fm<0x000FC000u>(hi, one));
        const float2 f23 = make_float2(fm<0x007E0000u>(h2, one), fm<0x000FC000u>(h2, one));
        if (b & 1) {
          a1 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a1);
          a1 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a1);
        } else {
          a0 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a0);
          a0 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a0);
        }
      }
    }
  }
  if (V == 2) return 64.f * (s0 + s2) + 512.f * (s1 + s3);
  return 64.f * (a0.x + a1.x) + 512.f * (a0.y + a1.y);
}

// V5/V6: the tensor-pipe GEMV decode - f16 magic units (PRMT, IMAD.HI, dup,
// shift, 2 LOP3 per byte) consumed by mma.sync m16n8k16 (0.5 per byte).
// V5: dup via PRMT + SHF;  V6: dup via IMAD, shift alternating SHF / IMAD.HI.
__device__ __forceinline__ uint32_t lopm(uint32_t v, uint32_t m, uint32_t g) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(m), "r"(g)); return d;
}
template <int V>
__device__ __forceinline__ float dot_mma(uint4 c, uint32_t b0, uint32_t b1, uint64_t C, uint32_t M,
                                         const uint32_t (&sel)[4]) {
  float d[4] = {0.f, 0.f, 0.f, 0.f}, e[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t u[32];
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const uint32_t word = wi == 0 ? c.x : wi == 1 ? c.y : wi == 2 ? c.z : c.w;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t qb = prmt(word, 0u, sel[b]);
      uint32_t hi;
      if (V == 7) hi = qb * M + uint32_t(C);                      // 32-bit IMAD (timing only)
      else if (V == 8) hi = __umulhi(qb, M);                      // IMAD.HI, no 64-bit addend
      else if (V == 9) { hi = __umulhi(qb, M); hi += uint32_t(C >> 32); }  // IMAD.HI + IADD
      else hi = uint32_t((uint64_t(qb) * M + C) >> 32);
      uint32_t w2, w3;
      if (V == 5 || V == 7 || V == 8 || V == 9) { w2 = prmt(hi, 0u, 0x2121u); w3 = w2 >> 6; }
      else { w2 = hi * 0x00010001u; w3 = (b & 1) ? __umulhi(w2, 1u << 26) : (w2 >> 6); }
      u[8 * wi + 2 * b] = lopm(w3, 0x003F01F8u, 0x64005800u);
      u[8 * wi + 2 * b + 1] = lopm(w2, 0x003F01F8u, 0x64005800u);
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    float* acc = (t & 1) ? e : d;
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
        : "r"(u[4 * t]), "r"(u[4 * t + 1]), "r"(u[4 * t + 2]), "r"(u[4 * t + 3]), "r"(b0), "r"(b1));
  }
  return d[0] + d[1] + d[2] + d[3] + e[0] + e[1] + e[2] + e[3];
}

template <int V, int RPW>
__global__ void __launch_bounds__(512, 1) k(float* out, unsigned long long* cyc, int iters) {
  __shared__ __align__(16) uint8_t codes[16 * 32 * 16 * 4];
  for (int i = threadIdx.x; i < int(sizeof(codes)); i += blockDim.x) codes[i] = uint8_t(i * 37 + 11);
  float4 x[16];
  for (int i = 0; i < 16; ++i) x[i] = make_float4(i * 0.1f + threadIdx.x, 1.f, 2.f, 3.f);
  const uint32_t sel[4] = {0x4440u, 0x4441u, 0x4442u, 0x4443u};
  uint32_t one; asm volatile("mov.b32 %0, 0x3f800000;" : "=r"(one));
  const uint64_t C = 0x12345678ull * (threadIdx.x + 1);
  const uint32_t M = 0x9abcdefu + threadIdx.x;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc = 0.f;
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const uint4 c = *reinterpret_cast<const uint4*>(codes + (((warp * RPW + r + it) & 63) * 32 + lane) * 16);
      if constexpr (V >= 5) acc += dot_mma<V>(c, __float_as_uint(x[0].x), __float_as_uint(x[1].x), C, M, sel);
      else acc += dot<V>(c, x, C, M, sel, one);
    }
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V, int RPW>
void run(const char* name) {
  float* o; unsigned long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  const int iters = 256;
  k<V, RPW><<<148, 512>>>(o, c, iters);
  k<V, RPW><<<148, 512>>>(o, c, iters);
  unsigned long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps, each iters*RPW*16 bytes
  printf("%-36s %.2f cycles per warp-byte per SMSP  (%s)\n", name, double(h) / (4.0 * iters * RPW * 16),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0, 4>("V0 PRMT,IMAD.HI,SHF,4LOP3,2FFMA2");
  run<1, 4>("V1 IMAD.SHL instead of SHF");
  run<2, 4>("V2 4 scalar FFMA");
  run<3, 4>("V3 IMAD lo + SHF.R");
  run<5, 4>("V5 mma: PRMT dup + SHF");
  run<6, 4>("V6 mma: IMAD dup, SHF/IMAD.HI");
  run<7, 4>("V7 mma, 32-bit IMAD widen (timing)");
  run<8, 4>("V8 mma, IMAD.HI no addend (timing)");
  run<9, 4>("V9 mma, IMAD.HI + IADD (timing)");
  run<0, 1>("V0 RPW=1");
  run<0, 8>("V0 RPW=8");
  return 0;
}
