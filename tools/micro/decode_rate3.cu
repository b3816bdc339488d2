// Round-2 decode-recipe micro-benchmark: 2.06 widening on the FP64 pipe.
//
// The 2.06 decode needs clustered_code_value (coding.hpp:142-150):
// c = lround(double(q) * alpha + beta).  Round 1 widened each byte with one
// 64-bit-addend IMAD.WIDE on the FMA pipe (rt 4) and extracted fields with
// LOP3 on the ALU pipe, which bounded every recipe at ~15.6 cycles per
// warp-byte.  Here the widening moves to the FP64 pipe:
//   v  = 1 + q * 2^-12       (hi word 0x3FF0qq00 built by ONE PRMT, lo word 0)
//   t  = fma.rm(v, A, B)     A = 4096 alpha, B = beta + 0.5 - 4096 alpha (exact)
//   d  = add.rm(t, 2^52)     low word of d = floor(q alpha + beta + 0.5) = c
// (exact whenever q*alpha + beta is exact in double, which the upload checks
// by emulating these two instructions for all 256 q).
// The clean 15-bit codes of two bytes are packed W = c_a | c_b << 16 with one
// IMAD, W6 = W >> 6, and 4 LOP3 give 8 f16 "magic" fields for mma.sync.
//
// Reports SM cycles per warp-byte of packed codes per SMSP (lower is better)
// and checks the FP64 codes against the reference formula on the device.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o decode_rate3 decode_rate3.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t lopm(uint32_t v, uint32_t m, uint32_t g) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(m), "r"(g));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t umulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t shr(uint32_t a, uint32_t n) {
  uint32_t d;
  asm("shr.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(n));
  return d;
}
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// FP64 widening of byte t of word w -> clean code (low word)
__device__ __forceinline__ uint32_t widen64(uint32_t w, uint32_t sel, double A, double B, double mag) {
  const uint32_t hw = prmt(w, 0x3FF00000u, sel);
  const double v = __hiloint2double(int(hw), 0);
  double t, d;
  asm("fma.rm.f64 %0, %1, %2, %3;" : "=d"(t) : "d"(v), "d"(A), "d"(B));
  asm("add.rm.f64 %0, %1, %2;" : "=d"(d) : "d"(t), "d"(mag));
  return uint32_t(__double2loint(d));
}

enum { IMADHI = 0, FP64 = 1, FP64_ONLY = 2, IMADHI_ONLY = 3, FP64_NOSHIFT = 4 };

template <int R, int SHIFT_FMA>
__device__ __forceinline__ void row_units(uint32_t w, const uint32_t (&sel)[4], const uint32_t (&sel64)[4],
                                          uint64_t C, uint32_t M, double A, double B, double mag,
                                          uint32_t mk0, uint32_t mk3, uint32_t mg, uint32_t (&u)[8]) {
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    uint32_t W;
    if constexpr (R == IMADHI || R == IMADHI_ONLY) {
      const uint32_t qa = prmt(w, 0u, sel[2 * p]), qb = prmt(w, 0u, sel[2 * p + 1]);
      const uint32_t ha = uint32_t((uint64_t(qa) * M + C) >> 32), hb = uint32_t((uint64_t(qb) * M + C) >> 32);
      W = prmt(ha, hb, 0x6521u);  // code at [8,23) of each hi -> halves
    } else {
      const uint32_t ca = widen64(w, sel64[2 * p], A, B, mag), cb = widen64(w, sel64[2 * p + 1], A, B, mag);
      W = imad(cb, 65536u, ca);
    }
    if constexpr (R == IMADHI_ONLY || R == FP64_ONLY) {
      u[4 * p] = W;
      u[4 * p + 1] = W ^ 1u;
      u[4 * p + 2] = W ^ 2u;
      u[4 * p + 3] = W ^ 3u;
    } else {
      const uint32_t W6 = R == FP64_NOSHIFT ? W ^ 0x5555u : (SHIFT_FMA ? umulhi(W, 1u << 26) : shr(W, 6));
      u[4 * p + 0] = lopm(W, mk0, mg);   // c[0:6)  p = 0
      u[4 * p + 1] = lopm(W, mk3, mg);   // c[3:9)  p = 3
      u[4 * p + 2] = lopm(W6, mk0, mg);  // c[6:12) p = 0
      u[4 * p + 3] = lopm(W6, mk3, mg);  // c[9:15) p = 3
    }
  }
}

template <int R, int SHIFT_FMA, bool MMA, int WARPS, int NG>
__global__ void __launch_bounds__(WARPS * 32, 1) k(float* out, unsigned long long* cyc, int iters) {
  __shared__ __align__(16) uint32_t words[64 * 16 * 4];  // 64 groups x 16 rows x 4 words
  __shared__ uint32_t nib[64 * 16];
  for (int i = threadIdx.x; i < 64 * 16 * 4; i += blockDim.x) words[i] = uint32_t(i) * 2654435761u;
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) nib[i] = uint32_t(i) * 40503u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  uint32_t sel[4], sel64[4];
  for (int t = 0; t < 4; ++t) sel[t] = 0x4404u | (uint32_t(t) << 4);   // byte t -> pos 1
  for (int t = 0; t < 4; ++t) sel64[t] = 0x7640u | uint32_t(t) << 4;   // [0, q, F0, 3F]
  const uint64_t C = 0x123456789ull * (threadIdx.x + 1);
  const uint32_t M = 0x9abcdu + threadIdx.x;
  const double A = 4096.0 * (1.37 + threadIdx.x * 1e-3), B = 123.25 - A;
  double mag;
  asm volatile("mov.b64 %0, 0x4330000000000000;" : "=d"(mag));
  uint32_t mk0, mk3, mg;
  asm volatile("mov.b32 %0, 0x003F003F;" : "=r"(mk0));
  asm volatile("mov.b32 %0, 0x01F801F8;" : "=r"(mk3));
  asm volatile("mov.b32 %0, 0x64006400;" : "=r"(mg));
  uint32_t b[8];
  for (int i = 0; i < 8; ++i) b[i] = 0x3c003c00u + threadIdx.x + i;
  __syncthreads();
  float y0 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
  uint32_t sink = 0;
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      const int grp = (warp + it * NG + gi) & 63;
      const uint32_t w0 = words[(grp * 16 + g) * 4 + c];
      const uint32_t w1 = words[(grp * 16 + g + 8) * 4 + c];
      uint32_t u0[8], u1[8];
      row_units<R, SHIFT_FMA>(w0, sel, sel64, C, M, A, B, mag, mk0, mk3, mg, u0);
      row_units<R, SHIFT_FMA>(w1, sel, sel64, C, M, A, B, mag, mk0, mk3, mg, u1);
      if constexpr (MMA) {
        float d[4] = {-1.f, -1.f, -1.f, -1.f};
#pragma unroll
        for (int t = 0; t < 4; ++t)
          mma(d, u0[2 * t], u1[2 * t], u0[2 * t + 1], u1[2 * t + 1], b[2 * t], b[2 * t + 1]);
        const uint32_t n0 = nib[grp * 16 + g], n1 = nib[grp * 16 + g + 8];
        const float s0 = __uint_as_float(0x4B000000u | (n0 & 15u)) - 8388608.f;
        const float s1 = __uint_as_float(0x4B000000u | (n1 & 15u)) - 8388608.f;
        y0 = fmaf(s0, d[0], y0);
        y2 = fmaf(s1, d[2], y2);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) sink ^= u0[i] ^ (u1[i] << 1);
      }
    }
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = y0 + y1 + y2 + y3 + float(sink & 1);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int R, int SHIFT_FMA, bool MMA, int WARPS, int NG = 2>
void run(const char* name) {
  float* o;
  unsigned long long* c;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaMalloc(&c, 148 * 8);
  const int iters = 4096 / NG;
  k<R, SHIFT_FMA, MMA, WARPS, NG><<<148, WARPS * 32>>>(o, c, iters);
  k<R, SHIFT_FMA, MMA, WARPS, NG><<<148, WARPS * 32>>>(o, c, iters);
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? double(h[i]) : mx;
  // per SMSP: WARPS/4 warps, each iters * NG * 8 bytes (two rows x 4 bytes)
  printf("%-44s %6.2f cycles per warp-byte per SMSP  (%s)\n", name, mx / ((WARPS / 4) * double(iters) * NG * 8),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

// ---------------------------------------------------------------------------
// Exactness: FP64 recipe vs the reference formula for random rows of the
// reference synthetic distribution (synthetic.cpp:70-71) and small betas.
// ---------------------------------------------------------------------------
__global__ void check(const float* alpha, const float* beta, int rows, unsigned long long* bad_rows,
                      unsigned long long* bad_codes) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const double a = alpha[r], be = beta[r];
  const double A = 4096.0 * a;
  const double B = __dadd_rn(__dadd_rn(be, 0.5), -A);
  double mag;
  asm volatile("mov.b64 %0, 0x4330000000000000;" : "=d"(mag));
  int nb = 0;
  for (uint32_t q = 0; q < 256; ++q) {
    const long ref = lround(__dadd_rn(__dmul_rn(double(q), a), be));
    if (ref < 0 || ref >= 32768) continue;  // DomainError territory: never stored
    const uint32_t w = q << 16;
    const uint32_t c = widen64(w, 0x7620u, A, B, mag);  // byte 2 -> pos 1
    if (long(c) != ref) ++nb;
  }
  if (nb) {
    atomicAdd(bad_rows, 1ull);
    atomicAdd(bad_codes, (unsigned long long)nb);
  }
}

static uint64_t s_state = 88172645463325252ull;
static double urand() {
  s_state ^= s_state << 13;
  s_state ^= s_state >> 7;
  s_state ^= s_state << 17;
  return double(s_state >> 11) * 0x1.0p-53;
}

void exactness(const char* name, int mode) {
  const int rows = 1 << 20;
  float *ha = new float[rows], *hb = new float[rows];
  for (int i = 0; i < rows; ++i) {
    const float a = float(1.0 + urand() * (32767.0 / 512.0));
    ha[i] = a;
    if (mode == 0) hb[i] = float(urand() * (32767.0 - 255.0 * a));
    else if (mode == 1) hb[i] = float(urand() * 1e-3);
    else hb[i] = float(std::ldexp(urand(), -int(urand() * 40)));
  }
  float *da, *db;
  unsigned long long* dc;
  cudaMalloc(&da, rows * 4);
  cudaMalloc(&db, rows * 4);
  cudaMalloc(&dc, 16);
  cudaMemset(dc, 0, 16);
  cudaMemcpy(da, ha, rows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, rows * 4, cudaMemcpyHostToDevice);
  check<<<rows / 256, 256>>>(da, db, rows, dc, dc + 1);
  unsigned long long h[2];
  cudaMemcpy(h, dc, 16, cudaMemcpyDeviceToHost);
  printf("exactness %-30s rows %d  bad rows %llu  bad codes %llu  (%s)\n", name, rows, h[0], h[1],
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(da);
  cudaFree(db);
  cudaFree(dc);
  delete[] ha;
  delete[] hb;
}

int main() {
  exactness("synthetic beta", 0);
  exactness("beta < 1e-3", 1);
  exactness("beta 2^-40..1", 2);
  run<IMADHI, 0, true, 16>("IMAD.HI widen, SHF, mma (r01 PAIR)");
  run<FP64, 0, true, 16>("FP64 widen, SHF, mma");
  run<FP64, 1, true, 16>("FP64 widen, IMAD.HI shift, mma");
  run<FP64, 0, true, 32>("FP64 widen, SHF, mma, 32 warps");
  run<FP64, 1, true, 32>("FP64 widen, IMAD.HI shift, mma, 32 warps");
  run<FP64, 0, true, 8>("FP64 widen, SHF, mma, 8 warps");
  run<FP64, 0, true, 16, 4>("FP64 widen, SHF, mma, NG4");
  run<FP64_NOSHIFT, 0, true, 16>("FP64 widen, no shift (timing), mma");
  run<FP64, 0, false, 16>("FP64 widen + fields, no mma");
  run<FP64_ONLY, 0, false, 16>("FP64 widen + pack only");
  run<IMADHI_ONLY, 0, false, 16>("IMAD.HI widen + pack only");
  return 0;
}
