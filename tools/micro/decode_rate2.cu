// Round-2 decode-recipe micro-benchmark for the 2.06 tensor-pipe GEMV.
// Data in shared memory, B fragments in registers; reports SM cycles per
// warp-byte of packed codes per SMSP (lower is better) so recipes can be
// compared with profiles/r01_micro_decode_rate.txt.
//
// Per iteration a lane decodes one 64-weight group of two rows (g, g+8 of a
// 16-row mma tile): word c (4 bytes) of each row -> 16 f16x2 units -> 4
// mma.m16n8k16, then y += sc * D (the group scale), like the real kernel.
//
// Recipes:
//   PAIR : two bytes of one row share a word W = code_a | code_b << 16 (one
//          PRMT of the two widened values); W and W >> 6 give all 8 fields
//          with 4 LOP3 (f16 magic, p-free).
//   DUP  : round-1 recipe (code | code << 16 per byte, IMAD dup).
// Knobs: MMA on/off, scale epilogue on/off, shift on ALU (SHF) or FMA (IMAD.HI).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o decode_rate2 decode_rate2.cu
#include <cstdint>
#include <cstdio>

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
__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

enum { PAIR = 0, DUP = 1, PAIR3 = 2, FPW = 3, LO32 = 4, FPW2 = 5, FPW3 = 6, FPW4 = 7 };

// widen byte t (0..3) of word w with the row plan (C, M, sel base/step)
__device__ __forceinline__ uint32_t widen(uint32_t w, uint32_t sel, uint64_t C, uint32_t M) {
  const uint32_t qb = prmt(w, 0u, sel);
  return uint32_t((uint64_t(qb) * M + C) >> 32);
}

// 16 units of one row (4 bytes): u[8]
template <int R, bool SHF_ALU>
__device__ __forceinline__ void row_units(uint32_t w, const uint32_t (&sel)[4], uint64_t C, uint32_t M,
                                          uint32_t mk, uint32_t mg, uint32_t (&u)[8]) {
  if constexpr (R == PAIR) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const uint32_t ha = widen(w, sel[2 * p], C, M), hb = widen(w, sel[2 * p + 1], C, M);
      const uint32_t W = prmt(ha, hb, 0x6521u);  // code_a | code_b << 16 (code at [8,23) of hi)
      const uint32_t W6 = SHF_ALU ? (W >> 6) : __umulhi(W, 1u << 26);
      u[4 * p + 0] = lopm(W6, mk, mg);
      u[4 * p + 1] = lopm(W, mk, mg);
      u[4 * p + 2] = lopm(W6, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
      u[4 * p + 3] = lopm(W, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
    }
  } else if constexpr (R == PAIR3) {
    // plan at byte position 3 (code at [16,31) of hi): byte 0 isolated on
    // the FMA pipe (IMAD.SHL 24), bytes 1..3 by PRMT
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const uint32_t qa = p == 0 ? (w << 24) : prmt(w, 0u, 0x2444u);
      const uint32_t qb = prmt(w, 0u, p == 0 ? 0x1444u : 0x3444u);
      const uint32_t ha = uint32_t((uint64_t(qa) * M + C) >> 32), hb = uint32_t((uint64_t(qb) * M + C) >> 32);
      const uint32_t W = prmt(ha, hb, 0x7632u);
      const uint32_t W6 = SHF_ALU ? (W >> 6) : __umulhi(W, 1u << 26);
      u[4 * p + 0] = lopm(W6, mk, mg);
      u[4 * p + 1] = lopm(W, mk, mg);
      u[4 * p + 2] = lopm(W6, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
      u[4 * p + 3] = lopm(W, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
    }
  } else if constexpr (R == FPW) {
    // float widening: code = floor(q*alpha + (beta+0.5)) via FFMA.RM, then
    // + 2^23 rounded down puts the clean code in the low mantissa bits
    const float alpha = __uint_as_float(M | 0x3f800000u), cc = __uint_as_float(uint32_t(C) | 0x40000000u);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float qa = float(prmt(w, 0u, p == 0 ? 0x4440u : 0x4442u));
      const float qb = float(prmt(w, 0u, p == 0 ? 0x4441u : 0x4443u));
      const uint32_t ca = __float_as_uint(__fadd_rd(__fmaf_rd(qa, alpha, cc), 8388608.f));
      const uint32_t cb = __float_as_uint(__fadd_rd(__fmaf_rd(qb, alpha, cc), 8388608.f));
      const uint32_t W = prmt(ca, cb, 0x5410u);
      const uint32_t W6 = SHF_ALU ? (W >> 6) : __umulhi(W, 1u << 26);
      u[4 * p + 0] = lopm(W6, mk, mg);
      u[4 * p + 1] = lopm(W, mk, mg);
      u[4 * p + 2] = lopm(W6, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
      u[4 * p + 3] = lopm(W, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
    }
  } else if constexpr (R == FPW2 || R == FPW3 || R == FPW4) {
    // FPW2: q -> magic float 2^23 + q by PRMT, minus 2^23 (FADD), FFMA.RM, FADD.RM
    // FPW3: q -> float by byte-select I2F.U8 (conversion pipe), FFMA.RM, FADD.RM
    // FPW4: bytes 1,3 by I2F.U8, bytes 0,2 by PRMT magic
    const float alpha = __uint_as_float(M | 0x3f800000u), cc = __uint_as_float(uint32_t(C) | 0x40000000u);
    uint32_t magic;
    asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(magic));
    auto qf = [&](int t) -> float {
      const bool cv = R == FPW3 || (R == FPW4 && (t & 1));
      if (cv) {
        float f;
        if (t == 0) asm("cvt.rn.f32.u8 %0, %1;" : "=f"(f) : "h"(uint16_t(w)));
        else if (t == 1) asm("{.reg .u32 r; shr.u32 r, %1, 8; cvt.rn.f32.u8 %0, r;}" : "=f"(f) : "r"(w));
        else if (t == 2) asm("{.reg .u32 r; shr.u32 r, %1, 16; cvt.rn.f32.u8 %0, r;}" : "=f"(f) : "r"(w));
        else asm("{.reg .u32 r; shr.u32 r, %1, 24; cvt.rn.f32.u8 %0, r;}" : "=f"(f) : "r"(w));
        return f;
      }
      return __fadd_rn(__uint_as_float(prmt(w, magic, 0x7440u | uint32_t(t))), -8388608.f);
    };
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float qa = qf(2 * p), qb = qf(2 * p + 1);
      const uint32_t ca = __float_as_uint(__fadd_rd(__fmaf_rd(qa, alpha, cc), 8388608.f));
      const uint32_t cb = __float_as_uint(__fadd_rd(__fmaf_rd(qb, alpha, cc), 8388608.f));
      const uint32_t W = prmt(ca, cb, 0x5410u);
      const uint32_t W6 = SHF_ALU ? (W >> 6) : __umulhi(W, 1u << 26);
      u[4 * p + 0] = lopm(W6, mk, mg);
      u[4 * p + 1] = lopm(W, mk, mg);
      u[4 * p + 2] = lopm(W6, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
      u[4 * p + 3] = lopm(W, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
    }
  } else if constexpr (R == LO32) {
    // 32-bit IMAD widening (timing only: code = (q*M + C) >> 17 in the low word)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const uint32_t qa = p == 0 ? (w & 0xFFu) : prmt(w, 0u, 0x4442u);
      const uint32_t qb = prmt(w, 0u, p == 0 ? 0x4441u : 0x4443u);
      const uint32_t va = qa * M + uint32_t(C), vb = qb * M + uint32_t(C);
      const uint32_t W = __funnelshift_r(va, vb, 17);  // timing stand-in for the pack
      const uint32_t W6 = SHF_ALU ? (W >> 6) : __umulhi(W, 1u << 26);
      u[4 * p + 0] = lopm(W6, mk, mg);
      u[4 * p + 1] = lopm(W, mk, mg);
      u[4 * p + 2] = lopm(W6, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
      u[4 * p + 3] = lopm(W, mk ^ 0x01F801F8u ^ 0x003F003Fu, mg);
    }
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t hi = widen(w, sel[t], C, M);
      const uint32_t w2 = prmt(hi, 0u, 0x2121u);
      const uint32_t w3 = SHF_ALU ? (w2 >> 6) : __umulhi(w2, 1u << 26);
      u[2 * t] = lopm(w3, 0x003F01F8u, 0x64005800u);
      u[2 * t + 1] = lopm(w2, 0x003F01F8u, 0x64005800u);
    }
  }
}

template <int R, bool MMA, bool EPI, int WARPS, int SHFMODE, int NG>
__global__ void __launch_bounds__(WARPS * 32, 1) k(float* out, unsigned long long* cyc, int iters) {
  __shared__ __align__(16) uint32_t words[64 * 16 * 4];  // 64 groups x 16 rows x 4 words
  __shared__ uint32_t nib[64 * 16];
  for (int i = threadIdx.x; i < 64 * 16 * 4; i += blockDim.x) words[i] = uint32_t(i) * 2654435761u;
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) nib[i] = uint32_t(i) * 40503u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  uint32_t sel[4];
  for (int t = 0; t < 4; ++t) sel[t] = 0x4404u | (uint32_t(t) << 4);  // byte t -> pos 1
  const uint64_t C = 0x123456789ull * (threadIdx.x + 1);
  const uint32_t M = 0x9abcdu + threadIdx.x;
  uint32_t mk, mg;
  asm volatile("mov.b32 %0, 0x003F003F;" : "=r"(mk));
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
    if constexpr (SHFMODE == 0) {
      row_units<R, true>(w0, sel, C, M, mk, mg, u0);
      row_units<R, true>(w1, sel, C, M, mk, mg, u1);
    } else if constexpr (SHFMODE == 1) {
      row_units<R, false>(w0, sel, C, M, mk, mg, u0);
      row_units<R, false>(w1, sel, C, M, mk, mg, u1);
    } else {
      row_units<R, true>(w0, sel, C, M, mk, mg, u0);
      row_units<R, false>(w1, sel, C, M, mk, mg, u1);
    }
    if constexpr (MMA) {
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t < 4; ++t) mma(d, u0[2 * t], u1[2 * t], u0[2 * t + 1], u1[2 * t + 1], b[2 * (t & 3)], b[2 * (t & 3) + 1]);
      if constexpr (EPI) {
        const uint32_t n0 = nib[grp * 16 + g], n1 = nib[grp * 16 + g + 8];
        const float s0 = float(n0 & 15u), s1 = float(n1 & 15u);
        y0 = fmaf(s0, d[0], y0);
        y1 = fmaf(s0, d[1], y1);
        y2 = fmaf(s1, d[2], y2);
        y3 = fmaf(s1, d[3], y3);
      } else {
        y0 += d[0]; y1 += d[1]; y2 += d[2]; y3 += d[3];
      }
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

template <int R, bool MMA, bool EPI, int WARPS, int SHFMODE, int NG = 1>
void run(const char* name) {
  float* o;
  unsigned long long* c;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaMalloc(&c, 148 * 8);
  const int iters = 2048 / NG;
  k<R, MMA, EPI, WARPS, SHFMODE, NG><<<148, WARPS * 32>>>(o, c, iters);
  k<R, MMA, EPI, WARPS, SHFMODE, NG><<<148, WARPS * 32>>>(o, c, iters);
  unsigned long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // per SMSP: WARPS/4 warps, each iters * 8 bytes (two rows x 4 bytes)
  printf("%-48s %6.2f cycles per warp-byte per SMSP  (%s)\n", name, double(h) / ((WARPS / 4) * double(iters) * NG * 8),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<FPW, true, true, 16, 0, 2>("FPW mma epi w16 SHF NG2");
  run<FPW2, true, true, 16, 0, 2>("FPW2 mma epi w16 SHF NG2");
  run<FPW2, true, true, 16, 2, 2>("FPW2 mma epi w16 mixed NG2");
  run<FPW3, true, true, 16, 0, 2>("FPW3 mma epi w16 SHF NG2");
  run<FPW4, true, true, 16, 0, 2>("FPW4 mma epi w16 SHF NG2");
  run<FPW4, true, true, 16, 2, 2>("FPW4 mma epi w16 mixed NG2");
  run<FPW4, true, true, 32, 0, 2>("FPW4 mma epi w32 SHF NG2");
  run<FPW2, false, false, 16, 0, 2>("FPW2 nomma w16 SHF NG2");
  run<FPW3, false, false, 16, 0, 2>("FPW3 nomma w16 SHF NG2");
  run<FPW4, false, false, 16, 0, 2>("FPW4 nomma w16 SHF NG2");
  return 0;
}
