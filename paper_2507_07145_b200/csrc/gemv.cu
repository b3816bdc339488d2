// Kernel (b): fused decode + GEMV on CUDA cores (small batch M).
//
// Reference: ccq::gemv / gemv_batch (kernels.cpp:124-187).  The reference
// decodes each 64-weight group to f32 and accumulates in double; here the
// group is decoded in registers straight from the packed bytes and reduced
// in f32 (tolerance parity).
//
// Streaming structure (group size 64, the BASELINE shapes):
//   * persistent CTAs (one per SM); CTA i owns the contiguous output rows
//     [i*rows/G, (i+1)*rows/G) - balanced to one row;
//   * K is cut into nch chunks of CG <= 32 groups; warp w works on chunk
//     w % nch for the row "stream" w / nch.  Lane l owns group c*CG + l for
//     the whole kernel, so its 64 activations (f32, permuted per family so
//     every FFMA2 operand pair is an aligned register pair) and the group's
//     correction term Q are loaded into REGISTERS once (M = 1): no shared
//     memory traffic for x at all.  For M > 1, x is staged in shared memory.
//   * each warp streams its rows (RPW-row tiles, interleaved across streams)
//     through its own S-stage shared-memory ring, filled by 1-D bulk copies
//     (cp.async.bulk on the TMA engine) with mbarrier completion: no
//     register cost for bytes in flight, no block barriers in the main loop;
//   * per-(row, chunk) partials are reduced with warp shuffles into shared
//     memory and summed over chunks in a fixed order at the end: y is
//     written once per (row, token) - deterministic, no atomics.
//
// Decode arithmetic (per stored word, no lookup tables):
//   each state field is masked into the top mantissa bits of 1.0f
//   (LOP3 with 0x3F800000), giving f = 1 + s * 2^-c exactly; accumulating
//   f * x per "class" c and subtracting the row-independent term
//   Q = sum (2^c + zero_point) * x afterwards yields sum (s - zp) * x.
//   The 2.06 family first widens each clustered byte with one IMAD.WIDE
//   using the exact fixed-point plan built at upload (ccq_internal.hpp).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "ccq_internal.hpp"
#include "ptx.cuh"

namespace ccqb {
namespace {

constexpr uint32_t kOne = 0x3F800000u;  // 1.0f

__device__ __forceinline__ float as_f(uint32_t u) { return __uint_as_float(u); }

// ---------------------------------------------------------------------------
// Family traits for the group-64 streaming path.
//   PB   payload bytes per group
//   XG   floats per group in the permuted shared-memory x layout
//   CHB  bytes per row per 32-group chunk
// ---------------------------------------------------------------------------
template <int FAM>
struct G64;

// 2.06: 16 clustered bytes per group (side-band nibble scale).
//   byte b -> hi = widen(q) (code at bits [8,23)); h2 = hi << 6
//   f0 = 1 + s0/64  (hi  bits 17..22)   x[4b]
//   f1 = 1 + s1/512 (hi  bits 14..19)   x[4b+1]
//   f2 = 1 + s2/64  (h2  bits 17..22)   x[4b+2]
//   f3 = 1 + s3/512 (h2  bits 14..19)   x[4b+3]
//   natural x order; accumulator pair (A: /64, B: /512).
template <>
struct G64<kF206> {
  static constexpr int PB = 16, XG = 64, ZP = 32;
  __host__ __device__ static float cls(int i) { return (i & 1) ? 512.f : 64.f; }
  __host__ __device__ static int perm(int i) { return i; }  // position of weight i in x layout
  __host__ __device__ static bool exact_tail(int) { return false; }
};

// 2.75: 21 bytes x 3 states (4-bit, shifts 4,2,0) + tail byte (state hi
// nibble, scale lo nibble).  Per 32-bit word (4 bytes, 12 weights) byte b is
// brought to bits [15,23) (<< 15 - 8b), fields land at p = 19, 17, 15:
// f = 1 + s/16, 1 + s/64, 1 + s/256.  x layout per word (12 floats):
//   [x0 x1 | x3 x4 | x6 x7 | x9 x10 | x2 x5 | x8 x11]
// Word 5 holds byte 20 (weights 60..62) and the tail byte (weight 63, done
// exactly); its x slots: [x60 x61 | x62 x63].
template <>
struct G64<kF275> {
  static constexpr int PB = 22, XG = 64, ZP = 8;
  __host__ __device__ static float cls(int i) {
    if (i == 63) return 0.f;
    const int f = i % 3;
    return f == 0 ? 16.f : (f == 1 ? 64.f : 256.f);
  }
  __host__ __device__ static int perm(int i) {
    if (i >= 60) return 60 + (i - 60);
    const int w = i / 12, j = i % 12, b = j / 3, f = j % 3;
    const int slot = f < 2 ? (2 * b + f) : (8 + b);
    return 12 * w + slot;
  }
  __host__ __device__ static bool exact_tail(int i) { return i == 63; }
};

// 2.5: 16-bit hybrid words, 7 states of 3 bits (shifts 13,11,9,6,4,2,0), 9
// full words + tail word (state bits 13..15, 13-bit scale).  Per 32-bit word
// (2 stored words, 14 weights): low word fields via (v << 7) and (v << 14),
// high word via (v >> 9) and (v >> 2); classes per slot j:
//   j: 0   1   2    3  4   5    6
//   c: 8  32  128   8  32  128  512
// x layout per 32-bit word (16 floats, 14 used):
//   [j0 j1]lo [j2 j3]lo [j4 j5]lo [j0 j1]hi [j2 j3]hi [j4 j5]hi [j6lo j6hi] [pad pad]
// Word pair 4 = stored word 8 (7 weights, 56..62) + tail (weight 63): slots
// 64..71 hold x56..x62 in the same lo pattern, and x63.
template <>
struct G64<kF25> {
  static constexpr int PB = 20, XG = 80, ZP = 4;
  __host__ __device__ static float cls(int i) {
    if (i == 63) return 0.f;
    const int j = i % 7;
    const float c[7] = {8.f, 32.f, 128.f, 8.f, 32.f, 128.f, 512.f};
    return c[j];
  }
  __host__ __device__ static int perm(int i) {
    if (i == 63) return 64 + 14;
    const int word = i / 7, j = i % 7, u = word / 2, hi = word % 2;
    int slot;
    if (j < 6) slot = (hi ? 6 : 0) + j;
    else slot = 12 + hi;
    return 16 * u + slot;
  }
  __host__ __device__ static bool exact_tail(int i) { return i == 63; }
};


// (v & MASK) | one in ONE LOP3: `one` lives in a register (a second
// immediate would make the compiler split the op in two).
template <uint32_t MASK>
__device__ __forceinline__ float fm(uint32_t v, uint32_t one) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "n"(MASK), "r"(one));
  return __uint_as_float(d);
}

#ifdef CCQ_GEMV_TRACE
}  // namespace
__device__ unsigned long long g_trace[8192 * 16];
namespace {
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot)                                                                    \
  if (lane == 0) {                                                                     \
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);              \
    if (gwid < 8192) g_trace[gwid * 16 + (slot)] = gtime();                             \
  }
#else
#define TRACE(slot)
#endif

struct GemvArgs {
  DevLayout L;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int M;                       // tokens handled by this launch (<= MT)
  int64_t x_stride, y_stride;  // elements between token rows
  int streams;                 // row streams per CTA (warps = nch * streams)
  int rows_per_cta_max;
  int x_direct;                // M = 1: lanes load their group's x from global (no smem pass)
  int tail_split;              // M = 1, 2.06: split the leftover rows' bytes across warps
  int rows_first;              // longer row streams on the low warp ids
  int x_half;                  // M = 1, 2.06, 16-bit x: stage x in shared memory as is
  // grouped experts, one token per hit expert (offsets != nullptr): the model
  // stacks E experts of rows_e rows; CTA b serves hit expert b % nhit (rows
  // split over the CTAs of that expert), reading x row offsets[e] and
  // writing y row offsets[e] (expert-major, y_stride = rows_e).
  const int32_t* offsets;
  int E;
  int64_t rows_e;
};

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t i) {
  if (dtype == CCQ_DTYPE_F32) return static_cast<const float*>(x)[i];
  const uint16_t h = static_cast<const uint16_t*>(x)[i];
  if (dtype == CCQ_DTYPE_BF16) return __uint_as_float(uint32_t(h) << 16);
  return __half2float(__ushort_as_half(h));
}

// Activations of one group, permuted: either a register copy (M = 1) or a
// pointer into shared memory.
template <int FAM, bool REG>
struct XGroup;
template <int FAM>
struct XGroup<FAM, true> {
  float4 v[G64<FAM>::XG / 4];
  __device__ __forceinline__ float4 f4(int k) const { return v[k]; }
};
template <int FAM>
struct XGroup<FAM, false> {
  const float* p;
  __device__ __forceinline__ float4 f4(int k) const {
    return *reinterpret_cast<const float4*>(p + 4 * k);
  }
};

// ---------------------------------------------------------------------------
// Group decoders: return  sum_i (s_i - zp) * x_i  for one group (unscaled),
// given the group's payload in shared memory.
// ---------------------------------------------------------------------------

// 2.06: 16 clustered bytes.
template <class X>
__device__ __forceinline__ float dot_206(const uint8_t* gp, const X& x, float q,
                                         const WidenPlan& pl, const uint32_t (&sel)[4],
                                         uint32_t one) {
  const uint4 c = lds128(gp);
  float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const uint32_t word = wi == 0 ? c.x : wi == 1 ? c.y : wi == 2 ? c.z : c.w;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t qb = prmt(word, 0u, sel[b]);
      const uint32_t hi = uint32_t((uint64_t(qb) * pl.M + pl.C) >> 32);
      // IMAD.SHL (FMA pipe) measured faster than SHF here (tools/micro/dot_rate.cu);
      // CCQ_H2_SHF builds the ALU variant for A/B runs
#ifdef CCQ_H2_SHF
      uint32_t h2;
      asm("shf.l.wrap.b32 %0, %1, %1, 6;" : "=r"(h2) : "r"(hi));  // hi < 2^23: no wrap-around bits
#else
      const uint32_t h2 = hi << 6;
#endif
      const float2 f01 = make_float2(fm<0x007E0000u>(hi, one), fm<0x000FC000u>(hi, one));
      const float2 f23 = make_float2(fm<0x007E0000u>(h2, one), fm<0x000FC000u>(h2, one));
      const float4 xx = x.f4(4 * wi + b);
      if (b & 1) {
        a1 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a1);
        a1 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a1);
      } else {
        a0 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a0);
        a0 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a0);
      }
    }
  }
  return fmaf(64.f, a0.x + a1.x, fmaf(512.f, a0.y + a1.y, -q));
}

// dot_206 over the byte pair SL (bytes 2 SL, 2 SL + 1) of the group, without
// the - q term: the split-row tail of gemv_stream, where the rows left over by
// the static row split are decoded two bytes per warp.
template <int SL, class X>
__device__ __forceinline__ float dot_206_pair(const uint8_t* gp, const X& x, const WidenPlan& pl,
                                              const uint32_t (&sel)[4], uint32_t one) {
  const uint32_t word = *reinterpret_cast<const uint32_t*>(gp + 4 * (SL / 2));
  float2 a = make_float2(0.f, 0.f);
#pragma unroll
  for (int b = 2 * (SL & 1); b < 2 * (SL & 1) + 2; ++b) {
    const uint32_t qb = prmt(word, 0u, sel[b]);
    const uint32_t hi = uint32_t((uint64_t(qb) * pl.M + pl.C) >> 32);
    const uint32_t h2 = hi << 6;
    const float2 f01 = make_float2(fm<0x007E0000u>(hi, one), fm<0x000FC000u>(hi, one));
    const float2 f23 = make_float2(fm<0x007E0000u>(h2, one), fm<0x000FC000u>(h2, one));
    const float4 xx = x.f4(4 * (SL / 2) + b);
    a = __ffma2_rn(f01, make_float2(xx.x, xx.y), a);
    a = __ffma2_rn(f23, make_float2(xx.z, xx.w), a);
  }
  return fmaf(64.f, a.x, 512.f * a.y);
}

// 2.06 with the widening on the FP64 pipe (plan64, model.cu build_plan64):
// per byte one PRMT builds the high word of v = 1 + q 2^-12, fma.rm gives
// t = floor-exact q alpha + beta + 1/2, and two add.rm with 2^44 / 2^38 leave
// the code at bits [8,23) / [14,29) of the low word - the same `hi` /
// `hi << 6` as the IMAD.WIDE plan, with the FMA pipe (the binding one for
// this recipe, profiles/r02_micro_*) left to the FFMA2s.
template <class X>
__device__ __forceinline__ float dot_206_w64(const uint8_t* gp, const X& x, float q, double A, double B,
                                             uint32_t one) {
  const uint4 c = lds128(gp);
  double m44, m38;
  asm("mov.b64 %0, 0x42B0000000000000;" : "=d"(m44));  // 2^44
  asm("mov.b64 %0, 0x4250000000000000;" : "=d"(m38));  // 2^38
  float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const uint32_t word = wi == 0 ? c.x : wi == 1 ? c.y : wi == 2 ? c.z : c.w;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t hw = prmt(word, 0x3FF00000u, 0x7604u | (uint32_t(b) << 4));
      const double v = __hiloint2double(int(hw), 0);
      double t, d1, d2;
      asm("fma.rm.f64 %0, %1, %2, %3;" : "=d"(t) : "d"(v), "d"(A), "d"(B));
      asm("add.rm.f64 %0, %1, %2;" : "=d"(d1) : "d"(t), "d"(m44));
      asm("add.rm.f64 %0, %1, %2;" : "=d"(d2) : "d"(t), "d"(m38));
      const uint32_t hi = uint32_t(__double2loint(d1)), h2 = uint32_t(__double2loint(d2));
      const float2 f01 = make_float2(fm<0x007E0000u>(hi, one), fm<0x000FC000u>(hi, one));
      const float2 f23 = make_float2(fm<0x007E0000u>(h2, one), fm<0x000FC000u>(h2, one));
      const float4 xx = x.f4(4 * wi + b);
      if (b & 1) {
        a1 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a1);
        a1 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a1);
      } else {
        a0 = __ffma2_rn(f01, make_float2(xx.x, xx.y), a0);
        a0 = __ffma2_rn(f23, make_float2(xx.z, xx.w), a0);
      }
    }
  }
  return fmaf(64.f, a0.x + a1.x, fmaf(512.f, a0.y + a1.y, -q));
}

// 2.75: 22 bytes (21 full bytes of 3 states + tail byte: state | scale).
// Returns the dot and the embedded scale code via *sc.
template <class X>
__device__ __forceinline__ float dot_275(const uint8_t* gp, const X& x, float q, uint32_t one,
                                         float* sc) {
  // align by pointer arithmetic (an integer round trip would lose the
  // shared-memory address space and turn these into generic loads)
  const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(gp) & 3u);
  const uint32_t* a4 = reinterpret_cast<const uint32_t*>(gp - mis);
  const uint32_t sh = mis * 8u;  // 0 or 16
  uint32_t w[6];
  {
    uint32_t raw[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) raw[i] = a4[i];
#pragma unroll
    for (int i = 0; i < 6; ++i) w[i] = __funnelshift_r(raw[i], raw[i + 1], sh);
  }
  float2 p1 = make_float2(0.f, 0.f), p1b = make_float2(0.f, 0.f), p2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int wi = 0; wi < 5; ++wi) {
    const uint32_t v = w[wi];
    const uint32_t u[4] = {v << 15, v << 7, v >> 1, v >> 9};
    const float4 x0 = x.f4(3 * wi), x1 = x.f4(3 * wi + 1), x2 = x.f4(3 * wi + 2);
    p1 = __ffma2_rn(make_float2(fm<0x00780000u>(u[0], one), fm<0x001E0000u>(u[0], one)), make_float2(x0.x, x0.y), p1);
    p1b = __ffma2_rn(make_float2(fm<0x00780000u>(u[1], one), fm<0x001E0000u>(u[1], one)), make_float2(x0.z, x0.w), p1b);
    p1 = __ffma2_rn(make_float2(fm<0x00780000u>(u[2], one), fm<0x001E0000u>(u[2], one)), make_float2(x1.x, x1.y), p1);
    p1b = __ffma2_rn(make_float2(fm<0x00780000u>(u[3], one), fm<0x001E0000u>(u[3], one)), make_float2(x1.z, x1.w), p1b);
    p2 = __ffma2_rn(make_float2(fm<0x00078000u>(u[0], one), fm<0x00078000u>(u[1], one)), make_float2(x2.x, x2.y), p2);
    p2 = __ffma2_rn(make_float2(fm<0x00078000u>(u[2], one), fm<0x00078000u>(u[3], one)), make_float2(x2.z, x2.w), p2);
  }
  // word 5: byte 20 (weights 60..62) and the tail byte 21
  const uint32_t v = w[5];
  const uint32_t u0 = v << 15;
  const float4 xt = x.f4(15);
  p1 = __ffma2_rn(make_float2(fm<0x00780000u>(u0, one), fm<0x001E0000u>(u0, one)), make_float2(xt.x, xt.y), p1);
  const float c256 = fmaf(fm<0x00078000u>(u0, one), xt.z, p2.x + p2.y);
  float dot = fmaf(16.f, p1.x + p1b.x, fmaf(64.f, p1.y + p1b.y, fmaf(256.f, c256, -q)));
  dot = fmaf(float(int((v >> 12) & 0xF) - 8), xt.w, dot);
  *sc = float((v >> 8) & 0xF);
  return dot;
}

// 2.5: 20 bytes = 10 16-bit words (9 full + tail: state | 13-bit scale).
template <class X>
__device__ __forceinline__ float dot_25(const uint8_t* gp, const X& x, float q, uint32_t one,
                                        float* sc) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(gp);
  uint32_t w[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) w[i] = p[i];
  float2 pa = make_float2(0.f, 0.f), pb = pa, pc = pa, pd = pa;
  float dot = 0.f;
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const uint32_t v = w[u];
    const uint32_t a7 = v << 7, a14 = v << 14, b9 = v >> 9, b2 = v >> 2;
    const float4 x0 = x.f4(4 * u), x1 = x.f4(4 * u + 1), x2 = x.f4(4 * u + 2), x3 = x.f4(4 * u + 3);
    pa = __ffma2_rn(make_float2(fm<0x00700000u>(a7, one), fm<0x001C0000u>(a7, one)), make_float2(x0.x, x0.y), pa);
    pb = __ffma2_rn(make_float2(fm<0x00070000u>(a7, one), fm<0x00700000u>(a14, one)), make_float2(x0.z, x0.w), pb);
    pc = __ffma2_rn(make_float2(fm<0x001C0000u>(a14, one), fm<0x00070000u>(a14, one)), make_float2(x1.x, x1.y), pc);
    if (u < 4) {
      pa = __ffma2_rn(make_float2(fm<0x00700000u>(b9, one), fm<0x001C0000u>(b9, one)), make_float2(x1.z, x1.w), pa);
      pb = __ffma2_rn(make_float2(fm<0x00070000u>(b9, one), fm<0x00700000u>(b2, one)), make_float2(x2.x, x2.y), pb);
      pc = __ffma2_rn(make_float2(fm<0x001C0000u>(b2, one), fm<0x00070000u>(b2, one)), make_float2(x2.z, x2.w), pc);
      pd = __ffma2_rn(make_float2(fm<0x0001C000u>(a14, one), fm<0x0001C000u>(b2, one)), make_float2(x3.x, x3.y), pd);
    } else {
      const float d6 = fmaf(fm<0x0001C000u>(a14, one), x3.x, pd.x + pd.y);
      dot = fmaf(8.f, pa.x + pb.y, fmaf(32.f, pa.y + pc.x, fmaf(128.f, pb.x + pc.y, fmaf(512.f, d6, -q))));
      dot = fmaf(float(int(v >> 29) - 4), x3.z, dot);
      *sc = float((v >> 16) & 0x1FFFu);
    }
  }
  return dot;
}

// ---------------------------------------------------------------------------
// Warp-level reduction of N values per lane (N a power of two <= 32): after
// the call, lane l holds the warp total of value (l >> (5 - log2 N)).
// N - 1 + 5 - log2(N) shuffles instead of 5N.
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ float reduce_multi(float (&v)[N], int lane) {
  float cur[N];
#pragma unroll
  for (int i = 0; i < N; ++i) cur[i] = v[i];
  int n = N;
  int off = 16;
#pragma unroll
  for (int k = 0; (1 << k) < N; ++k) {
    const int half = n / 2;
    const bool up = lane & off;
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      if (j < half) {
        const float send = up ? cur[j] : cur[j + half];
        const float keep = up ? cur[j + half] : cur[j];
        cur[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    n = half;
    off >>= 1;
  }
  float t = cur[0];
#pragma unroll
  for (; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  return t;
}

template <int XDT>
__device__ __forceinline__ void load_x64(const void* x, int64_t base, float (&out)[64]) {
  constexpr int dtype = XDT;
  if constexpr (dtype == CCQ_DTYPE_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(x) + base);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float4 v = __ldg(p + i);
      out[4 * i] = v.x;
      out[4 * i + 1] = v.y;
      out[4 * i + 2] = v.z;
      out[4 * i + 3] = v.w;
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + base);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = __ldg(p + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (dtype == CCQ_DTYPE_BF16) {
          out[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
          out[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        } else {
          out[8 * i + 2 * j] = __half2float(__ushort_as_half(uint16_t(w[j] & 0xFFFF)));
          out[8 * i + 2 * j + 1] = __half2float(__ushort_as_half(uint16_t(w[j] >> 16)));
        }
      }
    }
  }
}

template <int XDT>
__device__ __forceinline__ void load_x64_smem(const uint8_t* xs, int64_t base, float (&out)[64]) {
  if constexpr (XDT == CCQ_DTYPE_F32) {
    const uint8_t* p = xs + base * 4;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint4 v = lds128(p + 16 * i);
      out[4 * i] = __uint_as_float(v.x);
      out[4 * i + 1] = __uint_as_float(v.y);
      out[4 * i + 2] = __uint_as_float(v.z);
      out[4 * i + 3] = __uint_as_float(v.w);
    }
  } else {
    const uint8_t* p = xs + base * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = lds128(p + 16 * i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (XDT == CCQ_DTYPE_BF16) {
          out[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
          out[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        } else {
          out[8 * i + 2 * j] = __half2float(__ushort_as_half(uint16_t(w[j] & 0xFFFF)));
          out[8 * i + 2 * j + 1] = __half2float(__ushort_as_half(uint16_t(w[j] >> 16)));
        }
      }
    }
  }
}

template <int FAM, int XDT>
__device__ __forceinline__ void load_group_x_reg(const void* xin, int64_t g, XGroup<FAM, true>& xg) {
  using T = G64<FAM>;
  float xr[64];
  load_x64<XDT>(xin, g * 64, xr);
#pragma unroll
  for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const int p = T::perm(i);
    float4& f = xg.v[p >> 2];
    if ((p & 3) == 0) f.x = xr[i];
    else if ((p & 3) == 1) f.y = xr[i];
    else if ((p & 3) == 2) f.z = xr[i];
    else f.w = xr[i];
  }
}

// ---------------------------------------------------------------------------
// The streaming kernel.
// Shared memory: [partials: rows_per_cta_max][nch][MT] f32
//                [x (M > 1 only): MT][gpr][XG] f32
//                [rings: warps][S][SB] | [mbarriers: warps][S]
// One stage SB = RPW * (CGB codes + 16 nibble bytes + 16 plan bytes).
// ---------------------------------------------------------------------------
template <int FAM, int RPW, int MT, int S, int XDT, bool W64 = false>
__global__ void __launch_bounds__(512, 1) gemv_stream(GemvArgs a) {
  using T = G64<FAM>;
  constexpr bool XREG = MT == 1;
  constexpr bool SIDE = FAM == kF206;
  constexpr int CGB = (32 * T::PB + 15) & ~15;
  constexpr int REC = CGB + (SIDE ? 32 : 0);  // one (chunk, row) record
  constexpr int SBR = RPW * REC;                // the tile's records
  constexpr int SB = SBR + (W64 ? RPW * 16 : 0);  // + the rows' FP64 plans
  extern __shared__ __align__(128) uint8_t smem[];
  const DevLayout& L = a.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int nch = L.nch;
  const int c = warp % nch;
  const int64_t gpr = L.gpr;
  int64_t r_begin, r_end, row_base = 0, tok = 0;
  if (a.offsets) {
    // hit experts in expert order (E <= 512): ballot compaction; the offsets
    // are written before this launch by the host or an earlier kernel
    __shared__ int hit[512];
    __shared__ int wcount[16], nhit_s;
    griddep_wait();
    for (int e0 = 0; e0 < a.E; e0 += blockDim.x) {
      const int e = e0 + threadIdx.x;
      const bool has = e < a.E && a.offsets[e + 1] > a.offsets[e];
      const unsigned bal = __ballot_sync(0xffffffffu, has);
      if (lane == 0) wcount[warp] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = e0 == 0 ? 0 : nhit_s;
        for (int w = 0; w < nwarps; ++w) { const int t = wcount[w]; wcount[w] = acc; acc += t; }
        nhit_s = acc;
      }
      __syncthreads();
      if (has) hit[wcount[warp] + __popc(bal & ((1u << lane) - 1u))] = e;
      __syncthreads();
    }
    const int nhit = nhit_s;
    const int h = int(blockIdx.x) % nhit, local = int(blockIdx.x) / nhit;
    const int cnt = (int(gridDim.x) - h + nhit - 1) / nhit;
    const int e = hit[h];
    row_base = int64_t(e) * a.rows_e;
    tok = a.offsets[e];
    r_begin = row_base + int64_t(local) * a.rows_e / cnt;
    r_end = row_base + int64_t(local + 1) * a.rows_e / cnt;
  } else {
    r_begin = int64_t(blockIdx.x) * L.rows / gridDim.x;
    r_end = int64_t(blockIdx.x + 1) * L.rows / gridDim.x;
  }
  const int nrows = int(r_end - r_begin);
  const void* xin = a.x_dtype == CCQ_DTYPE_F32
                        ? static_cast<const void*>(static_cast<const float*>(a.x) + tok * a.x_stride)
                        : static_cast<const void*>(static_cast<const uint16_t*>(a.x) + tok * a.x_stride);

  float* part = reinterpret_cast<float*>(smem);
  float* xs = part + ((a.rows_per_cta_max * nch * MT + 31) & ~31);
  const int64_t xstride = gpr * T::XG;  // floats per token (permuted, swizzled for M = 1)
  float* qs = xs + MT * xstride;         // M = 1: Q per group
  uint64_t* xbar = reinterpret_cast<uint64_t*>(qs + (XREG ? ((gpr + 31) & ~int64_t(31)) : 0) + 16);
  uint8_t* rings = reinterpret_cast<uint8_t*>(xbar + 2);
  uint8_t* ring = rings + size_t(warp) * S * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rings + size_t(nwarps) * S * SB) + warp * S;
  // split-row tail (M = 1, 2.06): the rows left over by the static split
  // (nrows % streams) land, one bulk copy per chunk, in tbuf; their bytes are
  // decoded by several warps each (tpart: per row, chunk and byte slice)
  constexpr bool TSPLIT = MT == 1 && FAM == kF206 && !W64;
  const bool tsplit = TSPLIT && a.tail_split;
  const int tmax = a.streams - 1;
  uint8_t* tbuf = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(rings + size_t(nwarps) * S * SB + size_t(nwarps) * S * 8) + 127) & ~uintptr_t(127));
  uint64_t* tbars = reinterpret_cast<uint64_t*>(tbuf + size_t(tmax) * nch * REC);
  float* tpart = reinterpret_cast<float*>(tbars + nch);
  const int base_rows = nrows / a.streams;
  const int ntail = tsplit ? nrows - base_rows * a.streams : 0;

  const int g0 = c * kChunk;
  const int ng = int(gpr - g0 < kChunk ? gpr - g0 : kChunk);
  const int g = g0 + lane;
  const bool active = lane < ng;

  TRACE(0);
#ifdef CCQ_GEMV_TRACE
  if (lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gwid < 8192) g_trace[gwid * 16 + 12] = smid;
  }
#endif
  // 1. Barriers.  Activations arrive with ONE bulk copy per CTA (not one L2
  //    read per warp - all SMs read the same few lines of x, which hot-spots
  //    L2 slices).
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  if (ntail > 0 && warp < nch && lane == 0) mbar_init(&tbars[warp], 1);
  fence_mbar_init();
  __syncthreads();

  // 2. Static, balanced split: stream j of chunk c owns the contiguous rows
  //    [w_begin, w_end) of this CTA (balanced to one row), streamed as RPW-row
  //    tiles through the warp's S-stage ring.  Weight copies are issued BEFORE
  //    the grid-dependency wait (PDL): they do not depend on the previous
  //    kernel, so they overlap its tail.
  const int stream = warp / nch;
  // rows_first: the streams that take one row more than the rest are the
  // LOW warp ids (ceil split), which the warp scheduler favours - the longer
  // streams then finish with the others instead of decoding their last row
  // alone on an otherwise idle SM sub-partition (profiles/r02_trace_gemv_tail.txt)
  const int64_t rb = a.rows_first ? a.streams - 1 : 0;
  const int64_t w_begin = tsplit ? r_begin + int64_t(stream) * base_rows : r_begin + (int64_t(stream) * nrows + rb) / a.streams;
  const int64_t w_end = tsplit ? w_begin + base_rows : r_begin + (int64_t(stream + 1) * nrows + rb) / a.streams;
  const int ntl = int((w_end - w_begin + RPW - 1) / RPW);
  const uint8_t* src = L.record(c, 0);
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int t, int s) {
    if (lane == 0 && t < ntl) {
      const int64_t r0 = w_begin + int64_t(t) * RPW;
      const uint32_t nr = uint32_t(w_end - r0 < RPW ? w_end - r0 : RPW);
      // codes (+ nibbles + plan) of nr consecutive rows: ONE bulk copy
      mbar_arrive_expect_tx(&bars[s], nr * REC + (W64 ? nr * 16 : 0));
      bulk_g2s_evict_first(ring + s * SB, src + r0 * REC, nr * REC, &bars[s], pol);
      if constexpr (W64) bulk_g2s(ring + s * SB + SBR, L.plan64 + r0, nr * 16, &bars[s]);
    }
  };
#pragma unroll
  for (int s = 0; s < S; ++s) issue(s, s);
  if (ntail > 0 && stream == 0 && lane == 0) {  // this chunk's tail rows: one copy
    mbar_arrive_expect_tx(&tbars[c], uint32_t(ntail) * REC);
    bulk_g2s_evict_first(tbuf + size_t(c) * tmax * REC, src + (r_begin + int64_t(a.streams) * base_rows) * REC,
                         uint32_t(ntail) * REC, &tbars[c], pol);
  }
  TRACE(8);
  griddep_launch_dependents();
  // the epilogue's row scale, loaded now (static data) rather than after the loop
  const bool sup_early = nrows * MT <= int(blockDim.x);
  const float sup_pre = sup_early && int(threadIdx.x) < nrows * MT ? L.super[r_begin + threadIdx.x / MT] : 0.f;
  griddep_wait();  // x (and y) belong to the previous kernel from here on
  TRACE(6);

  // 3. Activations to the permuted register layout (M = 1) or shared memory.
  XGroup<FAM, XREG> xg;
  float qv[MT];
  if constexpr (XREG) {
   if (a.x_direct) {
    // Each lane loads its own group's 64 activations (L1-cached global loads,
    // 128 B bf16 / 256 B f32) and converts them in registers: no shared-memory
    // pass and no block barrier before the loop.
    if (active && a.M > 0) {
      load_group_x_reg<FAM, XDT>(xin, g, xg);
      float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (T::exact_tail(i)) continue;
        const int p = T::perm(i);
        const float4 f = xg.v[p >> 2];
        const float xv = (p & 3) == 0 ? f.x : (p & 3) == 1 ? f.y : (p & 3) == 2 ? f.z : f.w;
        q4[i & 3] = fmaf(T::cls(i) + float(T::ZP), xv, q4[i & 3]);
      }
      qv[0] = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    } else {
#pragma unroll
      for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      qv[0] = 0.f;
    }
   } else if (XDT != CCQ_DTYPE_F32 && a.x_half) {
    // 2.06 with 16-bit activations: the CTA copies x into shared memory as
    // is (16-byte pieces, XOR-swizzled by (group & 7)), each lane loads its
    // group's 128 bytes and widens them to f32 in registers - half the shared
    // memory reads of the f32 staging below, which 8 streams per chunk repeat.
    uint16_t* xs16 = reinterpret_cast<uint16_t*>(xs);
    // x_half == 2: the group sums Q = sum (class + zero point) * x are formed
    // here, once per group (8 threads x 8 activations, butterfly over the 8),
    // instead of by every one of the nwarps / nch streams that share a chunk.
    const bool coop_q = a.x_half == 2;
    for (int base = int(threadIdx.x) & ~31; base < int(gpr) * 8; base += int(blockDim.x)) {
      const int qd = base + lane, gg = qd >> 3, ch = qd & 7;
      const bool ok = qd < int(gpr) * 8;
      float qp = 0.f;
      if (ok) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(xin) + int64_t(gg) * 64 + ch * 8));
        *reinterpret_cast<uint4*>(xs16 + gg * 64 + ((ch ^ (gg & 7)) << 3)) = v;
        if (coop_q) {
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int i = ch * 8 + j;
            if (T::exact_tail(i)) continue;
            const uint32_t h = (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xFFFFu);
            const float xv = XDT == CCQ_DTYPE_BF16 ? __uint_as_float(h << 16) : __half2float(__ushort_as_half(uint16_t(h)));
            qp = fmaf(T::cls(i) + float(T::ZP), xv, qp);
          }
        }
      }
      if (coop_q) {
        qp += __shfl_xor_sync(0xFFFFFFFFu, qp, 1);
        qp += __shfl_xor_sync(0xFFFFFFFFu, qp, 2);
        qp += __shfl_xor_sync(0xFFFFFFFFu, qp, 4);
        if (ok && ch == 0) qs[gg] = qp;
      }
    }
    TRACE(9);
    __syncthreads();
    TRACE(10);
    if (active && a.M > 0) {
      // natural order in, the family's permuted register layout out (T::perm
      // is compile-time: the placement is register renaming)
      float xr[64];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 v = lds128(xs16 + g * 64 + ((k ^ (g & 7)) << 3));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (XDT == CCQ_DTYPE_BF16) {
            xr[8 * k + 2 * j] = __uint_as_float(w[j] << 16);
            xr[8 * k + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
          } else {
            const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
            xr[8 * k + 2 * j] = h.x;
            xr[8 * k + 2 * j + 1] = h.y;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const int p = T::perm(i);
        float4& f = xg.v[p >> 2];
        if ((p & 3) == 0) f.x = xr[i];
        else if ((p & 3) == 1) f.y = xr[i];
        else if ((p & 3) == 2) f.z = xr[i];
        else f.w = xr[i];
      }
      if (coop_q) {
        qv[0] = qs[g];
      } else {
        float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          if (T::exact_tail(i)) continue;
          q4[i & 3] = fmaf(T::cls(i) + float(T::ZP), xr[i], q4[i & 3]);
        }
        qv[0] = (q4[0] + q4[1]) + (q4[2] + q4[3]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      qv[0] = 0.f;
    }
    TRACE(11);
   } else {
    // Cooperative pass straight from global memory (plain loads: they do not
    // queue behind this SM's weight bulk copies in the TMA unit): f32,
    // permuted per family, 16-byte chunks XOR-swizzled by (group & 15) so
    // the per-lane register loads below are conflict-free.
    for (int qd = threadIdx.x; qd < int(gpr) * 16; qd += blockDim.x) {
      const int gg = qd >> 4, i0 = (qd & 15) * 4;
      float v[4];
      const int64_t e0 = int64_t(gg) * 64 + i0;
      if constexpr (XDT == CCQ_DTYPE_F32) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(xin) + e0));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(xin) + e0));
        const uint32_t hw[4] = {t.x & 0xFFFFu, t.x >> 16, t.y & 0xFFFFu, t.y >> 16};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          v[i] = XDT == CCQ_DTYPE_BF16 ? __uint_as_float(hw[i] << 16) : __half2float(__ushort_as_half(uint16_t(hw[i])));
      }
      if constexpr (FAM == kF206) {  // identity permutation: one 16-byte store
        const int ch = i0 >> 2;
        *reinterpret_cast<float4*>(xs + gg * T::XG + ((ch ^ (gg & 15)) << 2)) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int p = T::perm(i0 + i), ch = p >> 2;
          const int pc = ch < 16 ? (ch ^ (gg & 15)) : ch;
          xs[gg * T::XG + pc * 4 + (p & 3)] = v[i];
        }
      }
    }
    TRACE(9);
    __syncthreads();
    TRACE(10);
    if (active && a.M > 0) {
      const float* xp = xs + int64_t(g) * T::XG;
#pragma unroll
      for (int k = 0; k < T::XG / 4; ++k) {
        const int pc = k < 16 ? (k ^ (g & 15)) : k;
        const uint4 v = lds128(xp + pc * 4);
        xg.v[k] = make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
      }
      // Q = sum_i (class_i + zero_point) * x_i, from registers (4 chains)
      float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (T::exact_tail(i)) continue;
        const int p = T::perm(i);
        const float4 f = xg.v[p >> 2];
        const float xv = (p & 3) == 0 ? f.x : (p & 3) == 1 ? f.y : (p & 3) == 2 ? f.z : f.w;
        q4[i & 3] = fmaf(T::cls(i) + float(T::ZP), xv, q4[i & 3]);
      }
      qv[0] = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    } else {
#pragma unroll
      for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      qv[0] = 0.f;
    }
    TRACE(11);
   }
  } else {
    for (int64_t e = threadIdx.x; e < int64_t(MT) * gpr * 64; e += blockDim.x) {
      const int m = int(e / (gpr * 64));
      const int64_t k = e - int64_t(m) * gpr * 64;
      const float v = m < a.M ? load_x(xin, a.x_dtype, int64_t(m) * a.x_stride + k) : 0.f;
      xs[m * xstride + (k >> 6) * T::XG + T::perm(int(k & 63))] = v;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      float q = 0.f;
      if (active) {
        const float* xq = xs + m * xstride + int64_t(g) * T::XG;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (!T::exact_tail(i)) q = fmaf(T::cls(i) + float(T::ZP), xq[T::perm(i)], q);
      }
      qv[m] = q;
    }
  }
  uint32_t one;
  asm volatile("mov.b32 %0, 0x3f800000;" : "=r"(one));
  TRACE(1);
  int ntiles_done = 0;

#pragma unroll 1
  for (int t0 = 0; t0 < ntl; t0 += S) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int t = t0 + s;
    if (t >= ntl) break;
    const int64_t r0 = w_begin + int64_t(t) * RPW;
    float acc[RPW * MT];
#pragma unroll
    for (int i = 0; i < RPW * MT; ++i) acc[i] = 0.f;
    mbar_wait(&bars[s], uint32_t((t / S) & 1));
    if (t == 0) { TRACE(2); }
    if (t == ntl - 1) { TRACE(13); }
    if (t == ntl - 2) { TRACE(15); }
    ++ntiles_done;
    const uint8_t* st = ring + s * SB;
    // rows of this tile (the last tile of a stream may be short): rows past
    // it hold a previous tile's bytes and are skipped, not decoded
    const int nr = int(w_end - r0 < RPW ? w_end - r0 : RPW);
    if (active) {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        if (r > 0 && r >= nr) break;
        const uint8_t* gp = st + r * REC + lane * T::PB;
        WidenPlan pl;
        uint32_t sel[4];
        float sc206 = 0.f;
        if constexpr (SIDE) {
          if constexpr (!W64) {
            const uint4 pv = lds128(st + r * REC + CGB + 16);
            pl.C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
            pl.M = pv.z;
            pl.sel = pv.w;
            const uint32_t base = pv.w & 0xFFFFu, step = pv.w >> 16;
            sel[0] = base;
            sel[1] = base + step;
            sel[2] = base + 2 * step;
            sel[3] = base + 3 * step;
          }
          const uint8_t nib = st[r * REC + CGB + (lane >> 1)];
          sc206 = float((nib >> (4 * (lane & 1))) & 0xF);
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          XGroup<FAM, XREG> xm = xg;
          if constexpr (!XREG) xm.p = xs + m * xstride + int64_t(g) * T::XG;
          float sc, dot;
          if constexpr (FAM == kF206 && W64) {
            const double2 p64 = *reinterpret_cast<const double2*>(st + SBR + r * 16);
            dot = dot_206_w64(gp, xm, qv[m], p64.x, p64.y, one);
            sc = sc206;
          } else if constexpr (FAM == kF206) {
            dot = dot_206(gp, xm, qv[m], pl, sel, one);
            sc = sc206;
          } else if constexpr (FAM == kF275) {
            dot = dot_275(gp, xm, qv[m], one, &sc);
          } else {
            dot = dot_25(gp, xm, qv[m], one, &sc);
          }
          acc[r * MT + m] = sc * dot;
        }
      }
    }
    if (t + S < ntl) {  // refill this stage with tile t + S
      __syncwarp();
      fence_proxy_async_smem();
      issue(t + S, s);
    }

    // Chunk partial of each (row, token): one multi-value warp reduction.
    const float v = reduce_multi<RPW * MT>(acc, lane);
    constexpr int SPAN = 32 / (RPW * MT);
    if ((lane & (SPAN - 1)) == 0) {
      const int idx = lane / SPAN;
      const int r = idx / MT, m = idx % MT;
      if (r0 + r < w_end) part[(int(r0 + r - r_begin) * nch + c) * MT + m] = v;
    }
    if (t == ntl - 1) { TRACE(14); }
  }
  }
  if constexpr (TSPLIT) {
    // (tail row, byte pair) items, 8 per row, dealt round-robin to the streams
    // of this chunk
    if (ntail > 0 && stream < ntail * 8) mbar_wait(&tbars[c], 0u);
    for (int it = stream; it < ntail * 8; it += a.streams) {
      const int tr = it >> 3, sl = it & 7;
      const uint8_t* st = tbuf + (size_t(c) * tmax + tr) * REC;
      float v = 0.f;
      if (active) {
        WidenPlan pl;
        const uint4 pv = lds128(st + CGB + 16);
        pl.C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
        pl.M = pv.z;
        pl.sel = pv.w;
        const uint32_t base = pv.w & 0xFFFFu, step = pv.w >> 16;
        const uint32_t sel[4] = {base, base + step, base + 2 * step, base + 3 * step};
        const uint8_t* gp = st + lane * T::PB;
        float d;
        switch (sl) {
          case 0: d = dot_206_pair<0>(gp, xg, pl, sel, one) - qv[0]; break;
          case 1: d = dot_206_pair<1>(gp, xg, pl, sel, one); break;
          case 2: d = dot_206_pair<2>(gp, xg, pl, sel, one); break;
          case 3: d = dot_206_pair<3>(gp, xg, pl, sel, one); break;
          case 4: d = dot_206_pair<4>(gp, xg, pl, sel, one); break;
          case 5: d = dot_206_pair<5>(gp, xg, pl, sel, one); break;
          case 6: d = dot_206_pair<6>(gp, xg, pl, sel, one); break;
          default: d = dot_206_pair<7>(gp, xg, pl, sel, one); break;
        }
        const uint8_t nib = st[CGB + (lane >> 1)];
        v = float((nib >> (4 * (lane & 1))) & 0xF) * d;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) tpart[(tr * nch + c) * 8 + sl] = v;
    }
  }
  TRACE(3);
#ifdef CCQ_GEMV_TRACE
  if (lane == 0) {
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gwid < 8192) g_trace[gwid * 16 + 5] = ntiles_done;
  }
#endif
  __syncthreads();
  // Sum chunk partials in a fixed order; scale by the row super scale.
  for (int e = threadIdx.x; e < nrows * MT; e += blockDim.x) {
    const int rl = e / MT, m = e % MT;
    if (m >= a.M) continue;
    float v = 0.f;
    const int tr = rl - a.streams * base_rows;
    if (ntail > 0 && tr >= 0) {
      for (int cc = 0; cc < nch; ++cc)
        for (int sl = 0; sl < 8; ++sl) v += tpart[(tr * nch + cc) * 8 + sl];
    } else {
      for (int cc = 0; cc < nch; ++cc) v += part[(rl * nch + cc) * MT + m];
    }
    const int64_t row = r_begin + rl;
    v *= sup_early ? sup_pre : L.super[row];
    const int64_t yi = (tok + m) * a.y_stride + (row - row_base);
    if (a.y_dtype == CCQ_DTYPE_F32)
      static_cast<float*>(a.y)[yi] = v;
    else
      static_cast<__nv_bfloat16*>(a.y)[yi] = __float2bfloat16_rn(v);
  }
  TRACE(4);
}

// ---------------------------------------------------------------------------
// Resident-prefetch GEMV (M = 1): the latency-hiding variant for chains of
// decode GEMVs.
//
// A token's GEMV chain is x-dependent but its WEIGHTS are not, and on B200
// the 2.06 decode (not HBM) bounds the loop.  So each CTA is kept small
// (8 warps, <= ~113 KB shared memory, <= 128 registers) to let TWO CTAs share
// an SM: while layer i decodes, layer i+1's CTA is already resident (PDL),
// has bulk-copied as much of its weight slice as fits into shared memory and
// waits in griddepcontrol.wait.  The HBM stream of layer i+1 therefore
// overlaps layer i's decode; after the wait only x (L1/L2), the decode of
// shared-memory-resident records and a short fixed-order epilogue remain.
// Tiles beyond the ring capacity stream through the same ring (refilled as
// consumed).  Activations go straight from global memory to registers (no
// shared-memory staging, no block barrier before the loop).
// ---------------------------------------------------------------------------
struct ResArgs {
  DevLayout L;
  const void* x;
  void* y;
  int y_dtype;
  int streams;            // row streams per CTA (warps = nch * streams)
  int S;                  // ring stages per warp
  int rows_per_cta_max;
};

template <int FAM, int RPW, int XDT>
__global__ void __launch_bounds__(256, 2) gemv_res(ResArgs a) {
  using T = G64<FAM>;
  constexpr bool SIDE = FAM == kF206;
  constexpr int CGB = (32 * T::PB + 15) & ~15;
  constexpr int REC = CGB + (SIDE ? 32 : 0);
  constexpr int SB = RPW * REC;
  extern __shared__ __align__(128) uint8_t smem[];
  const DevLayout& L = a.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int nch = L.nch, S = a.S;
  const int c = warp % nch, stream = warp / nch;
  const int64_t r_begin = int64_t(blockIdx.x) * L.rows / gridDim.x;
  const int64_t r_end = int64_t(blockIdx.x + 1) * L.rows / gridDim.x;
  const int nrows = int(r_end - r_begin);
  const int64_t w_begin = r_begin + int64_t(stream) * nrows / a.streams;
  const int64_t w_end = r_begin + int64_t(stream + 1) * nrows / a.streams;
  const int ntl = int((w_end - w_begin + RPW - 1) / RPW);

  float* part = reinterpret_cast<float*>(smem);
  uint8_t* rings = smem + ((size_t(a.rows_per_cta_max) * nch * 4 + 127) & ~size_t(127));
  uint8_t* ring = rings + size_t(warp) * S * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rings + size_t(nwarps) * S * SB) + warp * S;

  // 1. Weights first: they do not depend on the previous kernel.
  const uint8_t* src = L.record(c, 0);
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int t, int s) {
    const int64_t r0 = w_begin + int64_t(t) * RPW;
    const uint32_t nr = uint32_t(w_end - r0 < RPW ? w_end - r0 : RPW);
    mbar_arrive_expect_tx(&bars[s], nr * REC);
    bulk_g2s_evict_first(ring + size_t(s) * SB, src + r0 * REC, nr * REC, &bars[s], pol);
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    const int pre = ntl < S ? ntl : S;
    for (int t = 0; t < pre; ++t) issue(t, t);
  }
  __syncwarp();
  griddep_launch_dependents();
  griddep_wait();  // x (and y) belong to the previous kernel until here

  // 2. This lane's group of activations -> registers; Q = sum (class + zp) x.
  const int g0 = c * kChunk;
  const int ng = int(L.gpr - g0 < kChunk ? L.gpr - g0 : kChunk);
  const bool active = lane < ng;
  XGroup<FAM, true> xg;
  float q = 0.f;
  if (active) {
    load_group_x_reg<FAM, XDT>(a.x, g0 + lane, xg);
    float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if (T::exact_tail(i)) continue;
      const int p = T::perm(i);
      const float4 f = xg.v[p >> 2];
      const float xv = (p & 3) == 0 ? f.x : (p & 3) == 1 ? f.y : (p & 3) == 2 ? f.z : f.w;
      q4[i & 3] = fmaf(T::cls(i) + float(T::ZP), xv, q4[i & 3]);
    }
    q = (q4[0] + q4[1]) + (q4[2] + q4[3]);
  } else {
#pragma unroll
    for (int k = 0; k < T::XG / 4; ++k) xg.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint32_t one;
  asm volatile("mov.b32 %0, 0x3f800000;" : "=r"(one));

  // 3. Decode the resident (and streamed) tiles.
#pragma unroll 1
  for (int t = 0; t < ntl; ++t) {
    const int s = t % S;
    const int64_t r0 = w_begin + int64_t(t) * RPW;
    float acc[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) acc[i] = 0.f;
    mbar_wait(&bars[s], uint32_t((t / S) & 1));
    const uint8_t* st = ring + size_t(s) * SB;
    const int nr = int(w_end - r0 < RPW ? w_end - r0 : RPW);
    if (active) {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        if (r > 0 && r >= nr) break;
        const uint8_t* gp = st + r * REC + lane * T::PB;
        float sc, dot;
        if constexpr (FAM == kF206) {
          const uint4 pv = lds128(st + r * REC + CGB + 16);
          WidenPlan pl;
          pl.C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
          pl.M = pv.z;
          pl.sel = pv.w;
          const uint32_t base = pv.w & 0xFFFFu, step = pv.w >> 16;
          const uint32_t sel[4] = {base, base + step, base + 2 * step, base + 3 * step};
          const uint8_t nib = st[r * REC + CGB + (lane >> 1)];
          sc = float((nib >> (4 * (lane & 1))) & 0xF);
          dot = dot_206(gp, xg, q, pl, sel, one);
        } else if constexpr (FAM == kF275) {
          dot = dot_275(gp, xg, q, one, &sc);
        } else {
          dot = dot_25(gp, xg, q, one, &sc);
        }
        acc[r] = sc * dot;
      }
    }
    if (t + S < ntl) {  // refill this stage (tiles beyond the ring capacity)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) issue(t + S, s);
    }
    const float v = reduce_multi<RPW>(acc, lane);
    constexpr int SPAN = 32 / RPW;
    if ((lane & (SPAN - 1)) == 0) {
      const int r = lane / SPAN;
      if (r0 + r < w_end) part[int(r0 + r - r_begin) * nch + c] = v;
    }
  }
  __syncthreads();
  // 4. Fixed-order sum over chunks, row super scale, one write per row.
  for (int rl = threadIdx.x; rl < nrows; rl += blockDim.x) {
    float v = 0.f;
    for (int cc = 0; cc < nch; ++cc) v += part[rl * nch + cc];
    const int64_t row = r_begin + rl;
    v *= L.super[row];
    if (a.y_dtype == CCQ_DTYPE_F32) static_cast<float*>(a.y)[row] = v;
    else static_cast<__nv_bfloat16*>(a.y)[row] = __float2bfloat16_rn(v);
  }
}

// ---------------------------------------------------------------------------
// Generic fallback for any group geometry / token count: one warp per row,
// lanes stride over groups, exact per-weight decode (kernels.cpp:60-93).
// ---------------------------------------------------------------------------
struct GenericArgs {
  DevLayout L;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int64_t M;
};

template <int FAM>
__global__ void __launch_bounds__(256) gemv_generic(GenericArgs a) {
  constexpr FamilyConst fc = family_const(FAM);
  constexpr int TM = 8;
  const int lane = threadIdx.x & 31;
  const DevLayout& L = a.L;
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= L.rows) return;
  WidenPlan pl{};
  if constexpr (fc.cluster) pl = L.plan[row];
  const float sup = L.super[row];
  for (int64_t m0 = 0; m0 < a.M; m0 += TM) {
    float acc[TM];
#pragma unroll
    for (int t = 0; t < TM; ++t) acc[t] = 0.f;
    for (int64_t gj = lane; gj < L.gpr; gj += 32) {
      const uint8_t* p = L.group(row, gj);
      auto word = [&](int w) -> uint32_t {
        const uint8_t* q = p + w * fc.word_bytes;
        return fc.word_bytes == 2 ? (uint32_t(q[0]) | (uint32_t(q[1]) << 8)) : uint32_t(q[0]);
      };
      uint32_t sc;
      if (L.geo.embedded_scale) sc = word(L.geo.full_words) & fc.scale_mask;
      else sc = L.nibble(row, gj);
      const float scale = __fmul_rn(float(sc), sup);
      int idx = 0;
      for (int w = 0; w < L.geo.words_per_group; ++w) {
        uint32_t code = word(w);
        if constexpr (fc.cluster) code = widen_hi(code, pl) >> 8;
        const int nk = w < L.geo.full_words ? fc.wpw : 1;
        for (int k = 0; k < nk; ++k, ++idx) {
          const float wv = __fmul_rn(float(int((code >> fc.shifts[k]) & fc.weight_mask) - fc.zero_point), scale);
          const int64_t col = gj * L.geo.group_size + idx;
#pragma unroll
          for (int t = 0; t < TM; ++t)
            if (m0 + t < a.M) acc[t] = fmaf(wv, load_x(a.x, a.x_dtype, (m0 + t) * L.cols + col), acc[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const float v = warp_sum(acc[t]);
      if (lane == 0 && m0 + t < a.M) {
        if (a.y_dtype == CCQ_DTYPE_F32) static_cast<float*>(a.y)[(m0 + t) * L.rows + row] = v;
        else static_cast<__nv_bfloat16*>(a.y)[(m0 + t) * L.rows + row] = __float2bfloat16_rn(v);
      }
    }
  }
}



template <int FAM, int RPW, int MT, int S, int XDT, bool W64 = false>
int launch_stream_dt(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M0, int64_t Mn,
                  void* y, int y_dtype, cudaStream_t s, const int32_t* offsets = nullptr, int E = 0,
                  int64_t rows_e = 0, int nhit = 0) {
  using T = G64<FAM>;
  constexpr int CGB = (32 * T::PB + 15) & ~15;
  constexpr int SB = RPW * (CGB + (FAM == kF206 ? 32 : 0)) + (W64 ? RPW * 16 : 0);
  if (m->rec != uint32_t(CGB + (FAM == kF206 ? 32 : 0))) return fail(CCQ_ERR_CONFIG, "unexpected device record size");
  GemvArgs a{};
  a.L = layout_of(m);
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  const size_t yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  a.x = static_cast<const uint8_t*>(x) + size_t(M0) * size_t(m->cols) * xb;
  a.y = static_cast<uint8_t*>(y) + size_t(M0) * size_t(m->rows) * yb;
  a.x_dtype = x_dtype;
  a.y_dtype = y_dtype;
  a.M = int(Mn);
  a.x_stride = m->cols;
  a.y_stride = m->rows;
  // direct per-lane x loads beat the f32 shared-memory pass on K-heavy layers,
  // but the bf16 shared-memory staging (x_half) beats both everywhere
  // (profiles/r02_gemv_xdirect.txt): direct loads are opt-in (CCQ_X_DIRECT=1)
  static const int xd = std::getenv("CCQ_X_DIRECT") ? std::atoi(std::getenv("CCQ_X_DIRECT")) : 0;
  static const int xh = std::getenv("CCQ_X_HALF") ? std::atoi(std::getenv("CCQ_X_HALF")) : 2;
  a.x_half = MT == 1 && x_dtype != CCQ_DTYPE_F32 && xh >= 1 &&
             (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && m->cols % 64 == 0 ? xh : 0;
  static const int ts = std::getenv("CCQ_GEMV_TAIL") ? std::atoi(std::getenv("CCQ_GEMV_TAIL")) : 1;
  const bool tsplit_ok = MT == 1 && FAM == kF206 && !W64 && ts == 1;
  a.tail_split = tsplit_ok;
  static const int rf = std::getenv("CCQ_GEMV_ROWS_FIRST") ? std::atoi(std::getenv("CCQ_GEMV_ROWS_FIRST")) : 1;
  a.rows_first = rf;
  a.x_direct = MT == 1 && (xd == 1 || (xd < 0 && m->nch > 2)) &&
               (reinterpret_cast<uintptr_t>(x) & (x_dtype == CCQ_DTYPE_F32 ? 15u : 15u)) == 0 && m->cols % 64 == 0;

  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  int max_smem = max_smem_optin(dev);
  max_smem -= 2304;  // static shared memory (grouped hit list)
  int64_t grid = std::min<int64_t>(sms, m->rows);
  a.rows_per_cta_max = int((m->rows + grid - 1) / grid);
  if (offsets) {  // grouped: >= 1 CTA per hit expert, tokens in place
    if (nhit < 1 || nhit > sms || E > 512) return 1;  // caller falls back
    a.offsets = offsets;
    a.E = E;
    a.rows_e = rows_e;
    a.x = x;
    a.y = y;
    a.M = 1;
    a.y_stride = rows_e;
    grid = sms;
    a.rows_per_cta_max = int((rows_e + (grid / nhit) - 1) / (grid / nhit));
  }
  const size_t xbytes = size_t(MT) * m->gpr * T::XG * 4 + (MT == 1 ? size_t((m->gpr + 31) & ~int64_t(31)) * 4 : 0);
  const size_t pbytes = size_t((a.rows_per_cta_max * m->nch * MT + 31) & ~31) * 4;
  const size_t xraw = 0;
  // As many row streams as the register file (16 warps) and shared memory allow.
  size_t smem = 0;
  int warps = 0;
  static const int max_streams = std::getenv("CCQ_GEMV_STREAMS") ? std::atoi(std::getenv("CCQ_GEMV_STREAMS")) : 0;
  const int s0 = std::max(1, 16 / m->nch);
  for (a.streams = max_streams > 0 ? std::min(max_streams, s0) : s0; a.streams >= 1; --a.streams) {
    warps = m->nch * a.streams;
    smem = pbytes + xbytes + 64 + 16 + xraw + size_t(warps) * S * SB + size_t(warps) * S * 8 + 128;
    if (tsplit_ok)  // split-row tail: records, barriers, partials (+ alignment)
      smem += 128 + size_t(a.streams - 1) * m->nch * (size_t(SB) / RPW) + size_t(m->nch) * 8 +
              size_t(a.streams - 1) * m->nch * 32;
    if (smem <= size_t(max_smem)) break;
  }
  if (a.streams < 1) return fail(CCQ_ERR_CONFIG, "shared memory budget exceeded in the streaming GEMV");
  auto kern = gemv_stream<FAM, RPW, MT, S, XDT, W64>;
  if (int st = ensure_smem(reinterpret_cast<const void*>(kern), smem)) return st;
  // Programmatic stream serialization: the prologue and the weight copies of
  // this launch overlap the tail of the previous kernel in the stream (the
  // kernel waits on griddepcontrol before touching x or y).
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(warps * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv launch");
}

// Shared memory one CTA may use so that two CTAs fit on an SM.
int half_sm_smem(int dev) {
  static int cached[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int per_sm = 0, reserved = 0;
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    if (per_sm <= 0) per_sm = 233472;
    cached[dev] = per_sm / 2 - reserved;
  }
  return cached[dev];
}

// Resident-prefetch GEMV launch (M = 1, nch <= 8).  Returns kNotApplicable when the
// shape does not suit it (the caller takes the streaming kernel).
template <int FAM, int RPW, int XDT>
int launch_res_dt(const ccq_dev_model* m, const void* x, void* y, int y_dtype, cudaStream_t s) {
  using T = G64<FAM>;
  constexpr int CGB = (32 * T::PB + 15) & ~15;
  constexpr int REC = CGB + (FAM == kF206 ? 32 : 0);
  constexpr int SB = RPW * REC;
  if (m->rec != uint32_t(REC) || m->nch > 8) return kNotApplicable;
  int dev = 0;
  cudaGetDevice(&dev);
  ResArgs a{};
  a.L = layout_of(m);
  a.x = x;
  a.y = y;
  a.y_dtype = y_dtype;
  const int64_t grid = std::min<int64_t>(num_sms(dev), m->rows);
  a.rows_per_cta_max = int((m->rows + grid - 1) / grid);
  a.streams = std::max(1, 8 / m->nch);
  const int warps = m->nch * a.streams;
  const int64_t rows_per_stream = (a.rows_per_cta_max + a.streams - 1) / a.streams;
  const int need = int((rows_per_stream + RPW - 1) / RPW);
  const size_t pbytes = (size_t(a.rows_per_cta_max) * m->nch * 4 + 127) & ~size_t(127);
  const int budget = half_sm_smem(dev);
  const int cap = int((int64_t(budget) - int64_t(pbytes) - 128) / (int64_t(warps) * (SB + 8)));
  if (cap < 2) return kNotApplicable;
  a.S = std::min(cap, std::max(need, 1));
  const size_t smem = pbytes + size_t(warps) * a.S * (SB + 8) + 128;
  auto kern = gemv_res<FAM, RPW, XDT>;
  if (int st = ensure_smem(reinterpret_cast<const void*>(kern), smem)) return st;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(warps * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv launch");
}

template <int FAM>
int launch_res(const ccq_dev_model* m, const void* x, int x_dtype, void* y, int y_dtype, cudaStream_t s) {
  static const bool off = !(std::getenv("CCQ_GEMV_RES") && std::atoi(std::getenv("CCQ_GEMV_RES")) == 1);
  if (off) return kNotApplicable;
  switch (x_dtype) {
    case CCQ_DTYPE_F32: return launch_res_dt<FAM, 4, CCQ_DTYPE_F32>(m, x, y, y_dtype, s);
    case CCQ_DTYPE_BF16: return launch_res_dt<FAM, 4, CCQ_DTYPE_BF16>(m, x, y, y_dtype, s);
    default: return launch_res_dt<FAM, 4, CCQ_DTYPE_F16>(m, x, y, y_dtype, s);
  }
}

template <int FAM, int RPW, int MT, int S>
int launch_stream(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M0, int64_t Mn,
                  void* y, int y_dtype, cudaStream_t s) {
  // measured slower in the full kernel (13.6 vs 13.0 us at 4096 -> 14336,
  // profiles/r02_gemv_w64.txt): opt-in only
  static const bool w64_on = std::getenv("CCQ_W64") && std::atoi(std::getenv("CCQ_W64")) == 1;
  if constexpr (FAM == kF206 && MT == 1) {
    if (w64_on && m->w64 && m->plan64) {
      switch (x_dtype) {
        case CCQ_DTYPE_F32: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_F32, true>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
        case CCQ_DTYPE_BF16: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_BF16, true>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
        default: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_F16, true>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
      }
    }
  }
  switch (x_dtype) {
    case CCQ_DTYPE_F32: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_F32>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
    case CCQ_DTYPE_BF16: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_BF16>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
    default: return launch_stream_dt<FAM, RPW, MT, S, CCQ_DTYPE_F16>(m, x, x_dtype, M0, Mn, y, y_dtype, s);
  }
}

template <int FAM>
int launch_fam(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
               cudaStream_t s) {
  using T = G64<FAM>;
  const int64_t xk = m->gpr * T::XG * 4;  // smem bytes per staged token
  for (int64_t m0 = 0; m0 < M;) {
    const int64_t left = M - m0;
    int st;
    if (left >= 4 && xk * 4 <= 96 * 1024) {
      st = launch_stream<FAM, 2, 4, 2>(m, x, x_dtype, m0, 4, y, y_dtype, s);
      m0 += 4;
    } else if (left >= 2 && xk * 2 <= 120 * 1024) {
      st = launch_stream<FAM, 2, 2, 2>(m, x, x_dtype, m0, 2, y, y_dtype, s);
      m0 += 2;
    } else {
      static const int rpw = std::getenv("CCQ_GEMV_RPW") ? std::atoi(std::getenv("CCQ_GEMV_RPW")) : 4;
      if (M == 1 && (st = launch_res<FAM>(m, x, x_dtype, y, y_dtype, s)) != kNotApplicable) {
        // resident-prefetch kernel took it
      } else if (rpw == 2) st = launch_stream<FAM, 2, 1, 6>(m, x, x_dtype, m0, 1, y, y_dtype, s);
      else if (rpw == 1) st = launch_stream<FAM, 1, 1, 8>(m, x, x_dtype, m0, 1, y, y_dtype, s);
      else st = launch_stream<FAM, 4, 1, 3>(m, x, x_dtype, m0, 1, y, y_dtype, s);
      m0 += 1;
    }
    if (st != CCQ_OK) return st;
  }
  return CCQ_OK;
}

template <int FAM>
int launch_generic(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                   int y_dtype, cudaStream_t s) {
  GenericArgs a{layout_of(m), x, y, x_dtype, y_dtype, M};
  gemv_generic<FAM><<<unsigned((m->rows + 7) / 8), 256, 0, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv launch");
}

}  // namespace

int max_smem_optin(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cached[device] = v > 0 ? v : 232448;
  }
  return cached[device];
}

int ensure_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  CCQ_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kern, dev}];
  if (have >= bytes) return CCQ_OK;
  CCQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  have = bytes;
  return CCQ_OK;
}

int num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v > 0 ? v : 148;
  }
  return cached[device];
}

// Dispatch (measured, profiles/r01_sweep.json): the CUDA-core streaming GEMV
// takes M = 1.
bool gemv_fast_supported(const ccq_dev_model* m, int64_t M) {
  // M = 1 only: batches go to the tensor-pipe GEMV (when their activations
  // fit one launch) or to the tcgen05 GEMM (profiles/r01_sweep.json)
  if (m->geo.group_size != 64 || m->nch > 16) return false;
  return M <= 1;
}

// Grouped experts with ONE token per hit expert on the streaming kernel
// (returns 1 when not applicable: the caller tries the next path).
int launch_grouped_stream(const ccq_dev_model* st, int E, int64_t rows_e, const int32_t* offsets_dev,
                          int nhit, const void* x, int x_dtype, void* y, int y_dtype, cudaStream_t s) {
  if (!offsets_dev || st->geo.group_size != 64 || st->nch > 16 || rows_e % 16 != 0) return 1;
  if (std::getenv("CCQ_NO_GROUPED_STREAM")) return 1;
  auto go = [&](auto fam_tag) -> int {
    constexpr int FAM = decltype(fam_tag)::value;
    switch (x_dtype) {
      case CCQ_DTYPE_F32:
        return launch_stream_dt<FAM, 4, 1, 3, CCQ_DTYPE_F32>(st, x, x_dtype, 0, 1, y, y_dtype, s, offsets_dev, E, rows_e, nhit);
      case CCQ_DTYPE_BF16:
        return launch_stream_dt<FAM, 4, 1, 3, CCQ_DTYPE_BF16>(st, x, x_dtype, 0, 1, y, y_dtype, s, offsets_dev, E, rows_e, nhit);
      default:
        return launch_stream_dt<FAM, 4, 1, 3, CCQ_DTYPE_F16>(st, x, x_dtype, 0, 1, y, y_dtype, s, offsets_dev, E, rows_e, nhit);
    }
  };
  switch (st->family) {
    case kF275: return go(std::integral_constant<int, kF275>{});
    case kF25: return go(std::integral_constant<int, kF25>{});
    default: return go(std::integral_constant<int, kF206>{});
  }
}

int launch_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                cudaStream_t s) {
  if (gemv_hmma_supported(m, M, x_dtype, x)) {
    const int st = launch_gemv_hmma(m, x, x_dtype, M, y, y_dtype, s);
    if (st != kNotApplicable) return st;
  }
  if (x_dtype != CCQ_DTYPE_F32 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && M >= mma_min_tokens() &&
      gemv_mma_supported(m, M))
    return launch_gemv_mma(m, x, x_dtype, M, y, y_dtype, s);
  // the streaming kernel reads x with 16-byte (f32) / 8-byte (bf16, f16)
  // vector loads: an unaligned view takes the scalar kernel
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
  const bool aligned = (xa & (x_dtype == CCQ_DTYPE_F32 ? 15u : 7u)) == 0;
  const bool fast = m->geo.group_size == 64 && m->nch <= 16 && aligned;
  switch (m->family) {
    case kF275:
      return fast ? launch_fam<kF275>(m, x, x_dtype, M, y, y_dtype, s)
                  : launch_generic<kF275>(m, x, x_dtype, M, y, y_dtype, s);
    case kF25:
      return fast ? launch_fam<kF25>(m, x, x_dtype, M, y, y_dtype, s)
                  : launch_generic<kF25>(m, x, x_dtype, M, y, y_dtype, s);
    default:
      return fast ? launch_fam<kF206>(m, x, x_dtype, M, y, y_dtype, s)
                  : launch_generic<kF206>(m, x, x_dtype, M, y, y_dtype, s);
  }
}

}  // namespace ccqb

#ifdef CCQ_GEMV_TRACE
extern "C" int ccq_trace_dump(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ccqb::g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif
