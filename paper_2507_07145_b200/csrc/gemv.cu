// Kernel (b): fused decode + GEMV on CUDA cores (small batch M).
//
// Reference: ccq::gemv / gemv_batch (kernels.cpp:124-187).  The reference
// decodes each 64-weight group to f32 and accumulates in double; here the
// group is decoded in registers straight from the packed bytes and reduced
// in f32 (tolerance parity).
//
// Streaming structure (group size 64, the BASELINE shapes):
//   * persistent CTAs (one per SM), 8-16 warps each;
//   * activations x[M][K] are staged once per CTA in shared memory as f32,
//     in a per-family permuted order so every FFMA2 operand pair is a
//     naturally aligned float2, together with one correction term Q per
//     (token, group);
//   * each warp owns whole row tiles (RPW rows x all of K) and streams them
//     through its own S-stage shared-memory ring filled by 1-D bulk copies
//     (cp.async.bulk, the TMA engine) with mbarrier completion - no register
//     cost for bytes in flight and no block-wide barriers in the main loop;
//   * lane l decodes group (32c + l) of every row of the tile, so one load of
//     its 64 activations serves RPW rows;
//   * partial sums are reduced with warp shuffles; y is written once per
//     (row, token) - deterministic, no atomics.
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

struct GemvArgs {
  const uint8_t* codes;
  const uint8_t* nibbles;
  const float* super;
  const WidenPlan* plan;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int64_t rows, cols, gpr;
  uint64_t code_stride, nib_stride;
  int M;  // tokens handled by this launch (<= MT)
  int64_t x_stride, y_stride;  // elements between token rows
  int64_t tiles;
  int nchunks;
  int stages;
};

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t i) {
  if (dtype == CCQ_DTYPE_F32) return static_cast<const float*>(x)[i];
  const uint16_t h = static_cast<const uint16_t*>(x)[i];
  if (dtype == CCQ_DTYPE_BF16) return __uint_as_float(uint32_t(h) << 16);
  return __half2float(__ushort_as_half(h));
}

// ---------------------------------------------------------------------------
// Per-family group consumers.  Each returns nothing; they accumulate the
// group's  sum (s - zp) * x  (unscaled) into dot[r][m] for RPW rows.
// ---------------------------------------------------------------------------

template <int RPW, int MT>
__device__ __forceinline__ void consume_206(const uint8_t* stage, int lane, const float* xs,
                                            const float* qs, int64_t gstride_x, int64_t qstride,
                                            const WidenPlan (&pl)[RPW], const uint32_t (&sel)[RPW][4],
                                            const float (&scf)[RPW], float (&acc)[RPW][MT]) {
  constexpr int CHB = 32 * 16;
  uint4 c[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) c[r] = lds128(stage + r * (CHB + 16) + lane * 16);
  float2 a[RPW][MT];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int m = 0; m < MT; ++m) a[r][m] = make_float2(0.f, 0.f);
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    float4 xv[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        xv[m][k] = *reinterpret_cast<const float4*>(xs + m * gstride_x + wi * 16 + 4 * k);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const uint32_t word = wi == 0 ? c[r].x : wi == 1 ? c[r].y : wi == 2 ? c[r].z : c[r].w;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t q = prmt(word, 0u, sel[r][b]);
        const uint32_t hi = uint32_t((uint64_t(q) * pl[r].M + pl[r].C) >> 32);
        const uint32_t h2 = hi << 6;
        const float2 f01 = make_float2(as_f((hi & 0x007E0000u) | kOne), as_f((hi & 0x000FC000u) | kOne));
        const float2 f23 = make_float2(as_f((h2 & 0x007E0000u) | kOne), as_f((h2 & 0x000FC000u) | kOne));
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const float4 xx = xv[m][b];
          a[r][m] = __ffma2_rn(f01, make_float2(xx.x, xx.y), a[r][m]);
          a[r][m] = __ffma2_rn(f23, make_float2(xx.z, xx.w), a[r][m]);
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const float q = qs[m * qstride];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float dot = fmaf(64.f, a[r][m].x, fmaf(512.f, a[r][m].y, -q));
      acc[r][m] = fmaf(scf[r], dot, acc[r][m]);
    }
  }
}

template <int RPW, int MT>
__device__ __forceinline__ void consume_275(const uint8_t* stage, int lane, const float* xs,
                                            const float* qs, int64_t gstride_x, int64_t qstride,
                                            float (&acc)[RPW][MT]) {
  constexpr int CHB = 32 * 22;
  // 22 bytes at stage + 22*lane (2-byte aligned): load 6 aligned words and
  // realign by 0 or 2 bytes.
  uint32_t w[RPW][6];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const uint8_t* p = stage + r * (CHB + 16) + 22 * lane;
    const uint32_t* a4 = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
    const uint32_t sh = (reinterpret_cast<uintptr_t>(p) & 3u) * 8u;  // 0 or 16
    uint32_t raw[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) raw[i] = a4[i];
#pragma unroll
    for (int i = 0; i < 6; ++i) w[r][i] = __funnelshift_r(raw[i], raw[i + 1], sh);
  }
  float2 p1[RPW][MT], p2[RPW][MT];  // p1 = (c16, c64), p2 = (c256, c256')
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      p1[r][m] = make_float2(0.f, 0.f);
      p2[r][m] = make_float2(0.f, 0.f);
    }
#pragma unroll
  for (int wi = 0; wi < 5; ++wi) {
    float4 xv[MT][3];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        xv[m][k] = *reinterpret_cast<const float4*>(xs + m * gstride_x + 12 * wi + 4 * k);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const uint32_t v = w[r][wi];
      const uint32_t u0 = v << 15, u1 = v << 7, u2 = v >> 1, u3 = v >> 9;
      const uint32_t u[4] = {u0, u1, u2, u3};
      float2 f01[4];
      float f2[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        f01[b] = make_float2(as_f((u[b] & 0x00780000u) | kOne), as_f((u[b] & 0x001E0000u) | kOne));
        f2[b] = as_f((u[b] & 0x00078000u) | kOne);
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        p1[r][m] = __ffma2_rn(f01[0], make_float2(xv[m][0].x, xv[m][0].y), p1[r][m]);
        p1[r][m] = __ffma2_rn(f01[1], make_float2(xv[m][0].z, xv[m][0].w), p1[r][m]);
        p1[r][m] = __ffma2_rn(f01[2], make_float2(xv[m][1].x, xv[m][1].y), p1[r][m]);
        p1[r][m] = __ffma2_rn(f01[3], make_float2(xv[m][1].z, xv[m][1].w), p1[r][m]);
        p2[r][m] = __ffma2_rn(make_float2(f2[0], f2[1]), make_float2(xv[m][2].x, xv[m][2].y), p2[r][m]);
        p2[r][m] = __ffma2_rn(make_float2(f2[2], f2[3]), make_float2(xv[m][2].z, xv[m][2].w), p2[r][m]);
      }
    }
  }
  // Word 5: byte 20 (weights 60..62) and the tail byte 21.
  {
    float4 xv[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) xv[m] = *reinterpret_cast<const float4*>(xs + m * gstride_x + 60);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const uint32_t v = w[r][5];
      const uint32_t u0 = v << 15;
      const float2 f01 = make_float2(as_f((u0 & 0x00780000u) | kOne), as_f((u0 & 0x001E0000u) | kOne));
      const float f2 = as_f((u0 & 0x00078000u) | kOne);
      const float tail_state = float(int((v >> 12) & 0xF) - 8);
      const float sc = float((v >> 8) & 0xF);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        p1[r][m] = __ffma2_rn(f01, make_float2(xv[m].x, xv[m].y), p1[r][m]);
        const float c256 = fmaf(f2, xv[m].z, p2[r][m].x + p2[r][m].y);
        float dot = fmaf(16.f, p1[r][m].x, fmaf(64.f, p1[r][m].y, fmaf(256.f, c256, -qs[m * qstride])));
        dot = fmaf(tail_state, xv[m].w, dot);
        acc[r][m] = fmaf(sc, dot, acc[r][m]);
      }
    }
  }
}

template <int RPW, int MT>
__device__ __forceinline__ void consume_25(const uint8_t* stage, int lane, const float* xs,
                                           const float* qs, int64_t gstride_x, int64_t qstride,
                                           float (&acc)[RPW][MT]) {
  constexpr int CHB = 32 * 20;
  uint32_t w[RPW][5];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(stage + r * (CHB + 16) + 20 * lane);
#pragma unroll
    for (int i = 0; i < 5; ++i) w[r][i] = p[i];
  }
  // Accumulator pairs: pa = (j0,j1) (8,32); pb = (j2,j3) (128,8);
  //                    pc = (j4,j5) (32,128); pd = (j6lo, j6hi) (512,512)
  float2 pa[RPW][MT], pb[RPW][MT], pc[RPW][MT], pd[RPW][MT];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      pa[r][m] = pb[r][m] = pc[r][m] = pd[r][m] = make_float2(0.f, 0.f);
    }
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    float4 xv[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        xv[m][k] = *reinterpret_cast<const float4*>(xs + m * gstride_x + 16 * u + 4 * k);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const uint32_t v = w[r][u];
      // low stored word: v<<7 puts shifts 13,11,9 at 20,18,16; v<<14 puts 6,4,2,0 at 20,18,16,14
      const uint32_t a7 = v << 7, a14 = v << 14;
      // high stored word: v>>9 puts 29,27,25 at 20,18,16; v>>2 puts 22,20,18,16 at 20,18,16,14
      const uint32_t b9 = v >> 9, b2 = v >> 2;
      const float2 lo01 = make_float2(as_f((a7 & 0x00700000u) | kOne), as_f((a7 & 0x001C0000u) | kOne));
      const float2 lo23 = make_float2(as_f((a7 & 0x00070000u) | kOne), as_f((a14 & 0x00700000u) | kOne));
      const float2 lo45 = make_float2(as_f((a14 & 0x001C0000u) | kOne), as_f((a14 & 0x00070000u) | kOne));
      const float2 hi01 = make_float2(as_f((b9 & 0x00700000u) | kOne), as_f((b9 & 0x001C0000u) | kOne));
      const float2 hi23 = make_float2(as_f((b9 & 0x00070000u) | kOne), as_f((b2 & 0x00700000u) | kOne));
      const float2 hi45 = make_float2(as_f((b2 & 0x001C0000u) | kOne), as_f((b2 & 0x00070000u) | kOne));
      const float2 j6 = make_float2(as_f((a14 & 0x0001C000u) | kOne), as_f((b2 & 0x0001C000u) | kOne));
      if (u < 4) {
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          pa[r][m] = __ffma2_rn(lo01, make_float2(xv[m][0].x, xv[m][0].y), pa[r][m]);
          pb[r][m] = __ffma2_rn(lo23, make_float2(xv[m][0].z, xv[m][0].w), pb[r][m]);
          pc[r][m] = __ffma2_rn(lo45, make_float2(xv[m][1].x, xv[m][1].y), pc[r][m]);
          pa[r][m] = __ffma2_rn(hi01, make_float2(xv[m][1].z, xv[m][1].w), pa[r][m]);
          pb[r][m] = __ffma2_rn(hi23, make_float2(xv[m][2].x, xv[m][2].y), pb[r][m]);
          pc[r][m] = __ffma2_rn(hi45, make_float2(xv[m][2].z, xv[m][2].w), pc[r][m]);
          pd[r][m] = __ffma2_rn(j6, make_float2(xv[m][3].x, xv[m][3].y), pd[r][m]);
        }
      } else {
        // stored word 8 (full, low half) + tail word 9 (high half).
        const float tail_state = float(int(v >> 29) - 4);
        const float sc = float((v >> 16) & 0x1FFFu);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          pa[r][m] = __ffma2_rn(lo01, make_float2(xv[m][0].x, xv[m][0].y), pa[r][m]);
          pb[r][m] = __ffma2_rn(lo23, make_float2(xv[m][0].z, xv[m][0].w), pb[r][m]);
          pc[r][m] = __ffma2_rn(lo45, make_float2(xv[m][1].x, xv[m][1].y), pc[r][m]);
          const float d6 = fmaf(j6.x, xv[m][3].x, pd[r][m].x + pd[r][m].y);
          float dot = fmaf(8.f, pa[r][m].x + pb[r][m].y,
                           fmaf(32.f, pa[r][m].y + pc[r][m].x,
                                fmaf(128.f, pb[r][m].x + pc[r][m].y, fmaf(512.f, d6, -qs[m * qstride]))));
          dot = fmaf(tail_state, xv[m][3].z, dot);
          acc[r][m] = fmaf(sc, dot, acc[r][m]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The streaming kernel.
// Shared memory: [x: MT][gpr][XG] f32 | [Q: MT][gpr] f32 | per-warp rings:
//   stages x RPW x (CHB + 16 nibble bytes) | mbarriers
// ---------------------------------------------------------------------------
template <int FAM, int RPW, int MT>
__global__ void __launch_bounds__(512, 1) gemv_stream(GemvArgs a) {
  using T = G64<FAM>;
  constexpr int CHB = 32 * T::PB;
  constexpr int RB = CHB + 16;  // ring bytes per row per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t gpr = a.gpr;
  float* xs = reinterpret_cast<float*>(smem);
  const int64_t xstride = gpr * T::XG;  // floats per token
  float* qs = xs + MT * xstride;
  uint8_t* rings = reinterpret_cast<uint8_t*>(qs + ((MT * gpr + 31) / 32) * 32);
  const int S = a.stages;
  uint8_t* ring = rings + size_t(warp) * S * RPW * RB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rings + size_t(nwarps) * S * RPW * RB) + warp * S;

  // Work: whole row tiles, round-robin over all warps of the grid.
  const int64_t gw = int64_t(blockIdx.x) * nwarps + warp;
  const int64_t W = int64_t(gridDim.x) * nwarps;
  const int nch = a.nchunks;
  const int64_t my_tiles = gw < a.tiles ? (a.tiles - gw + W - 1) / W : 0;
  const int64_t n_items = my_tiles * nch;

  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  __syncwarp();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t item) {
    const int s = int(item % S);
    const int64_t tile = gw + (item / nch) * W;
    const int c = int(item % nch);
    const int g0 = c * 32;
    const int ng = int((gpr - g0 < 32 ? gpr - g0 : 32));
    const uint32_t cb = uint32_t((ng * T::PB + 15) & ~15);
    const uint32_t nb = uint32_t(((ng + 1) / 2 + 15) & ~15);
    const int64_t r0 = tile * RPW;
    const int nr = int((a.rows - r0 < RPW ? a.rows - r0 : int64_t(RPW)));
    const bool side = FAM == kF206;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[s], uint32_t(nr) * (cb + (side ? nb : 0u)));
      for (int r = 0; r < nr; ++r) {
        uint8_t* dst = ring + (size_t(s) * RPW + r) * RB;
        bulk_g2s_evict_first(dst, a.codes + (r0 + r) * a.code_stride + int64_t(g0) * T::PB, cb,
                             &bars[s], pol);
        if (side)
          bulk_g2s_evict_first(dst + CHB, a.nibbles + (r0 + r) * a.nib_stride + g0 / 2, nb,
                               &bars[s], pol);
      }
    }
  };

  // Prefetch the first stages while x is being staged.
  const int64_t pre = (n_items < S ? n_items : int64_t(S));
  for (int64_t i = 0; i < pre; ++i) issue(i);

  // Stage x (f32, permuted per family) and the per-group correction Q.
  for (int64_t e = threadIdx.x; e < int64_t(MT) * gpr * 64; e += blockDim.x) {
    const int m = int(e / (gpr * 64));
    const int64_t k = e - int64_t(m) * gpr * 64;
    const int64_t g = k >> 6;
    const int i = int(k & 63);
    const float v = m < a.M ? load_x(a.x, a.x_dtype, int64_t(m) * a.x_stride + k) : 0.f;
    xs[m * xstride + g * T::XG + T::perm(i)] = v;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < int64_t(MT) * gpr; e += blockDim.x) {
    const int m = int(e / gpr);
    const int64_t g = e - int64_t(m) * gpr;
    const float* xg = xs + m * xstride + g * T::XG;
    float q = 0.f;
    for (int i = 0; i < 64; ++i)
      if (!T::exact_tail(i)) q = fmaf(T::cls(i) + float(T::ZP), xg[T::perm(i)], q);
    qs[m * gpr + g] = q;
  }
  __syncthreads();

  float acc[RPW][MT];
  WidenPlan pl[RPW];
  uint32_t sel[RPW][4];
  float scf[RPW];
  int64_t cur_tile = -1;
  for (int64_t it = 0; it < n_items; ++it) {
    const int s = int(it % S);
    const int64_t tile = gw + (it / nch) * W;
    const int c = int(it % nch);
    const int64_t r0 = tile * RPW;
    if (tile != cur_tile) {
      cur_tile = tile;
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[r][m] = 0.f;
        if constexpr (FAM == kF206) {
          const int64_t row = (r0 + r < a.rows ? r0 + r : a.rows - 1);
          pl[r] = a.plan[row];
          // byte b of a word -> byte position sh/8 of q (zeros elsewhere)
          const uint32_t pos = pl[r].sh >> 3;
#pragma unroll
          for (int b = 0; b < 4; ++b) sel[r][b] = (0x4444u & ~(0xFu << (4 * pos))) | (uint32_t(b) << (4 * pos));
        }
      }
    }
    mbar_wait(&bars[s], uint32_t((it / S) & 1));
    const int g = c * 32 + lane;
    if (g < gpr) {
      const uint8_t* st = ring + size_t(s) * RPW * RB;
      const float* xg = xs + g * T::XG;
      const float* qg = qs + g;
      if constexpr (FAM == kF206) {
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          const uint8_t nib = st[r * RB + CHB + (lane >> 1)];
          scf[r] = float((nib >> (4 * (lane & 1))) & 0xF);
        }
        consume_206<RPW, MT>(st, lane, xg, qg, xstride, gpr, pl, sel, scf, acc);
      } else if constexpr (FAM == kF275) {
        consume_275<RPW, MT>(st, lane, xg, qg, xstride, gpr, acc);
      } else {
        consume_25<RPW, MT>(st, lane, xg, qg, xstride, gpr, acc);
      }
    }
    __syncwarp();
    fence_proxy_async_smem();
    if (it + S < n_items) issue(it + S);

    if (c == nch - 1) {
      // Tile done: reduce across lanes, scale by the row super scale, store.
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[r][m] = warp_sum(acc[r][m]);
      if (lane < RPW * MT) {
        const int r = lane / MT, m = lane % MT;
        const int64_t row = r0 + r;
        float v = 0.f;
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
          for (int mm = 0; mm < MT; ++mm)
            if (rr == r && mm == m) v = acc[rr][mm];
        if (row < a.rows && m < a.M) {
          v *= a.super[row];
          if (a.y_dtype == CCQ_DTYPE_F32)
            static_cast<float*>(a.y)[int64_t(m) * a.y_stride + row] = v;
          else
            static_cast<__nv_bfloat16*>(a.y)[int64_t(m) * a.y_stride + row] = __float2bfloat16_rn(v);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Generic fallback for any group geometry / token count: one warp per row,
// lanes stride over groups, exact per-weight decode (kernels.cpp:60-93).
// ---------------------------------------------------------------------------
struct GenericArgs {
  const uint8_t* codes;
  const uint8_t* nibbles;
  const float* super;
  const WidenPlan* plan;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int64_t rows, cols, gpr, M;
  uint64_t code_stride, nib_stride;
  Geometry geo;
};

template <int FAM>
__global__ void __launch_bounds__(256) gemv_generic(GenericArgs a) {
  constexpr FamilyConst fc = family_const(FAM);
  constexpr int TM = 8;
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= a.rows) return;
  WidenPlan pl{};
  if constexpr (fc.cluster) pl = a.plan[row];
  const float sup = a.super[row];
  for (int64_t m0 = 0; m0 < a.M; m0 += TM) {
    float acc[TM];
#pragma unroll
    for (int t = 0; t < TM; ++t) acc[t] = 0.f;
    for (int64_t gj = lane; gj < a.gpr; gj += 32) {
      const uint8_t* p = a.codes + row * a.code_stride + gj * a.geo.payload_bytes;
      auto word = [&](int w) -> uint32_t {
        const uint8_t* q = p + w * fc.word_bytes;
        return fc.word_bytes == 2 ? (uint32_t(q[0]) | (uint32_t(q[1]) << 8)) : uint32_t(q[0]);
      };
      uint32_t sc;
      if (a.geo.embedded_scale) sc = word(a.geo.full_words) & fc.scale_mask;
      else sc = (a.nibbles[row * a.nib_stride + gj / 2] >> (4 * (gj & 1))) & 0xF;
      const float scale = __fmul_rn(float(sc), sup);
      int idx = 0;
      for (int w = 0; w < a.geo.words_per_group; ++w) {
        uint32_t code = word(w);
        if constexpr (fc.cluster) code = widen_hi(code, pl) >> 8;
        const int nk = w < a.geo.full_words ? fc.wpw : 1;
        for (int k = 0; k < nk; ++k, ++idx) {
          const float wv = __fmul_rn(float(int((code >> fc.shifts[k]) & fc.weight_mask) - fc.zero_point), scale);
          const int64_t col = gj * a.geo.group_size + idx;
#pragma unroll
          for (int t = 0; t < TM; ++t)
            if (m0 + t < a.M) acc[t] = fmaf(wv, load_x(a.x, a.x_dtype, (m0 + t) * a.cols + col), acc[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const float v = warp_sum(acc[t]);
      if (lane == 0 && m0 + t < a.M) {
        if (a.y_dtype == CCQ_DTYPE_F32) static_cast<float*>(a.y)[(m0 + t) * a.rows + row] = v;
        else static_cast<__nv_bfloat16*>(a.y)[(m0 + t) * a.rows + row] = __float2bfloat16_rn(v);
      }
    }
  }
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

template <int FAM, int RPW, int MT>
int launch_stream(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M0, int64_t Mn,
                  void* y, int y_dtype, cudaStream_t s) {
  using T = G64<FAM>;
  constexpr int RB = 32 * T::PB + 16;
  GemvArgs a{};
  a.codes = m->codes;
  a.nibbles = m->nibbles;
  a.super = m->super;
  a.plan = m->plan;
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  const size_t yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  a.x = static_cast<const uint8_t*>(x) + size_t(M0) * size_t(m->cols) * xb;
  a.y = static_cast<uint8_t*>(y) + size_t(M0) * size_t(m->rows) * yb;
  a.x_dtype = x_dtype;
  a.y_dtype = y_dtype;
  a.rows = m->rows;
  a.cols = m->cols;
  a.gpr = m->gpr;
  a.code_stride = m->code_stride;
  a.nib_stride = m->nib_stride;
  a.M = int(Mn);
  a.x_stride = m->cols;
  a.y_stride = m->rows;
  a.tiles = (m->rows + RPW - 1) / RPW;
  a.nchunks = int((m->gpr + 31) / 32);

  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  const size_t xbytes = size_t(MT) * m->gpr * T::XG * 4 + size_t((MT * m->gpr + 31) / 32) * 32 * 4;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // Warps per CTA: enough tiles for every warp, balanced across the grid.
  int best_w = 4;
  double best_eff = -1;
  for (int w = 16; w >= 4; --w) {
    const double W = double(sms) * w;
    const double per = double(a.tiles) / W;
    const double eff = per / std::ceil(per) * std::min(1.0, per * 4.0);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best_w = w;
    }
  }
  int stages = 4;
  size_t smem = 0;
  for (;; --stages) {
    smem = xbytes + size_t(best_w) * stages * RPW * RB + size_t(best_w) * stages * 8 + 128;
    if (smem <= size_t(max_smem) || stages == 2) break;
  }
  while (smem > size_t(max_smem) && best_w > 2) {
    --best_w;
    smem = xbytes + size_t(best_w) * stages * RPW * RB + size_t(best_w) * stages * 8 + 128;
  }
  if (smem > size_t(max_smem)) return fail(CCQ_ERR_CONFIG, "activations too large for the streaming GEMV");
  a.stages = stages;
  auto kern = gemv_stream<FAM, RPW, MT>;
  static thread_local size_t configured[3][5][5] = {};
  size_t& conf = configured[FAM][RPW][MT];
  if (conf < smem) {
    CCQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    conf = smem;
  }
  const int64_t warps_needed = a.tiles;
  const int64_t grid = std::min<int64_t>(sms, (warps_needed + best_w - 1) / best_w);
  kern<<<unsigned(grid), unsigned(best_w * 32), smem, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv launch");
}

template <int FAM>
int launch_fam(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
               cudaStream_t s) {
  for (int64_t m0 = 0; m0 < M;) {
    const int64_t left = M - m0;
    int st;
    if (left >= 4 && m->gpr * 64 * 4 * 4 <= 160 * 1024) {
      st = launch_stream<FAM, 2, 4>(m, x, x_dtype, m0, 4, y, y_dtype, s);
      m0 += 4;
    } else if (left >= 2 && m->gpr * 64 * 2 * 4 <= 160 * 1024) {
      st = launch_stream<FAM, 4, 2>(m, x, x_dtype, m0, 2, y, y_dtype, s);
      m0 += 2;
    } else {
      st = launch_stream<FAM, 4, 1>(m, x, x_dtype, m0, 1, y, y_dtype, s);
      m0 += 1;
    }
    if (st != CCQ_OK) return st;
  }
  return CCQ_OK;
}

template <int FAM>
int launch_generic(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                   int y_dtype, cudaStream_t s) {
  GenericArgs a{m->codes, m->nibbles, m->super, m->plan, x, y, x_dtype, y_dtype,
                m->rows, m->cols, m->gpr, M, m->code_stride, m->nib_stride, m->geo};
  gemv_generic<FAM><<<unsigned((m->rows + 7) / 8), 256, 0, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv launch");
}

}  // namespace

bool gemv_fast_supported(const ccq_dev_model* m, int64_t M) {
  return m->geo.group_size == 64 && M <= 8 && m->gpr * 64 * 4 <= 100 * 1024;
}

int launch_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                cudaStream_t s) {
  const bool fast = m->geo.group_size == 64 && m->gpr * 64 * 4 <= 100 * 1024;
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
