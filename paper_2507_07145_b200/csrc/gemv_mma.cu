// Kernel (b), tensor-pipe version: fused decode + GEMV for small batches
// (M <= 16 tokens per launch chunk), all three CCQ families, group size 64.
//
// Reference: ccq::gemv / gemv_batch (kernels.cpp:124-187).
//
// Why the tensor pipe for a GEMV: on sm_100a the CUDA-core decode+FFMA loop
// is bound by the FMA pipe (IMAD.HI for the 2.06 widening plus one FMA lane
// per weight; profiles/r01_micro_pipes.txt: FFMA2 3.64 cycles per warp
// instruction per SMSP).  Here the fields are decoded straight into EXACT f16
// "magic" values 1024 + s*2^p (two fields per LOP3) and dotted with
// warp-level mma.sync.m16n8k16 (f32 accumulate) - the dot product leaves the
// ALU/FMA pipes entirely, and batches up to 8 (16) tokens cost the same
// instructions as one.
//
//   per 64-weight group g, per 16-row tile, per token n:
//     D = sum_k A[r,k] B[k,n] + C,   A = 1024 + s*2^p (f16, exact),
//                                     B = x*2^(s_n - p)   (f16, exact for bf16 x),
//                                     C = -Q[g,n],  Q = sum_k (1024 + zp*2^p) B
//       = 2^s_n * sum_k (s_k - zp) x_k            (only f32 rounding)
//     y[n,r] += sc[r,g] * D       (f32, one FFMA per output per group)
//   y[n,r] *= super[r] * 2^-s_n   at the end.
//
// Work split: persistent CTAs (one per SM) own contiguous 16-row tiles; an
// item is (16-row tile, 8-group K block).  Each warp takes a contiguous range
// of items (tile-major), streams them through its own S-stage shared-memory
// ring filled by 2-D TMA (one box of 16 rows x 8 groups, 128-B swizzle for
// the 16-B groups of 2.06), and keeps its partial outputs in registers until
// its tile changes.  Partials are summed per tile in warp order at the end:
// deterministic, no atomics.
//
// Fragment layout of mma.m16n8k16 (lane L, g = L/4, c = L%4):
//   A: a0 = (row g,   k 2c..2c+1)  a1 = (row g+8, k 2c..2c+1)
//      a2 = (row g,   k 2c+8..+9)  a3 = (row g+8, k 2c+8..+9)
//   B: b0 = (k 2c..2c+1, n g)      b1 = (k 2c+8..+9, n g)
//   C/D: d0,d1 = (row g, n 2c, 2c+1)  d2,d3 = (row g+8, n 2c, 2c+1)
// Lane c decodes 16 of the group's 64 weights for rows g and g+8 as 8 f16x2
// "units"; unit 2t (2t+1) is the a0/a1 (a2/a3) operand of K slice t.  Which
// weight (and field power p) sits in which unit is fixed per family
// (unit_wp below); the activations are staged in the same order.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ccq_internal.hpp"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace ccqb {
namespace {

constexpr int kRowsT = 16;    // rows per tile (MMA M)
constexpr int kBlkG = 8;      // groups per staged K block
constexpr uint32_t kMagic = 0x64006400u;  // f16x2 (1024, 1024)

template <int FAM>
struct MF;
template <>
struct MF<kF206> {
  static constexpr int PB = 16, ZP = 32, BOX = 128, SIDE = 32;  // + nibbles/plan box
};
template <>
struct MF<kF275> {
  static constexpr int PB = 22, ZP = 8, BOX = 176, SIDE = 0;
};
template <>
struct MF<kF25> {
  static constexpr int PB = 20, ZP = 4, BOX = 160, SIDE = 0;
};

// (weight index within the group, field power p) of element e (0 = low half,
// 1 = high half) of unit u (0..7) produced by lane c (0..3).
struct WP {
  int w, p;
};
__host__ __device__ constexpr WP unit_wp(int fam, int c, int u, int e) {
  if (fam == kF206) {
    // byte b = 4c + t; units (s3, 8 s2), (s1, 8 s0); shifts [9,6,3,0] -> weights 4b..4b+3
    const int b = 4 * c + u / 2;
    if ((u & 1) == 0) return e == 0 ? WP{4 * b + 3, 0} : WP{4 * b + 2, 3};
    return e == 0 ? WP{4 * b + 1, 0} : WP{4 * b, 3};
  }
  if (fam == kF275) {
    // bytes B = 5c..5c+4; byte B: shift 4 -> 3B, shift 2 -> 3B+1, shift 0 -> 3B+2
    const int B0 = 5 * c;
    if (u < 6) {
      const int B = B0 + (u / 3) * 2 + e;
      const int f = u % 3;  // 0: shift 0 (p0), 1: shift 2 (p2), 2: shift 4 (p4)
      return f == 0 ? WP{3 * B + 2, 0} : f == 1 ? WP{3 * B + 1, 2} : WP{3 * B, 4};
    }
    const int B4 = B0 + 4;
    if (u == 6) {
      if (e == 0) return WP{3 * B4, 4};
      // extra weight: b20 shift 4 / 2 / 0 for lanes 0..2, tail state (b21 >> 4) for lane 3
      return c == 0 ? WP{60, 4} : c == 1 ? WP{61, 2} : c == 2 ? WP{62, 0} : WP{63, 4};
    }
    return e == 0 ? WP{3 * B4 + 1, 2} : WP{3 * B4 + 2, 0};
  }
  // 2.5: words W = 2c (low half), 2c+1 (high half); field k of word w is
  // weight 7w + k with shifts [13,11,9,6,4,2,0]
  if (u < 7) {
    const int w = 2 * c + e;
    // u: 0 sh0 p0, 1 sh2 p2, 2 sh4 p4, 3 sh6 p6, 4 sh9 p0, 5 sh11 p2, 6 sh13 p4
    const int k = u == 0 ? 6 : u == 1 ? 5 : u == 2 ? 4 : u == 3 ? 3 : u == 4 ? 2 : u == 5 ? 1 : 0;
    const int p = u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 4 : u == 3 ? 6 : u == 4 ? 0 : u == 5 ? 2 : 4;
    return WP{7 * w + k, p};
  }
  // unit 7 from words 8 (and 9)
  if (c == 0) return e == 0 ? WP{56 + 6, 0} : WP{56 + 5, 2};
  if (c == 1) return e == 0 ? WP{56 + 4, 4} : WP{56 + 3, 6};
  if (c == 2) return e == 0 ? WP{56 + 2, 1} : WP{56 + 1, 3};
  return e == 0 ? WP{56 + 0, 5} : WP{63, 5};
}

__device__ __forceinline__ uint32_t lop_or(uint32_t v, uint32_t mask) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(kMagic));
  return d;
}
__device__ __forceinline__ uint32_t ld32(const uint8_t* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Per-row decode state that stays constant over an item.
struct RowCtx {
  uint64_t C;
  uint32_t M;
  uint32_t sel[4];
  uint32_t nib;  // 2.06: nibble word (8 groups) of this row's block
};

// Decode lane c's 16 weights of group j (0..7 within the staged block) of
// tile row `row` into 8 f16x2 units; returns the group's scale code.
template <int FAM>
__device__ __forceinline__ uint32_t decode_units(const uint8_t* tile, int row, int j, int c,
                                                 const RowCtx& rc, uint32_t (&u)[8]) {
  if constexpr (FAM == kF206) {
    const uint32_t w = ld32(tile + row * 128 + ((j ^ (row & 7)) << 4) + 4 * c);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t qb = prmt(w, 0u, rc.sel[t]);
      const uint32_t hi = uint32_t((uint64_t(qb) * rc.M + rc.C) >> 32);  // code at [8,23)
      const uint32_t w2 = prmt(hi, 0u, 0x2121u);                         // code | code << 16
      const uint32_t w3 = w2 >> 6;
      u[2 * t] = lop_or(w2, 0x01F8003Fu);      // (s3, 8 s2)
      u[2 * t + 1] = lop_or(w3, 0x01F8003Fu);  // (s1, 8 s0)
    }
    return (rc.nib >> (4 * j)) & 0xFu;
  } else if constexpr (FAM == kF275) {
    const uint8_t* rb = tile + row * MF<kF275>::BOX;
    const int A = 22 * j + 5 * c;
    const uint32_t w0 = ld32(rb + (A & ~3)), w1 = ld32(rb + (A & ~3) + 4);
    const uint32_t sh = 8u * uint32_t(A & 3);
    const uint32_t lo = __funnelshift_r(w0, w1, sh);
    const uint32_t hi = w1 >> sh;
    const int At = 22 * j + 20;
    const uint32_t wt = ld32(rb + (At & ~3));
    const uint32_t e0 = uint32_t(At & 3);  // byte index of b20 in wt (0 or 2)
    const uint32_t p0 = prmt(lo, 0u, 0x1100u), p1 = prmt(lo, 0u, 0x3322u);
    u[0] = lop_or(p0, 0x000F000Fu);
    u[1] = lop_or(p0, 0x003C003Cu);
    u[2] = lop_or(p0, 0x00F000F0u);
    u[3] = lop_or(p1, 0x000F000Fu);
    u[4] = lop_or(p1, 0x003C003Cu);
    u[5] = lop_or(p1, 0x00F000F0u);
    const uint32_t eb = 4u + e0 + (c == 3 ? 1u : 0u);
    const uint32_t p2 = prmt(hi, wt, (eb << 12) | (eb << 8));
    const uint32_t me = c == 0 ? 0xF0u : c == 1 ? 0x3Cu : c == 2 ? 0x0Fu : 0xF0u;
    u[6] = lop_or(p2, 0x000000F0u | (me << 16));
    u[7] = lop_or(prmt(hi, 0u, 0x0000u), 0x000F003Cu);
    return (wt >> (8u * (e0 + 1u))) & 0xFu;
  } else {
    const uint8_t* gb = tile + row * MF<kF25>::BOX + 20 * j;
    const uint32_t v = ld32(gb + 4 * c), wt = ld32(gb + 16);
    const uint32_t s = v >> 9;
    u[0] = lop_or(v, 0x00070007u);
    u[1] = lop_or(v, 0x001C001Cu);
    u[2] = lop_or(v, 0x00700070u);
    u[3] = lop_or(v, 0x01C001C0u);
    u[4] = lop_or(s, 0x00070007u);
    u[5] = lop_or(s, 0x001C001Cu);
    u[6] = lop_or(s, 0x00700070u);
    const uint32_t sel = c == 0 ? 0x1010u : c == 1 ? 0x1010u : c == 2 ? 0x1111u : 0x3311u;
    const uint32_t mk = c == 0 ? 0x001C0007u : c == 1 ? 0x01C00070u : c == 2 ? 0x0038000Eu : 0x00E000E0u;
    u[7] = lop_or(prmt(wt, wt, sel), mk);
    return (wt >> 16) & 0x1FFFu;
  }
}

struct MmaArgs {
  const float* super;
  const WidenPlan* plan;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int M;            // tokens in this launch chunk (<= 8 * NT)
  int64_t rows, rows_pad, gpr;
  int nblk;         // K blocks of 8 groups per row
  int ntiles;       // 16-row tiles
  int slots;        // partial slots per warp
  int64_t x_ld, y_ld;  // elements between token rows of x / y
  uint32_t xs_bytes;   // staged activation bytes (gpr * M * 128)
};

template <int FAM, int NT, int S, int XDT>
__global__ void __launch_bounds__(384, 1)
    gemv_mma(const __grid_constant__ CUtensorMap tm_codes, const __grid_constant__ CUtensorMap tm_side,
             MmaArgs a) {
  using F = MF<FAM>;
  constexpr int MP = 8 * NT;                       // padded tokens
  constexpr int CODE_B = kRowsT * F::BOX;          // code box bytes
  constexpr int SIDE_B = kRowsT * F::SIDE;         // nibble + plan box bytes
  constexpr int STAGE = ((CODE_B + SIDE_B) + 1023) & ~1023;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, c = lane & 3;

  // shared memory: rings | xs | Q | partials | scale | barriers
  uint8_t* rings = smem;
  uint8_t* xs = rings + size_t(nw) * S * STAGE;                          // [gpr][M][4][32 B]
  float* qs = reinterpret_cast<float*>(xs + a.xs_bytes);                 // [gpr][MP]
  float* part = qs + a.gpr * MP;                                         // [nw][slots][16][MP]
  float* tokscale = part + size_t(nw) * a.slots * kRowsT * MP;           // [MP] 2^-s_n
  int* tokmax = reinterpret_cast<int*>(tokscale + MP);                   // [MP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(tokmax + MP + 2) ;        // [nw][S]
  bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~uintptr_t(7));
  uint64_t* mybar = bars + warp * S;
  uint8_t* ring = rings + size_t(warp) * S * STAGE;

  // CTA tiles and this warp's item range (tile-major items of 8-group blocks)
  const int t_begin = int(int64_t(blockIdx.x) * a.ntiles / gridDim.x);
  const int t_end = int(int64_t(blockIdx.x + 1) * a.ntiles / gridDim.x);
  const int nitems = (t_end - t_begin) * a.nblk;
  const int i0 = int(int64_t(warp) * nitems / nw), i1 = int(int64_t(warp + 1) * nitems / nw);
  const int nmine = i1 - i0;

  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
  if (threadIdx.x < MP) tokmax[threadIdx.x] = 0;
  fence_mbar_init();
  __syncthreads();

  auto issue = [&](int k) {  // item k of this warp into stage k % S
    if (lane == 0 && k < nmine) {
      const int it = i0 + k;
      const int tile = t_begin + it / a.nblk, blk = it % a.nblk;
      const int chunk = blk >> 2;
      const int ycoord = int(int64_t(chunk) * a.rows_pad + int64_t(tile) * kRowsT);
      uint8_t* st = ring + (k % S) * STAGE;
      mbar_arrive_expect_tx(&mybar[k % S], uint32_t(CODE_B + SIDE_B));
      tma_load_2d(st, &tm_codes, (blk & 3) * F::BOX, ycoord, &mybar[k % S]);
      if constexpr (F::SIDE > 0) tma_load_2d(st + CODE_B, &tm_side, 0, ycoord, &mybar[k % S]);
    }
  };
  if (lane == 0) {
    prefetch_tmap(&tm_codes);
    if constexpr (F::SIDE > 0) prefetch_tmap(&tm_side);
  }
#pragma unroll
  for (int k = 0; k < S; ++k) issue(k);
  griddep_launch_dependents();
  griddep_wait();  // x (and y) belong to the previous kernel until here

  // ---- activations: per-token power-of-two scale, then the unit layout ----
  const int M = a.M;
  const int64_t K = a.gpr * 64;
  {
    float mx[MP];
#pragma unroll
    for (int n = 0; n < MP; ++n) mx[n] = 0.f;
    for (int64_t e = int64_t(threadIdx.x) * 8; e < K; e += int64_t(blockDim.x) * 8) {
#pragma unroll
      for (int n = 0; n < MP; ++n) {
        if (n >= M) break;
        float v[8];
        if constexpr (XDT == CCQ_DTYPE_F32) {
          const float4 p = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + n * a.x_ld + e));
          const float4 q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + n * a.x_ld + e) + 1);
          v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w; v[4] = q.x; v[5] = q.y; v[6] = q.z; v[7] = q.w;
        } else {
          const uint4 p = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + n * a.x_ld + e));
          const uint32_t wv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if constexpr (XDT == CCQ_DTYPE_BF16) {
              v[2 * i] = __uint_as_float(wv[i] << 16);
              v[2 * i + 1] = __uint_as_float(wv[i] & 0xFFFF0000u);
            } else {
              v[2 * i] = __half2float(__ushort_as_half(uint16_t(wv[i] & 0xFFFFu)));
              v[2 * i + 1] = __half2float(__ushort_as_half(uint16_t(wv[i] >> 16)));
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[n] = fmaxf(mx[n], fabsf(v[i]));
      }
    }
#pragma unroll
    for (int n = 0; n < MP; ++n) {
      if (n >= M) break;
      float m = mx[n];
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0 && m > 0.f) atomicMax(&tokmax[n], __float_as_int(fminf(m, 3.0e38f)));
    }
  }
  __syncthreads();
  // token scale: put max|x| (times the largest 2^-p = 1) in [2^14, 2^15)
  const int gpr = int(a.gpr);
  // one job per (group G, token n, lane class c), c fastest: the 4 jobs of a
  // group/token sit in one lane quad and combine their Q partials by shuffle.
  const int njobs = gpr * M * 4;
  for (int job0 = threadIdx.x - lane; job0 < njobs; job0 += blockDim.x) {
    const int job = job0 + lane;
    const bool live = job < njobs;
    const int cc = job & 3, G = (job >> 2) / M, n = (job >> 2) % M;
    float qpart = 0.f;
    if (live) {
      const float mxv = __int_as_float(tokmax[n]);
      int ex = 0;
      if (mxv > 0.f) frexpf(mxv, &ex);
      int sh = mxv > 0.f ? 15 - ex : 0;
      sh = sh > 100 ? 100 : (sh < -100 ? -100 : sh);
      const float scale = ldexpf(1.f, sh);
      if (G == 0 && cc == 0) tokscale[n] = ldexpf(1.f, -sh);
      float xv[64];
      const int64_t base = int64_t(n) * a.x_ld + int64_t(G) * 64;
      if constexpr (XDT == CCQ_DTYPE_F32) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float4 p = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + base) + i);
          xv[4 * i] = p.x; xv[4 * i + 1] = p.y; xv[4 * i + 2] = p.z; xv[4 * i + 3] = p.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 p = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + base) + i);
          const uint32_t wv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if constexpr (XDT == CCQ_DTYPE_BF16) {
              xv[8 * i + 2 * q] = __uint_as_float(wv[q] << 16);
              xv[8 * i + 2 * q + 1] = __uint_as_float(wv[q] & 0xFFFF0000u);
            } else {
              xv[8 * i + 2 * q] = __half2float(__ushort_as_half(uint16_t(wv[q] & 0xFFFFu)));
              xv[8 * i + 2 * q + 1] = __half2float(__ushort_as_half(uint16_t(wv[q] >> 16)));
            }
          }
        }
      }
      uint32_t out[8];
      auto stage_units = [&](auto cconst) {
        constexpr int C = decltype(cconst)::value;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          constexpr int dummy = 0;
          (void)dummy;
          const WP w0 = unit_wp(FAM, C, u, 0), w1 = unit_wp(FAM, C, u, 1);
          const __half h0 = __float2half_rn(xv[w0.w] * scale * (1.f / float(1 << w0.p)));
          const __half h1 = __float2half_rn(xv[w1.w] * scale * (1.f / float(1 << w1.p)));
          qpart = fmaf(1024.f + float(F::ZP * (1 << w0.p)), __half2float(h0), qpart);
          qpart = fmaf(1024.f + float(F::ZP * (1 << w1.p)), __half2float(h1), qpart);
          out[u] = uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16);
        }
      };
      switch (cc) {
        case 0: stage_units(std::integral_constant<int, 0>{}); break;
        case 1: stage_units(std::integral_constant<int, 1>{}); break;
        case 2: stage_units(std::integral_constant<int, 2>{}); break;
        default: stage_units(std::integral_constant<int, 3>{}); break;
      }
      uint4* dst = reinterpret_cast<uint4*>(xs + ((size_t(G) * M + n) * 4 + cc) * 32);
      dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
      dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
    qpart += __shfl_xor_sync(0xffffffffu, qpart, 1);
    qpart += __shfl_xor_sync(0xffffffffu, qpart, 2);
    if (live && cc == 0) qs[G * MP + n] = qpart;
  }
  __syncthreads();

  // ---- main loop ----
  float yacc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) yacc[nt][i] = 0.f;
  int cur_tile = nmine > 0 ? i0 / a.nblk : 0;
  const int first_tile = cur_tile;
  RowCtx rc[2];
  auto flush = [&](int tile) {
    float* pp = part + ((size_t(warp) * a.slots + (tile - first_tile)) * kRowsT) * MP;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int n0 = nt * 8 + 2 * c;
      pp[g * MP + n0] = yacc[nt][0];
      pp[g * MP + n0 + 1] = yacc[nt][1];
      pp[(g + 8) * MP + n0] = yacc[nt][2];
      pp[(g + 8) * MP + n0 + 1] = yacc[nt][3];
#pragma unroll
      for (int i = 0; i < 4; ++i) yacc[nt][i] = 0.f;
    }
  };

#pragma unroll 1
  for (int k = 0; k < nmine; ++k) {
    const int it = i0 + k;
    const int tile = it / a.nblk, blk = it % a.nblk;
    if (tile != cur_tile) {
      flush(cur_tile);
      cur_tile = tile;
    }
    const int s = k % S;
    mbar_wait(&mybar[s], uint32_t((k / S) & 1));
    const uint8_t* st = ring + s * STAGE;
    if constexpr (FAM == kF206) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = g + 8 * h;
        const uint4 pv = *reinterpret_cast<const uint4*>(st + CODE_B + r * 32 + 16);
        rc[h].C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
        rc[h].M = pv.z;
        const uint32_t base = pv.w & 0xFFFFu, step = pv.w >> 16;
        rc[h].sel[0] = base;
        rc[h].sel[1] = base + step;
        rc[h].sel[2] = base + 2 * step;
        rc[h].sel[3] = base + 3 * step;
        rc[h].nib = *reinterpret_cast<const uint32_t*>(st + CODE_B + r * 32 + (blk & 3) * 4);
      }
    }
    const int G0 = blk * kBlkG;
    const int ng = gpr - G0 < kBlkG ? gpr - G0 : kBlkG;
#pragma unroll 2
    for (int j = 0; j < ng; ++j) {
      const int G = G0 + j;
      uint32_t ua[8], ub[8];
      const uint32_t sca = decode_units<FAM>(st, g, j, c, rc[0], ua);
      const uint32_t scb = decode_units<FAM>(st, g + 8, j, c, rc[1], ub);
      float d[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int nq = nt * 8 + 2 * c;
        const float2 q2 = *reinterpret_cast<const float2*>(qs + G * MP + nq);
        d[nt][0] = -q2.x; d[nt][1] = -q2.y; d[nt][2] = -q2.x; d[nt][3] = -q2.y;
        const int nb = nt * 8 + g;
        uint4 b01 = make_uint4(0, 0, 0, 0), b23 = make_uint4(0, 0, 0, 0);
        if (nb < M) {
          const uint4* src = reinterpret_cast<const uint4*>(xs + ((size_t(G) * M + nb) * 4 + c) * 32);
          b01 = src[0];
          b23 = src[1];
        }
        const uint32_t bb[8] = {b01.x, b01.y, b01.z, b01.w, b23.x, b23.y, b23.z, b23.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t af[4] = {ua[2 * t], ub[2 * t], ua[2 * t + 1], ub[2 * t + 1]};
          mma16816(d[nt], af, bb[2 * t], bb[2 * t + 1]);
        }
      }
      const float fa = float(sca), fb = float(scb);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        yacc[nt][0] = fmaf(fa, d[nt][0], yacc[nt][0]);
        yacc[nt][1] = fmaf(fa, d[nt][1], yacc[nt][1]);
        yacc[nt][2] = fmaf(fb, d[nt][2], yacc[nt][2]);
        yacc[nt][3] = fmaf(fb, d[nt][3], yacc[nt][3]);
      }
    }
    // release the stage and refill it with item k + S
    __syncwarp();
    if (k + S < nmine) {
      fence_proxy_async_smem();
      issue(k + S);
    }
  }
  if (nmine > 0) flush(cur_tile);
  __syncthreads();

  // ---- per-tile sums in warp order, scaled by super and the token scale ----
  const int ntl = t_end - t_begin;
  for (int e = threadIdx.x; e < ntl * kRowsT * M; e += blockDim.x) {
    const int tl = e / (kRowsT * M), rem = e % (kRowsT * M);
    const int r = rem / M, n = rem % M;
    const int tile = t_begin + tl;
    const int64_t row = int64_t(tile) * kRowsT + r;
    if (row >= a.rows) continue;
    float v = 0.f;
    for (int w = 0; w < nw; ++w) {
      const int wi0 = int(int64_t(w) * nitems / nw), wi1 = int(int64_t(w + 1) * nitems / nw);
      if (wi1 <= wi0) continue;
      const int ft = t_begin + wi0 / a.nblk, lt = t_begin + (wi1 - 1) / a.nblk;
      if (tile < ft || tile > lt) continue;
      v += part[((size_t(w) * a.slots + (tile - ft)) * kRowsT + r) * MP + n];
    }
    v *= a.super[row] * tokscale[n];
    if (a.y_dtype == CCQ_DTYPE_F32)
      static_cast<float*>(a.y)[int64_t(n) * a.y_ld + row] = v;
    else
      static_cast<__nv_bfloat16*>(a.y)[int64_t(n) * a.y_ld + row] = __float2bfloat16_rn(v);
  }
}

struct Cfg {
  int warps, slots;
  size_t smem;
};

template <int FAM, int NT, int S>
Cfg plan_cfg(const ccq_dev_model* m, int M, int grid, int max_smem) {
  using F = MF<FAM>;
  constexpr int MP = 8 * NT;
  constexpr int STAGE = ((kRowsT * F::BOX + kRowsT * F::SIDE) + 1023) & ~1023;
  const int ntiles = int((m->rows + kRowsT - 1) / kRowsT);
  const int nblk = int((m->gpr + kBlkG - 1) / kBlkG);
  const int tiles_cta = (ntiles + grid - 1) / grid;
  for (int warps = 12; warps >= 4; warps -= 4) {
    const int items = tiles_cta * nblk;
    const int per_warp = (items + warps - 1) / warps;
    const int slots = per_warp / nblk + 2;
    const size_t smem = size_t(warps) * S * STAGE + size_t(m->gpr) * M * 128 + size_t(m->gpr) * MP * 4 +
                        size_t(warps) * slots * kRowsT * MP * 4 + MP * 8 + 16 + size_t(warps) * S * 8 + 1024 + 64;
    if (smem <= size_t(max_smem)) return Cfg{warps, slots, smem};
  }
  return Cfg{0, 0, 0};
}

template <int FAM, int NT, int S, int XDT>
int launch_chunk(const ccq_dev_model* m, const CUtensorMap& tmc, const CUtensorMap& tms, const void* x,
                 int M, void* y, int x_dtype, int y_dtype, int grid, const Cfg& cfg, cudaStream_t s) {
  MmaArgs a{};
  a.super = m->super;
  a.plan = m->plan;
  a.x = x;
  a.y = y;
  a.x_dtype = x_dtype;
  a.y_dtype = y_dtype;
  a.M = M;
  a.rows = m->rows;
  a.rows_pad = m->rows_pad;
  a.gpr = m->gpr;
  a.nblk = int((m->gpr + kBlkG - 1) / kBlkG);
  a.ntiles = int((m->rows + kRowsT - 1) / kRowsT);
  a.slots = cfg.slots;
  a.x_ld = m->cols;
  a.y_ld = m->rows;
  a.xs_bytes = uint32_t(m->gpr * M * 128);
  auto kern = gemv_mma<FAM, NT, S, XDT>;
  static size_t configured[3][3] = {};
  size_t& conf = configured[NT][XDT];
  if (conf < cfg.smem) {
    CCQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cfg.smem)));
    conf = cfg.smem;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(grid));
  lc.blockDim = dim3(unsigned(cfg.warps * 32));
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, tmc, tms, a);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv_mma launch");
}

template <int FAM>
int launch_fam_mma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                   cudaStream_t s) {
  using F = MF<FAM>;
  constexpr int S = 4;
  CUtensorMap tmc{}, tms{};
  int st = make_map_2d(&tmc, CU_TENSOR_MAP_DATA_TYPE_UINT8, m->codes, m->rec, uint64_t(m->nch) * m->rows_pad,
                       m->rec, F::BOX, kRowsT,
                       FAM == kF206 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != CCQ_OK) return st;
  if constexpr (F::SIDE > 0) {
    st = make_map_2d(&tms, CU_TENSOR_MAP_DATA_TYPE_UINT8, m->codes + m->cgb, F::SIDE,
                     uint64_t(m->nch) * m->rows_pad, m->rec, F::SIDE, kRowsT, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (st != CCQ_OK) return st;
  } else {
    tms = tmc;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int ntiles = int((m->rows + kRowsT - 1) / kRowsT);
  const int grid = std::min(num_sms(dev), ntiles);
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2, yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  for (int64_t m0 = 0; m0 < M;) {
    // largest token chunk whose staged activations fit next to the rings
    int chunk = int(std::min<int64_t>(M - m0, kMmaMaxTokens));
    Cfg cfg{};
    for (; chunk >= 1; --chunk) {
      cfg = chunk > 8 ? plan_cfg<FAM, 2, S>(m, chunk, grid, max_smem) : plan_cfg<FAM, 1, S>(m, chunk, grid, max_smem);
      if (cfg.warps) break;
    }
    if (chunk < 1) return fail(CCQ_ERR_CONFIG, "gemv_mma: activations do not fit in shared memory");
    const void* xc = static_cast<const uint8_t*>(x) + size_t(m0) * m->cols * xb;
    void* yc = static_cast<uint8_t*>(y) + size_t(m0) * m->rows * yb;
    if (chunk > 8) {
      switch (x_dtype) {
        case CCQ_DTYPE_F32: st = launch_chunk<FAM, 2, S, CCQ_DTYPE_F32>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        case CCQ_DTYPE_BF16: st = launch_chunk<FAM, 2, S, CCQ_DTYPE_BF16>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        default: st = launch_chunk<FAM, 2, S, CCQ_DTYPE_F16>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s);
      }
    } else {
      switch (x_dtype) {
        case CCQ_DTYPE_F32: st = launch_chunk<FAM, 1, S, CCQ_DTYPE_F32>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        case CCQ_DTYPE_BF16: st = launch_chunk<FAM, 1, S, CCQ_DTYPE_BF16>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        default: st = launch_chunk<FAM, 1, S, CCQ_DTYPE_F16>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s);
      }
    }
    if (st != CCQ_OK) return st;
    m0 += chunk;
  }
  return CCQ_OK;
}

}  // namespace

bool gemv_mma_supported(const ccq_dev_model* m, int64_t M) {
  (void)M;
  if (m->geo.group_size != 64 || m->cols % 64 != 0 || m->cols == 0) return false;
  if (std::getenv("CCQ_GEMV_STREAM")) return false;  // debug: force the CUDA-core kernel
  return true;
}

int launch_gemv_mma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                    cudaStream_t s) {
  switch (m->family) {
    case kF275: return launch_fam_mma<kF275>(m, x, x_dtype, M, y, y_dtype, s);
    case kF25: return launch_fam_mma<kF25>(m, x, x_dtype, M, y, y_dtype, s);
    default: return launch_fam_mma<kF206>(m, x, x_dtype, M, y, y_dtype, s);
  }
}

}  // namespace ccqb
