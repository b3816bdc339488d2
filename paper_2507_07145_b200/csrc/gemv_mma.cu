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
#include <vector>

#include "ccq_internal.hpp"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace ccqb {
namespace {

constexpr int kRowsT = 16;    // rows per tile (MMA M)
constexpr uint32_t kMagic = 0x64006400u;  // f16x2 (1024, 1024)

template <int FAM>
struct MF;
template <>
struct MF<kF206> {
  // 4-group K blocks (64-B box, 64-B swizzle) + nibbles/plan box
  static constexpr int PB = 16, ZP = 32, BLK = 4, BOX = 64, SIDE = 32;
};
template <>
struct MF<kF275> {
  static constexpr int PB = 22, ZP = 8, BLK = 8, BOX = 176, SIDE = 0;
};
template <>
struct MF<kF25> {
  static constexpr int PB = 20, ZP = 4, BLK = 4, BOX = 80, SIDE = 0;
};

__device__ __forceinline__ uint32_t lop_or(uint32_t v, uint32_t mask) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(kMagic));
  return d;
}
__device__ __forceinline__ uint32_t lop_mg(uint32_t v, uint32_t mask, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(magic));
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
template <int FAM, bool P2>
__device__ __forceinline__ uint32_t decode_units(const uint8_t* tile, int row, int j, int c,
                                                 const RowCtx& rc, uint32_t (&u)[8]) {
  if constexpr (FAM == kF206) {
    // `tile` already points at this lane's word of group j (see group())
    (void)row; (void)j; (void)c;
    const uint32_t w = ld32(tile);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t qb = prmt(w, 0u, rc.sel[t]);
      const uint32_t hi = uint32_t((uint64_t(qb) * rc.M + rc.C) >> 32);
      uint32_t w2, w3;
      if constexpr (P2) {
        // plan shifted down one byte: hi == code exactly; duplicate it into
        // both halves on the FMA pipe (IMAD) instead of the ALU (PRMT), and
        // alternate the >> 6 between the ALU (SHF) and the FMA pipe (IMAD.HI)
        w2 = hi * 0x00010001u;
        w3 = (t & 1) ? __umulhi(w2, 1u << 26) : (w2 >> 6);
      } else {
        w2 = prmt(hi, 0u, 0x2121u);  // code at [8,23): code | code << 16
        w3 = w2 >> 6;
      }
      // natural K order: unit 2t = (w 4b, 4b+1) = (s0, s1), unit 2t+1 = (s2, s3);
      // the p3 field takes magic 128 (ulp 1/8) so every unit value is
      // offset + s exactly, with no power of two left on the activation
      u[2 * t] = lop_mg(w3, 0x003F01F8u, 0x64005800u);
      u[2 * t + 1] = lop_mg(w2, 0x003F01F8u, 0x64005800u);
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

#ifdef CCQ_GEMV_TRACE
}  // namespace
__device__ unsigned long long g_mtrace[4096 * 8];
namespace {
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MTRACE(slot, val)                                                        \
  if (lane == 0) {                                                              \
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);       \
    if (gwid < 4096) g_mtrace[gwid * 8 + (slot)] = (val);                        \
  }
#else
#define MTRACE(slot, val)
#endif

struct MmaArgs {
  const float* super;
  const WidenPlan* plan;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int M;            // tokens in this launch chunk (<= 8 * NT)
  int64_t rows, rows_pad, gpr;
  int nblk;         // K blocks of MF::BLK groups per row
  int ntiles;       // 16-row tiles
  int slots;        // partial slots per warp
  int64_t x_ld, y_ld;  // elements between token rows of x / y
  uint32_t xs_bytes;   // staged activation bytes (gpr * M * 128)
  // record path (gemv_rec): device records, their stride, K chunks, ring depth
  const uint8_t* codes;
  uint32_t rec;
  int nch;
  int S;
  // grouped experts (gemv_rec206<.., true>): E stacked experts of rows_e rows,
  // tokens expert-major with offsets[E+1] (device); only experts with tokens run
  const int32_t* offsets;
  int E;
  int64_t rows_e;
};

// Activations -> shared memory in the f16 operand layout of the family (see
// the kernel comment): per-token power-of-two scale, -Q per (group, token).
// Called by every thread of the CTA (contains __syncthreads).
template <int FAM, int MP, int XDT>
__device__ __forceinline__ void stage_activations(const MmaArgs& a, uint8_t* xs, float* qs, float* tokscale,
                                                  int* tokmax, int M, int gpr, int lane, int tok0 = 0) {
  using F = MF<FAM>;
  // ---- activations: raw rows in by bulk copy, per-token power-of-two scale,
  //      then converted IN PLACE to f16 (same byte size) ----
  const uint32_t row_bytes = uint32_t(gpr) * 128u;
  const uint32_t tok_stride = row_bytes + 16u;  // +16 B: tokens land in different banks
  auto to_f32 = [](uint32_t wv, float& lo, float& hi) {
    if constexpr (XDT == CCQ_DTYPE_BF16) {
      lo = __uint_as_float(wv << 16);
      hi = __uint_as_float(wv & 0xFFFF0000u);
    } else {
      lo = __half2float(__ushort_as_half(uint16_t(wv & 0xFFFFu)));
      hi = __half2float(__ushort_as_half(uint16_t(wv >> 16)));
    }
  };
  const int chunks = gpr * 8;  // 16-byte chunks per token
  {
    // every thread loads 16-byte chunks of x straight from global memory,
    // keeps a running max per token and parks the raw bytes in xs
    float mx[MP];
#pragma unroll
    for (int n = 0; n < MP; ++n) mx[n] = 0.f;
    for (int idx = threadIdx.x; idx < chunks * M; idx += blockDim.x) {
      const int n = idx / chunks, i = idx - n * chunks;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + int64_t(tok0 + n) * a.x_ld) + i);
      *reinterpret_cast<uint4*>(xs + size_t(n) * tok_stride + size_t(i) * 16) = v;
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
      float m = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float lo, hi;
        to_f32(wv[q], lo, hi);
        m = fmaxf(m, fmaxf(fabsf(lo), fabsf(hi)));
      }
#pragma unroll
      for (int nn = 0; nn < MP; ++nn)
        if (nn == n) mx[nn] = fmaxf(mx[nn], m);
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
  auto token_scale = [&](int n) {
    const float mxv = __int_as_float(tokmax[n]);
    int ex = 0;
    if (mxv > 0.f) frexpf(mxv, &ex);
    int sh = mxv > 0.f ? 15 - ex : 0;
    return sh > 100 ? 100 : (sh < -100 ? -100 : sh);
  };
  if constexpr (FAM == kF206) {
    // natural K order: one 16-byte chunk (8 weights) per thread, in place;
    // Q of a group = 8 consecutive chunks, combined by shuffles.
    // Q coefficients: offset (128 for even, 1024 for odd weights) + zero point
    for (int job0 = threadIdx.x - lane; job0 < chunks * M; job0 += blockDim.x) {
      const int idx = job0 + lane;
      const bool live = idx < chunks * M;
      const int n = live ? idx / chunks : 0, i = live ? idx % chunks : 0;
      uint4* ptr = reinterpret_cast<uint4*>(xs + size_t(n) * tok_stride + size_t(i) * 16);
      float qpart = 0.f;
      if (live) {
        const int sh = token_scale(n);
        const float scale = ldexpf(1.f, sh);
        if (i == 0) tokscale[n] = ldexpf(1.f, -sh);
        const uint4 v = *ptr;
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float lo, hi;
          to_f32(wv[q], lo, hi);
          const __half2 h = __floats2half2_rn(lo * scale, hi * scale);
          const float2 hf = __half22float2(h);
          qpart = fmaf(128.f + float(F::ZP), hf.x, qpart);
          qpart = fmaf(1024.f + float(F::ZP), hf.y, qpart);
          o[q] = *reinterpret_cast<const uint32_t*>(&h);
        }
        *ptr = make_uint4(o[0], o[1], o[2], o[3]);
      }
      qpart += __shfl_xor_sync(0xffffffffu, qpart, 1);
      qpart += __shfl_xor_sync(0xffffffffu, qpart, 2);
      qpart += __shfl_xor_sync(0xffffffffu, qpart, 4);
      if (live && (i & 7) == 0) qs[(i >> 3) * MP + n] = -qpart;
    }
  } else {
    // permuted unit layout: one (token, group) per thread, all four lane
    // classes (no divergence), in place (the thread owns the group's 128 B)
    for (int job = threadIdx.x; job < gpr * M; job += blockDim.x) {
      const int n = job / gpr, G = job % gpr;
      uint8_t* gx = xs + size_t(n) * tok_stride + size_t(G) * 128;
      const int sh = token_scale(n);
      const float scale = ldexpf(1.f, sh);
      if (G == 0) tokscale[n] = ldexpf(1.f, -sh);
      float xv[64];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = *reinterpret_cast<const uint4*>(gx + 16 * i);
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) to_f32(wv[q], xv[8 * i + 2 * q], xv[8 * i + 2 * q + 1]);
      }
      float qsum = 0.f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t out[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const WP w0 = unit_wp(FAM, cc, u, 0), w1 = unit_wp(FAM, cc, u, 1);
          const __half h0 = __float2half_rn(xv[w0.w] * scale * (1.f / float(1 << w0.p)));
          const __half h1 = __float2half_rn(xv[w1.w] * scale * (1.f / float(1 << w1.p)));
          qsum = fmaf(1024.f + float(F::ZP * (1 << w0.p)), __half2float(h0), qsum);
          qsum = fmaf(1024.f + float(F::ZP * (1 << w1.p)), __half2float(h1), qsum);
          out[u] = uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16);
        }
        uint4* dst = reinterpret_cast<uint4*>(gx + cc * 32);
        dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
        dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
      }
      qs[G * MP + n] = -qsum;
    }
  }
  // tokens n in [M, MP): -Q = 0 so padded accumulator columns stay zero
  for (int e = threadIdx.x; e < gpr * (MP - M); e += blockDim.x)
    qs[(e / (MP - M)) * MP + M + e % (MP - M)] = 0.f;
  __syncthreads();
}

template <int FAM, int NT, int S, int XDT, bool P2, bool GROUPED = false>
__global__ void __launch_bounds__(512, 1)
    gemv_mma(const __grid_constant__ CUtensorMap tm_codes, const __grid_constant__ CUtensorMap tm_side,
             MmaArgs a) {
  static_assert(XDT != CCQ_DTYPE_F32, "f32 activations use the CUDA-core GEMV");
  using F = MF<FAM>;
  constexpr int MP = 8 * NT;                       // padded tokens
  constexpr int CODE_B = kRowsT * F::BOX;          // code box bytes
  constexpr int SIDE_B = kRowsT * F::SIDE;         // nibble + plan box bytes
  constexpr int STAGE = ((CODE_B + SIDE_B) + 511) & ~511;
  extern __shared__ uint8_t smem_raw[];
  // align by offset (not via an integer cast) so every derived pointer keeps
  // the shared address space and compiles to LDS, not generic LD
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int M = a.M;
  const int gpr = int(a.gpr);

  // shared memory: rings | xs | -Q | partials | token scales | warp ranges | barriers
  uint8_t* rings = smem;
  uint8_t* xs = rings + size_t(nw) * S * STAGE;                          // [M][gpr][4][32 B]
  float* qs = reinterpret_cast<float*>(xs + a.xs_bytes);                 // [gpr][MP]  (-Q)
  float* part = qs + a.gpr * MP;                                         // [nw][slots][16][MP]
  float* tokscale = part + size_t(nw) * a.slots * kRowsT * MP;           // [MP] 2^-s_n
  int* tokmax = reinterpret_cast<int*>(tokscale + MP);                   // [MP]
  int* wrange = tokmax + MP;                                             // [16][2] first/last tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(wrange + 64);             // [nw][S] + 1 (x copy)
  uint64_t* mybar = bars + warp * S;
  uint64_t* xbar = bars + nw * S;
  uint8_t* ring = rings + size_t(warp) * S * STAGE;

  // grouped experts: compact the experts that have tokens; their tiles are the work
  __shared__ int hit[256];
  __shared__ int nhit_s, wsum[16];
  int ntiles = a.ntiles;
  const int tpe = GROUPED ? int(a.rows_e / kRowsT) : 1;
  if constexpr (GROUPED) {
    const int e = threadIdx.x;
    const bool has = e < a.E && a.offsets[e + 1] > a.offsets[e];
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < nw; ++w) { const int t = wsum[w]; wsum[w] = acc; acc += t; }
      nhit_s = acc;
    }
    __syncthreads();
    if (has) hit[wsum[warp] + __popc(bal & ((1u << lane) - 1u))] = e;
    __syncthreads();
    ntiles = nhit_s * tpe;
  }
  // tile -> stack row of its first row, token range (expert-major x / y)
  auto tile_info = [&](int t, int64_t& row0, int& off, int& cnt) {
    if constexpr (GROUPED) {
      const int e = hit[t / tpe];
      row0 = int64_t(e) * a.rows_e + int64_t(t % tpe) * kRowsT;
      off = a.offsets[e];
      cnt = a.offsets[e + 1] - off;
    } else {
      row0 = int64_t(t) * kRowsT;
      off = 0;
      cnt = a.M;
    }
  };
  // CTA tiles and this warp's item range (tile-major items of K blocks)
  const int t_begin = int(int64_t(blockIdx.x) * ntiles / gridDim.x);
  const int t_end = int(int64_t(blockIdx.x + 1) * ntiles / gridDim.x);
  const int nitems = (t_end - t_begin) * a.nblk;
  int tok0 = 0, Mc = M;  // staged token window
  if constexpr (GROUPED) {
    Mc = 0;
    if (t_end > t_begin) {
      int64_t r0;
      int o0, c0, o1, c1;
      tile_info(t_begin, r0, o0, c0);
      tile_info(t_end - 1, r0, o1, c1);
      tok0 = o0;
      Mc = o1 + c1 - o0;
    }
  }
  const int i0 = int(int64_t(warp) * nitems / nw), i1 = int(int64_t(warp + 1) * nitems / nw);
  const int nmine = i1 - i0;

#ifdef CCQ_GEMV_TRACE
  MTRACE(0, gtime());
#endif
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
    wrange[2 * warp] = nmine > 0 ? i0 / a.nblk : 1 << 30;
    wrange[2 * warp + 1] = nmine > 0 ? (i1 - 1) / a.nblk : -1;
  }
  if (threadIdx.x == 0) mbar_init(xbar, 1);
  if (threadIdx.x < MP) tokmax[threadIdx.x] = 0;
  if (threadIdx.x < 32) wrange[32 + threadIdx.x] = 0;  // zero block for dead B lanes
  fence_mbar_init();
  __syncthreads();

  // item cursor for the TMA producer (lane 0): (tile, block) of item k,
  // advanced incrementally - no divisions in the loop
  int iss_tile = nmine > 0 ? t_begin + i0 / a.nblk : 0, iss_blk = nmine > 0 ? i0 % a.nblk : 0;
  auto issue = [&](int k) {  // item k (the next one in order) into stage k % S
    if (lane == 0 && k < nmine) {
      constexpr int BPC = kChunk / F::BLK;  // blocks per 32-group chunk
      const int chunk = iss_blk / BPC;
      int64_t row0;
      int toff_, tcnt_;
      tile_info(iss_tile, row0, toff_, tcnt_);
      const int ycoord = int(int64_t(chunk) * a.rows_pad + row0);
      uint8_t* st = ring + (k % S) * STAGE;
      mbar_arrive_expect_tx(&mybar[k % S], uint32_t(CODE_B + SIDE_B));
      tma_load_2d(st, &tm_codes, (iss_blk - chunk * BPC) * F::BOX, ycoord, &mybar[k % S]);
      if constexpr (F::SIDE > 0) tma_load_2d(st + CODE_B, &tm_side, 0, ycoord, &mybar[k % S]);
      if (++iss_blk == a.nblk) {
        iss_blk = 0;
        ++iss_tile;
      }
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
#ifdef CCQ_GEMV_TRACE
  MTRACE(1, gtime());
#endif

  const uint32_t row_bytes = uint32_t(gpr) * 128u;
  const uint32_t tok_stride = row_bytes + 16u;  // +16 B: tokens land in different banks
  stage_activations<FAM, MP, XDT>(a, xs, qs, tokscale, tokmax, Mc, gpr, lane, tok0);
#ifdef CCQ_GEMV_TRACE
  MTRACE(3, gtime());
  MTRACE(7, nmine);
#endif

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
      *reinterpret_cast<float2*>(pp + g * MP + n0) = make_float2(yacc[nt][0], yacc[nt][1]);
      *reinterpret_cast<float2*>(pp + (g + 8) * MP + n0) = make_float2(yacc[nt][2], yacc[nt][3]);
#pragma unroll
      for (int i = 0; i < 4; ++i) yacc[nt][i] = 0.f;
    }
  };
  // this lane's B operand rows: token nb = nt*8 + g; lanes past M read a
  // zero block (G stride 0) instead of branching
  const uint8_t* xb[NT];
  uint32_t gstride[NT];
  uint8_t* zblk = reinterpret_cast<uint8_t*>(wrange + 32);  // 128 B of zeros
  const float* qlane = qs + 2 * c;
  // B operand rows and -Q columns of a tile's tokens (grouped: the tile's
  // expert, as rows of the staged window)
  auto set_tokens = [&](int tile_abs) {
    int64_t r0;
    int toff, tcnt;
    tile_info(tile_abs, r0, toff, tcnt);
    toff -= tok0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int nb = nt * 8 + g;
      const bool live = nb < tcnt;
      xb[nt] = live ? xs + size_t(toff + nb) * tok_stride + c * 32 : zblk + c * 32;
      gstride[nt] = live ? 128u : 0u;
    }
    qlane = qs + toff + 2 * c;
  };
  if (nmine > 0) set_tokens(t_begin + i0 / a.nblk);

  // one 64-weight group: decode both rows, 4 K slices x NT token tiles of
  // mma, then y += sc * D
  auto group = [&](const uint8_t* st, int j, int G) {
    uint32_t ua[8], ub[8];
    uint32_t sca, scb;
    if constexpr (FAM == kF206) {
      // 64-B swizzle: 16-B chunk j of row r sits at r*64 + ((j ^ ((r >> 1) & 3)) << 4);
      // rows g and g+8 share the XOR term, so one per-lane offset serves both
      const uint8_t* p = st + g * 64 + ((j ^ ((g >> 1) & 3)) << 4) + 4 * c;
      sca = decode_units<FAM, P2>(p, g, j, c, rc[0], ua);
      scb = decode_units<FAM, P2>(p + 8 * 64, g + 8, j, c, rc[1], ub);
    } else {
      sca = decode_units<FAM, P2>(st, g, j, c, rc[0], ua);
      scb = decode_units<FAM, P2>(st, g + 8, j, c, rc[1], ub);
    }
    const float fa = float(sca), fb = float(scb);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float q0, q1;
      if constexpr (GROUPED) {  // odd token offsets: scalar loads
        q0 = qlane[G * MP + nt * 8];
        q1 = qlane[G * MP + nt * 8 + 1];
      } else {
        const float2 q2 = *reinterpret_cast<const float2*>(qlane + G * MP + nt * 8);
        q0 = q2.x;
        q1 = q2.y;
      }
      float d[4] = {q0, q1, q0, q1};
      const uint4* src = reinterpret_cast<const uint4*>(xb[nt] + uint32_t(G) * gstride[nt]);
      const uint4 b01 = src[0], b23 = src[1];
      const uint32_t bb[8] = {b01.x, b01.y, b01.z, b01.w, b23.x, b23.y, b23.z, b23.w};
      // two independent accumulator chains (slices 0,2 and 1,3): halves the
      // dependent-mma latency per group
      float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t af[4] = {ua[2 * t], ub[2 * t], ua[2 * t + 1], ub[2 * t + 1]};
        if (t & 1) mma16816(e, af, bb[2 * t], bb[2 * t + 1]);
        else mma16816(d, af, bb[2 * t], bb[2 * t + 1]);
      }
      yacc[nt][0] = fmaf(fa, d[0] + e[0], yacc[nt][0]);
      yacc[nt][1] = fmaf(fa, d[1] + e[1], yacc[nt][1]);
      yacc[nt][2] = fmaf(fb, d[2] + e[2], yacc[nt][2]);
      yacc[nt][3] = fmaf(fb, d[3] + e[3], yacc[nt][3]);
    }
  };

  int tile = cur_tile, blk = nmine > 0 ? i0 % a.nblk : 0;
  bool need_plan = true;
#pragma unroll 1
  for (int k = 0; k < nmine; ++k) {
    if (tile != cur_tile) {
      flush(cur_tile);
      cur_tile = tile;
      need_plan = true;
      if constexpr (GROUPED) set_tokens(t_begin + tile);
    }
    const int s = k % S;
    mbar_wait(&mybar[s], uint32_t((k / S) & 1));
#ifdef CCQ_GEMV_TRACE
    if (k == 0) { MTRACE(4, gtime()); }
#endif
    const uint8_t* st = ring + s * STAGE;
    if constexpr (FAM == kF206) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = g + 8 * h;
        if (need_plan) {  // the row plans change only with the tile
          const uint4 pv = *reinterpret_cast<const uint4*>(st + CODE_B + r * 32 + 16);
          rc[h].C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
          rc[h].M = pv.z;
          uint32_t base = pv.w & 0xFFFFu, step = pv.w >> 16;
          if constexpr (P2) {
            // derive the plan one byte lower: same M, C >> 8, byte position - 1
            // (exact: floor(floor(v / 2^8) / 2^32) == floor(v / 2^40))
            rc[h].C >>= 8;
            step = step > 1u ? step >> 4 : 1u;
            const uint32_t pos = step == 1u ? 0u : step == 16u ? 1u : step == 256u ? 2u : 3u;
            base = (0x4444u & ~(0xFu << (4u * pos))) & 0xFFFFu;
          }
          rc[h].sel[0] = base;
          rc[h].sel[1] = base + step;
          rc[h].sel[2] = base + 2 * step;
          rc[h].sel[3] = base + 3 * step;
        }
        // nibbles of this block's 4 groups: 2 bytes at (blk % 8) * 2
        rc[h].nib = uint32_t(*reinterpret_cast<const uint16_t*>(st + CODE_B + r * 32 + (blk & 7) * 2));
      }
      need_plan = false;
    }
    const int G0 = blk * F::BLK;
    if (gpr - G0 >= F::BLK) {
#pragma unroll
      for (int j = 0; j < F::BLK; ++j) group(st, j, G0 + j);
    } else {
#pragma unroll 1
      for (int j = 0; j < gpr - G0; ++j) group(st, j, G0 + j);
    }
    // release the stage and refill it with item k + S
    __syncwarp();
    if (k + S < nmine) {
      fence_proxy_async_smem();
      issue(k + S);
    }
    if (++blk == a.nblk) {
      blk = 0;
      ++tile;
    }
  }
  if (nmine > 0) flush(cur_tile);
#ifdef CCQ_GEMV_TRACE
  MTRACE(5, gtime());
#endif
  __syncthreads();

  // ---- per-tile sums in warp order, scaled by super and the token scale ----
  const int ntl = t_end - t_begin;
  for (int e = threadIdx.x; e < ntl * kRowsT * MP; e += blockDim.x) {
    const int tl = e / (kRowsT * MP), rem = e % (kRowsT * MP);
    const int r = rem / MP, n = rem % MP;
    int64_t row0;
    int toff, tcnt;
    tile_info(t_begin + tl, row0, toff, tcnt);
    const int64_t row = row0 + r;
    if (n >= tcnt || row >= a.rows) continue;
    float v = 0.f;
    for (int w = 0; w < nw; ++w) {
      const int ft = wrange[2 * w], lt = wrange[2 * w + 1];
      if (tl >= ft && tl <= lt) v += part[((size_t(w) * a.slots + (tl - ft)) * kRowsT + r) * MP + n];
    }
    v *= a.super[row] * tokscale[toff - tok0 + n];
    const int64_t yi = GROUPED ? int64_t(toff + n) * a.rows_e + (row % a.rows_e) : int64_t(n) * a.y_ld + row;
    if (a.y_dtype == CCQ_DTYPE_F32)
      static_cast<float*>(a.y)[yi] = v;
    else
      static_cast<__nv_bfloat16*>(a.y)[yi] = __float2bfloat16_rn(v);
  }
#ifdef CCQ_GEMV_TRACE
  MTRACE(6, gtime());
#endif
}


// ---------------------------------------------------------------------------
// 2.06 "record" variant: the data path of the CUDA-core streaming GEMV (16
// consecutive (chunk, row) records = ONE contiguous bulk copy per item, as
// many items in flight as shared memory holds - for the BASELINE shapes the
// whole CTA's weights are requested at kernel start) with the tensor-pipe
// decode above.  A dedicated producer warp refills the ring; consumer warps
// take (item, quarter) units round-robin (8 groups each) and write their
// partial sums to shared memory; per-(tile, row, token) sums are formed in a
// fixed order at the end.
// ---------------------------------------------------------------------------
template <int NT, int XDT, bool GROUPED>
__global__ void __launch_bounds__(416, 1)
    gemv_rec206(MmaArgs a) {
  constexpr int FAM = kF206;
  constexpr int MP = 8 * NT;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x >> 5) - 1;  // consumer warps; warp nw is the producer
  const int g = lane >> 2, c = lane & 3;
  const int M = a.M, gpr = int(a.gpr), nch = a.nch, S = a.S;
  const uint32_t rec = a.rec;
  const uint32_t stg = (16u * rec + 127u) & ~127u;

  // grouped: compact the experts that have tokens (hit[]), their tiles are the work
  __shared__ int hit[256];
  __shared__ int nhit_s, wsum[16];
  int ntiles = a.ntiles;
  const int tpe = GROUPED ? int(a.rows_e / kRowsT) : 1;
  if constexpr (GROUPED) {
    const int e = threadIdx.x;
    const bool has = e < a.E && a.offsets[e + 1] > a.offsets[e];
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) { const int t = wsum[w]; wsum[w] = acc; acc += t; }
      nhit_s = acc;
    }
    __syncthreads();
    if (has) hit[wsum[warp] + __popc(bal & ((1u << lane) - 1u))] = e;
    __syncthreads();
    ntiles = nhit_s * tpe;
  }
  // (tile index within this launch) -> stack row of its first row, expert, token range
  auto tile_info = [&](int t, int64_t& row0, int& off, int& cnt) {
    if constexpr (GROUPED) {
      const int e = hit[t / tpe];
      row0 = int64_t(e) * a.rows_e + int64_t(t % tpe) * kRowsT;
      off = a.offsets[e];
      cnt = a.offsets[e + 1] - off;
    } else {
      row0 = int64_t(t) * kRowsT;
      off = 0;
      cnt = a.M;
    }
  };
  const int t_begin = int(int64_t(blockIdx.x) * ntiles / gridDim.x);
  const int t_end = int(int64_t(blockIdx.x + 1) * ntiles / gridDim.x);
  const int ntl = t_end - t_begin;
  const int items = ntl * nch, units = items * 4;
  // grouped: this CTA stages only the tokens of the experts its tiles belong to
  // (expert-major layout: one contiguous window [tok0, tok0 + Mc))
  int tok0 = 0, Mc = M;
  if constexpr (GROUPED) {
    if (ntl > 0) {
      int64_t r0;
      int o0, c0, o1, c1;
      tile_info(t_begin, r0, o0, c0);
      tile_info(t_end - 1, r0, o1, c1);
      tok0 = o0;
      Mc = o1 + c1 - o0;
    } else {
      Mc = 0;
    }
  }

  uint8_t* ring = smem;
  uint8_t* xs = ring + size_t(S) * stg;
  float* qs = reinterpret_cast<float*>(xs + a.xs_bytes);
  float* part = qs + a.gpr * MP;                                     // [units][16][MP]
  float* tokscale = part + size_t(units) * kRowsT * MP;
  int* tokmax = reinterpret_cast<int*>(tokscale + MP);
  uint8_t* zblk = reinterpret_cast<uint8_t*>(tokmax + MP);           // 128 B zeros
  uint64_t* full = reinterpret_cast<uint64_t*>(zblk + 128);
  uint64_t* empty = full + S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
  }
  if (threadIdx.x < MP) tokmax[threadIdx.x] = 0;
  if (threadIdx.x < 32) reinterpret_cast<int*>(zblk)[threadIdx.x] = 0;
  fence_mbar_init();
  __syncthreads();

  const bool producer = warp == nw;
  auto produce = [&](int i) {
    const int s = i % S;
    const int chunk = i % nch;
    int64_t row0;
    int off, cnt;
    tile_info(t_begin + i / nch, row0, off, cnt);
    if (i >= S) mbar_wait(&empty[s], uint32_t(((i / S) - 1) & 1));
    mbar_arrive_expect_tx(&full[s], 16u * rec);
    bulk_g2s(ring + size_t(s) * stg, a.codes + (uint64_t(chunk) * a.rows_pad + uint64_t(row0)) * rec,
             16u * rec, &full[s]);
  };
  // weights do not depend on the previous kernel: first S items go out now
  if (producer && lane == 0)
    for (int i = 0; i < S && i < items; ++i) produce(i);
  griddep_launch_dependents();
  griddep_wait();

  stage_activations<FAM, MP, XDT>(a, xs, qs, tokscale, tokmax, Mc, gpr, lane, tok0);

  if (producer) {
    if (lane == 0)
      for (int i = S; i < items; ++i) produce(i);
  } else {
    const uint32_t row_bytes = uint32_t(gpr) * 128u, tok_stride = row_bytes + 16u;
#pragma unroll 1
    for (int u = warp; u < units; u += nw) {
      const int item = u >> 2, q = u & 3;
      int64_t row0;
      int toff, tcnt;
      tile_info(t_begin + item / nch, row0, toff, tcnt);
      toff -= tok0;  // row of the staged window
      const uint8_t* xb[NT];
      uint32_t gstride[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int nb = nt * 8 + g;
        const bool live = nb < tcnt;
        xb[nt] = live ? xs + size_t(toff + nb) * tok_stride + c * 32 : zblk + c * 32;
        gstride[nt] = live ? 128u : 0u;
      }
      const float* qlane = qs + toff + 2 * c;
      const int s = item % S;
      mbar_wait(&full[s], uint32_t((item / S) & 1));
      const uint8_t* st = ring + size_t(s) * stg;
      const int chunk = item % nch;
      RowCtx rc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint8_t* rr = st + (g + 8 * h) * rec;
        const uint4 pv = *reinterpret_cast<const uint4*>(rr + a.rec - 16);
        rc[h].C = (uint64_t(pv.x) | (uint64_t(pv.y) << 32)) >> 8;
        rc[h].M = pv.z;
        uint32_t step = pv.w >> 16;
        step = step > 1u ? step >> 4 : 1u;
        const uint32_t pos = step == 1u ? 0u : step == 16u ? 1u : step == 256u ? 2u : 3u;
        const uint32_t base = (0x4444u & ~(0xFu << (4u * pos))) & 0xFFFFu;
        rc[h].sel[0] = base;
        rc[h].sel[1] = base + step;
        rc[h].sel[2] = base + 2 * step;
        rc[h].sel[3] = base + 3 * step;
        rc[h].nib = *reinterpret_cast<const uint32_t*>(rr + a.rec - 32 + 4 * q);
      }
      float yacc[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) yacc[nt][i] = 0.f;
      const int G0 = chunk * kChunk + 8 * q;
      auto group = [&](int j) {
        const int G = G0 + j;
        uint32_t ua[8], ub[8];
        const uint8_t* p = st + g * rec + (8 * q + j) * 16 + 4 * c;
        const uint32_t sca = decode_units<FAM, true>(p, g, j, c, rc[0], ua);
        const uint32_t scb = decode_units<FAM, true>(p + 8 * rec, g + 8, j, c, rc[1], ub);
        const float fa = float(sca), fb = float(scb);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          // token offset may be odd (grouped experts): two scalar loads, not a float2
          const float q0 = qlane[G * MP + nt * 8], q1 = qlane[G * MP + nt * 8 + 1];
          float d[4] = {q0, q1, q0, q1};
          const uint4* src = reinterpret_cast<const uint4*>(xb[nt] + uint32_t(G) * gstride[nt]);
          const uint4 b01 = src[0], b23 = src[1];
          const uint32_t bb[8] = {b01.x, b01.y, b01.z, b01.w, b23.x, b23.y, b23.z, b23.w};
          float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t af[4] = {ua[2 * t], ub[2 * t], ua[2 * t + 1], ub[2 * t + 1]};
            if (t & 1) mma16816(e, af, bb[2 * t], bb[2 * t + 1]);
            else mma16816(d, af, bb[2 * t], bb[2 * t + 1]);
          }
          yacc[nt][0] = fmaf(fa, d[0] + e[0], yacc[nt][0]);
          yacc[nt][1] = fmaf(fa, d[1] + e[1], yacc[nt][1]);
          yacc[nt][2] = fmaf(fb, d[2] + e[2], yacc[nt][2]);
          yacc[nt][3] = fmaf(fb, d[3] + e[3], yacc[nt][3]);
        }
      };
      if (gpr - G0 >= 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) group(j);
      } else {
#pragma unroll 1
        for (int j = 0; j < gpr - G0; ++j) group(j);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this quarter no longer reads the stage
      float* pp = part + size_t(u) * kRowsT * MP;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int n0 = nt * 8 + 2 * c;
        *reinterpret_cast<float2*>(pp + g * MP + n0) = make_float2(yacc[nt][0], yacc[nt][1]);
        *reinterpret_cast<float2*>(pp + (g + 8) * MP + n0) = make_float2(yacc[nt][2], yacc[nt][3]);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ntl * kRowsT * MP; e += blockDim.x) {
    const int tl = e / (kRowsT * MP), rem = e % (kRowsT * MP);
    const int r = rem / MP, n = rem % MP;
    int64_t row0;
    int toff, tcnt;
    tile_info(t_begin + tl, row0, toff, tcnt);
    const int64_t row = row0 + r;
    if (n >= tcnt || row >= a.rows) continue;
    float v = 0.f;
    for (int ui = tl * nch * 4; ui < (tl + 1) * nch * 4; ++ui) v += part[(size_t(ui) * kRowsT + r) * MP + n];
    v *= a.super[row] * tokscale[toff - tok0 + n];
    // y: plain [M][rows]; grouped: expert-major tokens x rows_e
    const int64_t yi = GROUPED ? int64_t(toff + n) * a.rows_e + (row - (row0 - row0 % a.rows_e))
                               : int64_t(n) * a.y_ld + row;
    if (a.y_dtype == CCQ_DTYPE_F32)
      static_cast<float*>(a.y)[yi] = v;
    else
      static_cast<__nv_bfloat16*>(a.y)[yi] = __float2bfloat16_rn(v);
  }
}

// Shared-memory plan of the record variant; S = 0 when it does not apply.
struct RecCfg {
  int S;
  size_t smem;
};
inline RecCfg rec_cfg(const ccq_dev_model* m, int M, int grid, int max_smem, int ntiles_override = -1) {
  const int MP = M > 8 ? 16 : 8;
  max_smem -= 2048;  // static shared memory of the kernel (expert list)
  const int ntiles = ntiles_override >= 0 ? ntiles_override : int((m->rows + kRowsT - 1) / kRowsT);
  const int tiles_cta = (ntiles + grid - 1) / grid;
  const int items = tiles_cta * m->nch;
  const size_t stg = (size_t(16) * m->rec + 127) & ~size_t(127);
  const size_t fixed = size_t(m->gpr * 128 + 16) * M + size_t(m->gpr) * MP * 4 +
                       size_t(items) * 4 * kRowsT * MP * 4 + MP * 8 + 128 + 256;
  // S >= 3: consumer warps take every third item (12 warps x 4 quarters), so
  // with S = 2 a warp could wait on a slot still holding the item 2S before
  // its own and pass on the stale phase parity (8192 -> 28672 at M = 6).
  if (fixed + 3 * stg + size_t(items) * 16 > size_t(max_smem)) return RecCfg{0, 0};
  const int S = int(std::min<size_t>(size_t(items), (size_t(max_smem) - fixed) / (stg + 16)));
  return RecCfg{S, fixed + size_t(S) * (stg + 16)};
}

template <int NT, int XDT, bool GROUPED = false>
int launch_rec(const ccq_dev_model* m, const void* x, int M, void* y, int x_dtype, int y_dtype, int grid,
               const RecCfg& cfg, cudaStream_t s, const int32_t* offsets = nullptr, int E = 0,
               int64_t rows_e = 0) {
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
  a.ntiles = int((m->rows + kRowsT - 1) / kRowsT);
  a.x_ld = m->cols;
  a.y_ld = m->rows;
  a.xs_bytes = uint32_t((m->gpr * 128 + 16) * M);
  a.codes = m->codes;
  a.rec = m->rec;
  a.nch = m->nch;
  a.S = cfg.S;
  a.offsets = offsets;
  a.E = E;
  a.rows_e = rows_e;
  auto kern = gemv_rec206<NT, XDT, GROUPED>;
  if (int st = ensure_smem(reinterpret_cast<const void*>(kern), cfg.smem)) return st;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(unsigned(grid));
  lc.blockDim = dim3(13u * 32u);
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, kern, a);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv_rec206 launch");
}

struct Cfg {
  int warps, slots;
  size_t smem;
};

template <int FAM, int NT, int S>
Cfg plan_cfg(const ccq_dev_model* m, int M, int grid, int max_smem, int ntiles_override = -1) {
  using F = MF<FAM>;
  constexpr int MP = 8 * NT;
  constexpr int STAGE = ((kRowsT * F::BOX + kRowsT * F::SIDE) + 511) & ~511;
  max_smem -= 2048;  // static shared memory (grouped expert list)
  const int ntiles = ntiles_override >= 0 ? ntiles_override : int((m->rows + kRowsT - 1) / kRowsT);
  const int nblk = int((m->gpr + F::BLK - 1) / F::BLK);
  const int tiles_cta = (ntiles + grid - 1) / grid;
  static const int env_w = std::getenv("CCQ_MMA_WARPS") ? std::atoi(std::getenv("CCQ_MMA_WARPS")) : 0;
  for (int warps = env_w ? env_w : 16; warps >= 4; warps -= 4) {
    const int items = tiles_cta * nblk;
    const int per_warp = (items + warps - 1) / warps;
    const int slots = per_warp / nblk + 2;
    const size_t smem = size_t(warps) * S * STAGE + size_t(m->gpr * 128 + 16) * M + size_t(m->gpr) * MP * 4 +
                        size_t(warps) * slots * kRowsT * MP * 4 + MP * 8 + 256 + size_t(warps) * S * 8 + 8 + 1024 + 64;
    if (smem <= size_t(max_smem)) return Cfg{warps, slots, smem};
  }
  return Cfg{0, 0, 0};
}

template <int FAM, int NT, int S, int XDT, bool P2, bool GROUPED = false>
int launch_chunk(const ccq_dev_model* m, const CUtensorMap& tmc, const CUtensorMap& tms, const void* x,
                 int M, void* y, int x_dtype, int y_dtype, int grid, const Cfg& cfg, cudaStream_t s,
                 const int32_t* offsets = nullptr, int E = 0, int64_t rows_e = 0) {
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
  a.nblk = int((m->gpr + MF<FAM>::BLK - 1) / MF<FAM>::BLK);
  a.ntiles = int((m->rows + kRowsT - 1) / kRowsT);
  a.slots = cfg.slots;
  a.x_ld = m->cols;
  a.y_ld = m->rows;
  a.xs_bytes = uint32_t((m->gpr * 128 + 16) * M);
  a.offsets = offsets;
  a.E = E;
  a.rows_e = rows_e;
  auto kern = gemv_mma<FAM, NT, S, XDT, P2, GROUPED>;
  if (int st = ensure_smem(reinterpret_cast<const void*>(kern), cfg.smem)) return st;
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

template <int FAM, bool P2>
int launch_fam_mma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                   cudaStream_t s) {
  using F = MF<FAM>;
  constexpr int S = 4;
  CUtensorMap tmc{}, tms{};
  int st = make_map_2d(&tmc, CU_TENSOR_MAP_DATA_TYPE_UINT8, m->codes, m->rec, uint64_t(m->nch) * m->rows_pad,
                       m->rec, F::BOX, kRowsT,
                       FAM == kF206 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE);
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
  int max_smem = max_smem_optin(dev);
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
        case CCQ_DTYPE_BF16: st = launch_chunk<FAM, 2, S, CCQ_DTYPE_BF16, P2>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        default: st = launch_chunk<FAM, 2, S, CCQ_DTYPE_F16, P2>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s);
      }
    } else {
      switch (x_dtype) {
        case CCQ_DTYPE_BF16: st = launch_chunk<FAM, 1, S, CCQ_DTYPE_BF16, P2>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s); break;
        default: st = launch_chunk<FAM, 1, S, CCQ_DTYPE_F16, P2>(m, tmc, tms, xc, chunk, yc, x_dtype, y_dtype, grid, cfg, s);
      }
    }
    if (st != CCQ_OK) return st;
    m0 += chunk;
  }
  return CCQ_OK;
}

}  // namespace

// True when all M tokens fit one launch with >= 8 warps per CTA (no weight re-streaming).
bool gemv_mma_fits(const ccq_dev_model* m, int64_t M) {
  if (M < 1 || M > 8 || !gemv_mma_supported(m, M)) return false;
  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = max_smem_optin(dev);
  const int ntiles = int((m->rows + 15) / 16);
  const int grid = std::min(num_sms(dev), ntiles);
  Cfg cfg{};
  switch (m->family) {
    case kF275: cfg = plan_cfg<kF275, 1, 4>(m, int(M), grid, max_smem); break;
    case kF25: cfg = plan_cfg<kF25, 1, 4>(m, int(M), grid, max_smem); break;
    default: cfg = plan_cfg<kF206, 1, 4>(m, int(M), grid, max_smem); break;
  }
  return cfg.warps >= 8;
}

// Grouped experts on the TMA-box tensor-pipe GEMV (any family; partial sums
// are O(warps), so any number of routed tiles fits).
template <int FAM, bool P2>
int launch_grouped_box(const ccq_dev_model* st, int E, int64_t rows_e, const int32_t* offsets_dev, int ntiles,
                       int wmax, const void* x, int x_dtype, void* y, int y_dtype, cudaStream_t s) {
  using F = MF<FAM>;
  constexpr int S = 4;
  CUtensorMap tmc{}, tms{};
  int rc = make_map_2d(&tmc, CU_TENSOR_MAP_DATA_TYPE_UINT8, st->codes, st->rec, uint64_t(st->nch) * st->rows_pad,
                       st->rec, F::BOX, kRowsT, FAM == kF206 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc != CCQ_OK) return rc;
  if constexpr (F::SIDE > 0) {
    rc = make_map_2d(&tms, CU_TENSOR_MAP_DATA_TYPE_UINT8, st->codes + st->cgb, F::SIDE,
                     uint64_t(st->nch) * st->rows_pad, st->rec, F::SIDE, kRowsT, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc != CCQ_OK) return rc;
  } else {
    tms = tmc;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = max_smem_optin(dev);
  const int grid = std::min(num_sms(dev), ntiles);
  const Cfg cfg = wmax > 8 ? plan_cfg<FAM, 2, S>(st, wmax, grid, max_smem, ntiles)
                           : plan_cfg<FAM, 1, S>(st, wmax, grid, max_smem, ntiles);
  if (cfg.warps < 8) return 1;  // the expert compaction needs >= 256 threads
  if (wmax > 8)
    return x_dtype == CCQ_DTYPE_BF16
               ? launch_chunk<FAM, 2, S, CCQ_DTYPE_BF16, P2, true>(st, tmc, tms, x, wmax, y, x_dtype, y_dtype, grid, cfg, s, offsets_dev, E, rows_e)
               : launch_chunk<FAM, 2, S, CCQ_DTYPE_F16, P2, true>(st, tmc, tms, x, wmax, y, x_dtype, y_dtype, grid, cfg, s, offsets_dev, E, rows_e);
  return x_dtype == CCQ_DTYPE_BF16
             ? launch_chunk<FAM, 1, S, CCQ_DTYPE_BF16, P2, true>(st, tmc, tms, x, wmax, y, x_dtype, y_dtype, grid, cfg, s, offsets_dev, E, rows_e)
             : launch_chunk<FAM, 1, S, CCQ_DTYPE_F16, P2, true>(st, tmc, tms, x, wmax, y, x_dtype, y_dtype, grid, cfg, s, offsets_dev, E, rows_e);
}

// Kernel (d) for decode batches: all routed (expert, token) rows in ONE
// tensor-pipe GEMV launch over the tiles of the experts that have tokens.
// Returns 1 when not applicable (caller falls back to the grouped GEMM).
int launch_grouped_gemv(const ccq_dev_model* st, int E, int64_t rows_e, const int32_t* offsets_dev,
                        const int32_t* offsets_host, int64_t T, const void* x, int x_dtype, void* y,
                        int y_dtype, cudaStream_t s) {
  if (T < 1 || E > 256 || rows_e % kRowsT != 0 || st->geo.group_size != 64 || st->cols % 64 != 0 ||
      x_dtype == CCQ_DTYPE_F32 || (reinterpret_cast<uintptr_t>(x) & 15u) || !offsets_dev ||
      std::getenv("CCQ_NO_GROUPED_GEMV"))
    return 1;
  const bool rec_ok = st->family == kF206 && st->plan_pos_min >= 1 && st->rec == uint32_t(st->cgb + 32) &&
                      !std::getenv("CCQ_NO_REC");
  int nhit = 0;
  for (int e = 0; e < E; ++e) nhit += offsets_host[e + 1] > offsets_host[e] ? 1 : 0;
  if (nhit == 0) return CCQ_OK;
  const int tpe = int(rows_e / kRowsT);
  const int ntiles = nhit * tpe;
  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = max_smem_optin(dev);
  const int grid = std::min(num_sms(dev), ntiles);
  // the largest token window any CTA stages (same partition as the kernel)
  std::vector<int> hits;
  for (int e = 0; e < E; ++e)
    if (offsets_host[e + 1] > offsets_host[e]) hits.push_back(e);
  int wmax = 1;
  for (int b = 0; b < grid; ++b) {
    const int tb = int(int64_t(b) * ntiles / grid), te = int(int64_t(b + 1) * ntiles / grid);
    if (te <= tb) continue;
    const int e0 = hits[tb / tpe], e1 = hits[(te - 1) / tpe];
    wmax = std::max(wmax, offsets_host[e1 + 1] - offsets_host[e0]);
  }
  if (wmax > 16) return 1;  // some expert (or CTA window) has too many tokens: grouped GEMM
  const RecCfg rc = rec_ok ? rec_cfg(st, wmax, grid, max_smem, ntiles) : RecCfg{0, 0};
  if (rc.S <= 0) {
    switch (st->family) {
      case kF275: return launch_grouped_box<kF275, false>(st, E, rows_e, offsets_dev, ntiles, wmax, x, x_dtype, y, y_dtype, s);
      case kF25: return launch_grouped_box<kF25, false>(st, E, rows_e, offsets_dev, ntiles, wmax, x, x_dtype, y, y_dtype, s);
      default:
        return st->plan_pos_min >= 1
                   ? launch_grouped_box<kF206, true>(st, E, rows_e, offsets_dev, ntiles, wmax, x, x_dtype, y, y_dtype, s)
                   : launch_grouped_box<kF206, false>(st, E, rows_e, offsets_dev, ntiles, wmax, x, x_dtype, y, y_dtype, s);
    }
  }
  if (wmax > 8)
    return x_dtype == CCQ_DTYPE_BF16
               ? launch_rec<2, CCQ_DTYPE_BF16, true>(st, x, wmax, y, x_dtype, y_dtype, grid, rc, s, offsets_dev, E, rows_e)
               : launch_rec<2, CCQ_DTYPE_F16, true>(st, x, wmax, y, x_dtype, y_dtype, grid, rc, s, offsets_dev, E, rows_e);
  return x_dtype == CCQ_DTYPE_BF16
             ? launch_rec<1, CCQ_DTYPE_BF16, true>(st, x, wmax, y, x_dtype, y_dtype, grid, rc, s, offsets_dev, E, rows_e)
             : launch_rec<1, CCQ_DTYPE_F16, true>(st, x, wmax, y, x_dtype, y_dtype, grid, rc, s, offsets_dev, E, rows_e);
}

int mma_min_tokens() {
  const char* e = std::getenv("CCQ_FORCE_MMA");
  return (e && e[0] == '1') ? 1 : kMmaMinTokens;
}

bool gemv_mma_supported(const ccq_dev_model* m, int64_t M) {
  (void)M;
  // activations arrive by 16-byte bulk copies: need 16-B aligned rows
  if (m->geo.group_size != 64 || m->cols % 64 != 0 || m->cols == 0) return false;
  if (std::getenv("CCQ_GEMV_STREAM")) return false;  // debug: force the CUDA-core kernel
  return true;
}

int launch_gemv_mma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                    cudaStream_t s) {
  if (x_dtype == CCQ_DTYPE_F32 || (reinterpret_cast<uintptr_t>(x) & 15u))
    return fail(CCQ_ERR_CONFIG, "gemv_mma needs 16-byte aligned bf16/f16 activations");
  switch (m->family) {
    case kF275: return launch_fam_mma<kF275, false>(m, x, x_dtype, M, y, y_dtype, s);
    case kF25: return launch_fam_mma<kF25, false>(m, x, x_dtype, M, y, y_dtype, s);
    default: {
      if (m->plan_pos_min >= 1 && M <= 16 && m->rec == uint32_t(m->cgb + 32) && !std::getenv("CCQ_NO_REC")) {
        int dev = 0;
        cudaGetDevice(&dev);
        int max_smem = max_smem_optin(dev);
        const int grid = std::min<int>(num_sms(dev), int((m->rows + kRowsT - 1) / kRowsT));
        const RecCfg rc = rec_cfg(m, int(M), grid, max_smem);
        if (rc.S > 0) {
          if (M > 8)
            return x_dtype == CCQ_DTYPE_BF16 ? launch_rec<2, CCQ_DTYPE_BF16>(m, x, int(M), y, x_dtype, y_dtype, grid, rc, s)
                                             : launch_rec<2, CCQ_DTYPE_F16>(m, x, int(M), y, x_dtype, y_dtype, grid, rc, s);
          return x_dtype == CCQ_DTYPE_BF16 ? launch_rec<1, CCQ_DTYPE_BF16>(m, x, int(M), y, x_dtype, y_dtype, grid, rc, s)
                                           : launch_rec<1, CCQ_DTYPE_F16>(m, x, int(M), y, x_dtype, y_dtype, grid, rc, s);
        }
      }
      return m->plan_pos_min >= 1 ? launch_fam_mma<kF206, true>(m, x, x_dtype, M, y, y_dtype, s)
                                  : launch_fam_mma<kF206, false>(m, x, x_dtype, M, y, y_dtype, s);
    }
  }
}

}  // namespace ccqb

#ifdef CCQ_GEMV_TRACE
extern "C" int ccq_trace_dump_mma(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ccqb::g_mtrace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif
