// Kernel (b), round 2: the small-batch (M = 1..8) decode-GEMV on the warp
// tensor pipe, built around shared-memory-resident weights.
//
// Reference: ccq::gemv / gemv_batch (kernels.cpp:124-187): y = W x with the
// weights decoded group by group (decode_group, kernels.cpp:60-93) and
// accumulated in double.  Here a 16-row x 64-weight tile of one group is
// decoded straight from the packed bytes into exact f16 "magic" values
// (1024 + field * 2^p) and multiplied with mma.sync.m16n8k16 (f32
// accumulate) against the activations, which are staged ONCE per CTA as
// ready-made B fragments (f16x2, per-token power-of-two scaled).  A token
// per MMA column means M = 1..8 cost the same decode.
//
// Why this shape (profiles/r02_*):
//   * x lives in shared memory as broadcast B fragments (8 registers per
//     group instead of 64 floats per lane), so a lane keeps ~60 registers
//     and 2 CTAs (16 warps) fit an SM;
//   * two f16 fields per LOP3 (vs one f32 field per LOP3 on the CUDA-core
//     path) halves the ALU work of the decode, which bounds 2.06 on B200;
//   * weights do not depend on the previous kernel: every CTA bulk-copies its
//     first R (16-row, 32-group) stages BEFORE griddepcontrol.wait, and with
//     two CTAs per SM the next layer's stream overlaps this layer's decode.
//
// Work split: CTA b owns 16-row tiles [b*T/G, (b+1)*T/G); a unit is (tile,
// K chunk) = 16 contiguous device records = one bulk copy into a ring stage;
// each unit is cut into 4 slices of 8 groups processed by 4 warps; per-slice
// partials are summed in a fixed order at the end (deterministic, no atomics
// on data).  A ring stage is refilled by the last warp that finishes it.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "ccq_internal.hpp"
#include "ptx.cuh"

namespace ccqb {
namespace {

#ifdef CCQ_GEMV_TRACE
}  // namespace
__device__ unsigned long long g_trace_h[8192 * 8];
namespace {
__device__ __forceinline__ unsigned long long gtime_h() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HTRACE(slot)                                                     \
  if (lane == 0) {                                                       \
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); \
    if (gwid < 8192) g_trace_h[gwid * 8 + (slot)] = gtime_h();           \
  }
#else
#define HTRACE(slot)
#endif

constexpr int kSlices = 4;            // slices per unit (8 groups each)
constexpr int kGroupsPerSlice = kChunk / kSlices;

__device__ __forceinline__ uint32_t lop_or(uint32_t v, uint32_t mask, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(magic));
  return d;
}

__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------------------
// Family decode: lane t of a row's 64-weight group yields 8 f16x2 A values
// (16 weights) for the 4 k-steps; unit_wp() gives (weight, p) of each half so
// the staged B fragments match.  Register j of lane t feeds k-step j/2 as a0
// (j even) or a2 (j odd).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lds32(const void* p) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)));
  return v;
}
__device__ __forceinline__ uint2 lds64(const void* p) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_addr(p)));
  return v;
}

template <int FAM>
struct HF;

// 2.06: lane t takes stored bytes 4t..4t+3 (one 32-bit word).  Codes of two
// bytes are packed c_a | c_b << 16; W and W >> 6 give all 8 fields with 4
// LOP3 (mask 0x003F003F -> p = 0, 0x01F801F8 -> p = 3).
template <>
struct HF<kF206> {
  static constexpr int PB = 16, ZP = 32;
  // register j: pair = j / 4 (bytes 2*pair, 2*pair+1), kind = j % 4
  //   kind 0: shift 0 (slot 3) p 0; 1: shift 3 (slot 2) p 3;
  //   kind 2: shift 6 (slot 1) p 0; 3: shift 9 (slot 0) p 3
  __host__ __device__ static constexpr int weight(int t, int j, int half) {
    const int pair = j / 4, kind = j % 4;
    const int slot = 3 - kind;
    return 16 * t + 4 * (2 * pair + half) + slot;
  }
  __host__ __device__ static constexpr int p(int t, int j, int half) { return (j % 4) & 1 ? 3 : 0; }
  __device__ __forceinline__ static void decode(uint32_t w, const uint32_t (&sel)[4], uint64_t C, uint32_t M,
                                                uint32_t mg, uint32_t (&u)[8]) {
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
      const uint32_t qa = prmt(w, 0u, sel[2 * pr]), qb = prmt(w, 0u, sel[2 * pr + 1]);
      const uint32_t ha = uint32_t((uint64_t(qa) * M + C) >> 32);
      const uint32_t hb = uint32_t((uint64_t(qb) * M + C) >> 32);
      const uint32_t W = prmt(ha, hb, 0x6521u);  // code_a | code_b << 16 (codes at [8,23) of hi)
      const uint32_t W6 = W >> 6;
      u[4 * pr + 0] = lop_or(W, 0x003F003Fu, mg);
      u[4 * pr + 1] = lop_or(W, 0x01F801F8u, mg);
      u[4 * pr + 2] = lop_or(W6, 0x003F003Fu, mg);
      u[4 * pr + 3] = lop_or(W6, 0x01F801F8u, mg);
    }
  }
};

// 2.75 / 2.5: the unit order of the tcgen05 GEMM's decoders (unit_wp,
// ccq_internal.hpp; gemm_sm100.cu decode_gemm_275 / decode_gemm_25) without
// the scale multiply - the group scale is applied to the accumulator.
template <>
struct HF<kF275> {
  static constexpr int PB = 22, ZP = 8;
  __host__ __device__ static constexpr int weight(int t, int j, int h) { return unit_wp(kF275, t, j, h).w; }
  __host__ __device__ static constexpr int p(int t, int j, int h) { return unit_wp(kF275, t, j, h).p; }
  // lane t: bytes 5t..5t+4 of the group at g (2-byte aligned) and its bytes
  // 20 / 21 (the extra field, and the scale in byte 21's low nibble)
  __device__ __forceinline__ static uint32_t decode(const uint8_t* g, int t, uint32_t sel6, uint32_t mk6,
                                                    uint32_t mg, uint32_t (&u)[8]) {
    const uint8_t* p = g + 5 * t;
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(p) & 3u);
    const uint8_t* pa = p - mis;
    const uint32_t W0 = lds32(pa), W1 = lds32(pa + 4);
    const uint32_t lo = __funnelshift_r(W0, W1, 8u * mis);
    const uint32_t hi = W1 >> (8u * mis);
    const uint8_t* q = g + 20;
    const uint32_t mq = uint32_t(reinterpret_cast<uintptr_t>(q) & 3u);
    const uint32_t e = lds32(q - mq) >> (8u * mq);  // byte 20 at [0,8), byte 21 at [8,16)
    const uint32_t p0 = prmt(lo, 0u, 0x1100u), p1 = prmt(lo, 0u, 0x3322u);
    u[0] = lop_or(p0, 0x000F000Fu, mg);
    u[1] = lop_or(p0, 0x003C003Cu, mg);
    u[2] = lop_or(p0, 0x00F000F0u, mg);
    u[3] = lop_or(p1, 0x000F000Fu, mg);
    u[4] = lop_or(p1, 0x003C003Cu, mg);
    u[5] = lop_or(p1, 0x00F000F0u, mg);
    u[6] = lop_or(prmt(hi, e, sel6), mk6, mg);
    u[7] = lop_or(prmt(hi, 0u, 0x0000u), 0x000F003Cu, mg);
    return (e >> 8) & 0xFu;
  }
};

template <>
struct HF<kF25> {
  static constexpr int PB = 20, ZP = 4;
  __host__ __device__ static constexpr int weight(int t, int j, int h) { return unit_wp(kF25, t, j, h).w; }
  __host__ __device__ static constexpr int p(int t, int j, int h) { return unit_wp(kF25, t, j, h).p; }
  // lane t: stored words 2t, 2t+1 (one 32-bit word) and words 8, 9 (the
  // extra fields, and the 13-bit scale in word 9)
  __device__ __forceinline__ static uint32_t decode(const uint8_t* g, int t, uint32_t sel7, uint32_t mk7,
                                                    uint32_t mg, uint32_t (&u)[8]) {
    const uint32_t v = lds32(g + 4 * t), w4 = lds32(g + 16);
    const uint32_t sv = v >> 9;
    u[0] = lop_or(v, 0x00070007u, mg);
    u[1] = lop_or(v, 0x001C001Cu, mg);
    u[2] = lop_or(v, 0x00700070u, mg);
    u[3] = lop_or(v, 0x01C001C0u, mg);
    u[4] = lop_or(sv, 0x00070007u, mg);
    u[5] = lop_or(sv, 0x001C001Cu, mg);
    u[6] = lop_or(sv, 0x00700070u, mg);
    u[7] = lop_or(prmt(w4, w4, sel7), mk7, mg);
    return (w4 >> 16) & 0x1FFFu;
  }
};

struct HmmaArgs {
  DevLayout L;
  const void* x;
  void* y;
  int x_dtype, y_dtype;
  int M;                       // tokens (<= MT)
  int64_t x_stride, y_stride;  // elements between token rows
  int ntiles;                  // 16-row tiles of the model
  int R;                       // ring stages
  int units_max;               // per CTA
  int gpr_pad;                 // nch * 32
};

// sigma = 2^(15 - e) for max|x| in [2^(e-1), 2^e): max|x| sigma in [2^14, 2^15)
__device__ __forceinline__ float sigma_of(unsigned maxbits) {
  const float mx = __uint_as_float(maxbits);
  int e = 0;
  if (mx > 0.f) {
    frexpf(mx, &e);
    e = max(e, -100);
  }
  return ldexpf(1.f, 15 - e);
}

template <int XDT>
__device__ __forceinline__ float ldx(const void* x, int64_t i) {
  if constexpr (XDT == CCQ_DTYPE_BF16) {
    return __uint_as_float(uint32_t(static_cast<const uint16_t*>(x)[i]) << 16);
  } else {
    return __half2float(__ushort_as_half(static_cast<const uint16_t*>(x)[i]));
  }
}

template <int FAM, int MT, int XDT>
__global__ void __launch_bounds__(1024, 1) gemv_hmma(HmmaArgs a) {
  using F = HF<FAM>;
  constexpr int CGB = (32 * F::PB + 15) & ~15;
  constexpr int REC = CGB + (FAM == kF206 ? 32 : 0);
  constexpr int SB = 16 * REC;
  extern __shared__ __align__(128) uint8_t smem[];
  const DevLayout& L = a.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nch = L.nch, R = a.R;
  const int tile0 = int(int64_t(blockIdx.x) * a.ntiles / gridDim.x);
  const int tile1 = int(int64_t(blockIdx.x + 1) * a.ntiles / gridDim.x);
  const int nunits = (tile1 - tile0) * nch;

  // shared memory carve-up
  uint32_t* xf = reinterpret_cast<uint32_t*>(smem);                 // [MT][gpr_pad][4][8] f16x2
  float* qv = reinterpret_cast<float*>(xf + size_t(MT) * a.gpr_pad * 32);  // [gpr_pad][MT]
  float* part = qv + size_t(a.gpr_pad) * (MT < 4 ? 4 : MT);          // [units_max][4][16][MT]
  unsigned* smax = reinterpret_cast<unsigned*>(part + size_t(a.units_max) * kSlices * 16 * MT);  // [8]
  int* cnt = reinterpret_cast<int*>(smax + 8);                      // [R] slice arrivals
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(cnt + R) + 7) & ~uintptr_t(7));  // [R]
  uint8_t* ring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(full + R) + 127) & ~uintptr_t(127));  // [R][SB]

  HTRACE(0);
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int j) {  // unit j -> stage j % R
    const int s = j % R;
    const int tile = tile0 + j / nch, c = j % nch;
    mbar_arrive_expect_tx(&full[s], SB);
    bulk_g2s_evict_first(ring + size_t(s) * SB, L.record(c, int64_t(tile) * 16), SB, &full[s], pol);
  };
  // 1. Weights first (independent of the previous kernel).
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      mbar_init(&full[s], 1);
      cnt[s] = 0;
    }
    for (int m = 0; m < 8; ++m) smax[m] = 0u;
    fence_mbar_init();
    const int pre = nunits < R ? nunits : R;
    for (int j = 0; j < pre; ++j) issue(j);
  }
  griddep_launch_dependents();
  griddep_wait();  // x (and y) belong to the previous kernel until here
  HTRACE(1);
  __syncthreads();  // barrier / smax init visible

  // 2. Activations -> per-token power-of-two scale sigma (max|x| sigma in
  //    [2^14, 2^15)) -> f16x2 B fragments and -Q, Q = sum (1024 + zp 2^p) b.
  //    Item (m, g, t) = the 16 activations 64 g + 16 t .. + 15 of token m
  //    (two 16-byte loads); items are token-major and a token spans a whole
  //    number of warps, so the max is a warp reduction + one shared atomic.
  const int items = MT * a.gpr_pad * 4;
  auto load16 = [&](int it, uint4& v0, uint4& v1) -> bool {
    const int t4 = it & 3, g = (it >> 2) % a.gpr_pad, m = (it >> 2) / a.gpr_pad;
    if (m >= a.M || int64_t(g) * 64 >= L.cols) return false;
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + m * a.x_stride +
                                                    int64_t(g) * 64 + 16 * t4);
    v0 = __ldg(p);
    v1 = __ldg(p + 1);
    return true;
  };
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
    load16(it, v0, v1);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    float mx = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float lo, hi;
      if constexpr (XDT == CCQ_DTYPE_BF16) {
        lo = __uint_as_float(w[i] << 16);
        hi = __uint_as_float(w[i] & 0xFFFF0000u);
      } else {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        lo = f.x;
        hi = f.y;
      }
      mx = fmaxf(mx, fmaxf(fabsf(lo), fabsf(hi)));
    }
    const unsigned wm = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
    if (lane == 0) atomicMax(&smax[(it >> 2) / a.gpr_pad], wm);
  }
  __syncthreads();
  HTRACE(2);
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int t4 = it & 3, g = (it >> 2) % a.gpr_pad, m = (it >> 2) / a.gpr_pad;
    const bool ok = m < a.M && int64_t(g) * 64 < L.cols;
    const float sig = ok ? sigma_of(smax[m]) : 0.f;
    uint32_t r[8];
    float q = 0.f;
    const uint4* px = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.x) + (ok ? m * a.x_stride : 0) +
                                                     (ok ? int64_t(g) * 64 : 0));
    if constexpr (FAM == kF206) {
      // lane t's 16 weights are 16t .. 16t+15 for every t: uniform code
      float xv[16];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ok) v = __ldg(px + 2 * t4 + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if constexpr (XDT == CCQ_DTYPE_BF16) {
            xv[8 * i + 2 * k] = __uint_as_float(w[k] << 16);
            xv[8 * i + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
          } else {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
            xv[8 * i + 2 * k] = f.x;
            xv[8 * i + 2 * k + 1] = f.y;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p0 = F::p(0, j, 0), p1 = F::p(0, j, 1);
        const __half2 h = __floats2half2_rn(xv[F::weight(0, j, 0)] * sig * (1.f / float(1 << p0)),
                                            xv[F::weight(0, j, 1)] * sig * (1.f / float(1 << p1)));
        r[j] = *reinterpret_cast<const uint32_t*>(&h);
        const float2 b = __half22float2(h);
        q = fmaf(1024.f + float(F::ZP) * float(1 << p0), b.x, fmaf(1024.f + float(F::ZP) * float(1 << p1), b.y, q));
      }
    } else {
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) {
      if (tt != t4) continue;
      // only the 16-byte pieces of the group holding lane tt's 16 weights
      float xv[64];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bool need = false;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          for (int h = 0; h < 2; ++h) need |= F::weight(tt, j, h) / 8 == i;
        if (!need) continue;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ok) v = __ldg(px + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if constexpr (XDT == CCQ_DTYPE_BF16) {
            xv[8 * i + 2 * k] = __uint_as_float(w[k] << 16);
            xv[8 * i + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
          } else {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
            xv[8 * i + 2 * k] = f.x;
            xv[8 * i + 2 * k + 1] = f.y;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p0 = F::p(tt, j, 0), p1 = F::p(tt, j, 1);
        const __half2 h = __floats2half2_rn(xv[F::weight(tt, j, 0)] * sig * (1.f / float(1 << p0)),
                                            xv[F::weight(tt, j, 1)] * sig * (1.f / float(1 << p1)));
        r[j] = *reinterpret_cast<const uint32_t*>(&h);
        const float2 b = __half22float2(h);
        q = fmaf(1024.f + float(F::ZP) * float(1 << p0), b.x, fmaf(1024.f + float(F::ZP) * float(1 << p1), b.y, q));
      }
    }
    }
    uint4* dst = reinterpret_cast<uint4*>(xf + ((size_t(m) * a.gpr_pad + g) * 4 + t4) * 8);
    dst[0] = make_uint4(r[0], r[1], r[2], r[3]);
    dst[1] = make_uint4(r[4], r[5], r[6], r[7]);
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    if (t4 == 0) {
      if constexpr (MT == 1) reinterpret_cast<float4*>(qv)[g] = make_float4(-q, -q, -q, -q);
      else qv[size_t(g) * MT + m] = -q;
    }
  }
  __syncthreads();  // also publishes the barrier init to every warp
  HTRACE(3);

  // 3. Slices: warp w takes items w, w + nw, ...; item i = (unit i / 4, slice i % 4).
  const int g8 = lane >> 2, t = lane & 3;
  const int tok = MT == 1 ? 0 : (g8 < a.M ? g8 : 0);  // B column of this lane
  uint32_t mg;
  asm volatile("mov.b32 %0, 0x64006400;" : "=r"(mg));
  // lane-dependent selector / mask of the last unit (2.75: unit 6, 2.5: unit 7)
  uint32_t xsel = 0, xmk = 0;
  if constexpr (FAM == kF275) {
    const uint32_t eb = 4u + (t == 3 ? 1u : 0u);
    const uint32_t me = t == 0 ? 0xF0u : t == 1 ? 0x3Cu : t == 2 ? 0x0Fu : 0xF0u;
    xsel = (eb << 12) | (eb << 8);
    xmk = 0x000000F0u | (me << 16);
  } else if constexpr (FAM == kF25) {
    xsel = t == 0 ? 0x1010u : t == 1 ? 0x1010u : t == 2 ? 0x1111u : 0x3311u;
    xmk = t == 0 ? 0x001C0007u : t == 1 ? 0x01C00070u : t == 2 ? 0x0038000Eu : 0x00E000E0u;
  }
  const int nitems = nunits * kSlices;
#pragma unroll 1
  for (int i = warp; i < nitems; i += nw) {
    const int j = i / kSlices, sl = i % kSlices;
    const int s = j % R;
    const int c = j % nch;
    mbar_wait(&full[s], uint32_t((j / R) & 1));
#ifdef CCQ_GEMV_TRACE
    if (i == warp) { HTRACE(4); }
#endif
    const uint8_t* st = ring + size_t(s) * SB;
    const uint8_t* r0 = st + size_t(g8) * REC;
    const uint8_t* r1 = st + size_t(g8 + 8) * REC;
    // per-row widening plans (2.06)
    uint64_t C0 = 0, C1 = 0;
    uint32_t M0 = 0, M1 = 0, sel0[4] = {0, 0, 0, 0}, sel1[4] = {0, 0, 0, 0};
    if constexpr (FAM == kF206) {
      const uint4 p0 = lds128(r0 + CGB + 16), p1 = lds128(r1 + CGB + 16);
      C0 = uint64_t(p0.x) | (uint64_t(p0.y) << 32);
      M0 = p0.z;
      C1 = uint64_t(p1.x) | (uint64_t(p1.y) << 32);
      M1 = p1.z;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        sel0[b] = (p0.w & 0xFFFFu) + uint32_t(b) * (p0.w >> 16);
        sel1[b] = (p1.w & 0xFFFFu) + uint32_t(b) * (p1.w >> 16);
      }
    }
    uint32_t nib0 = 0, nib1 = 0;
    if constexpr (FAM == kF206) {
      nib0 = lds32(r0 + CGB + 4 * sl);
      nib1 = lds32(r1 + CGB + 4 * sl);
    }
    float yacc[4] = {0.f, 0.f, 0.f, 0.f};
    const int gbase = c * kChunk + sl * kGroupsPerSlice;
#pragma unroll 2
    for (int gi = 0; gi < kGroupsPerSlice; ++gi) {
      const int gl = sl * kGroupsPerSlice + gi;  // group within the chunk
      const int g = gbase + gi;
      const uint4 b01 = lds128(xf + ((size_t(tok) * a.gpr_pad + g) * 4 + t) * 8);
      const uint4 b23 = lds128(xf + ((size_t(tok) * a.gpr_pad + g) * 4 + t) * 8 + 4);
      float d[4];
      if constexpr (MT == 1) {
        const uint4 qq = lds128(qv + size_t(g) * 4);
        d[0] = __uint_as_float(qq.x);
        d[1] = __uint_as_float(qq.y);
        d[2] = __uint_as_float(qq.z);
        d[3] = __uint_as_float(qq.w);
      } else {
        const int tc = 2 * t < MT ? 2 * t : 0;
        const uint2 qq = lds64(qv + size_t(g) * MT + tc);
        d[0] = d[2] = __uint_as_float(qq.x);
        d[1] = d[3] = __uint_as_float(qq.y);
      }
      uint32_t u0[8], u1[8];
      float sc0, sc1;
      if constexpr (FAM == kF206) {
        const uint32_t w0 = lds32(r0 + gl * F::PB + 4 * t);
        const uint32_t w1 = lds32(r1 + gl * F::PB + 4 * t);
        F::decode(w0, sel0, C0, M0, mg, u0);
        F::decode(w1, sel1, C1, M1, mg, u1);
        sc0 = float((nib0 >> (4 * gi)) & 0xFu);
        sc1 = float((nib1 >> (4 * gi)) & 0xFu);
      } else {
        sc0 = float(F::decode(r0 + gl * F::PB, t, xsel, xmk, mg, u0));
        sc1 = float(F::decode(r1 + gl * F::PB, t, xsel, xmk, mg, u1));
      }
      // two independent accumulator chains (k-steps 0,1 and 2,3)
      float e[4] = {0.f, 0.f, 0.f, 0.f};
      hmma(d, u0[0], u1[0], u0[1], u1[1], b01.x, b01.y);
      hmma(e, u0[4], u1[4], u0[5], u1[5], b23.x, b23.y);
      hmma(d, u0[2], u1[2], u0[3], u1[3], b01.z, b01.w);
      hmma(e, u0[6], u1[6], u0[7], u1[7], b23.z, b23.w);
      d[0] += e[0];
      d[2] += e[2];
      if constexpr (MT > 1) {
        d[1] += e[1];
        d[3] += e[3];
      }
      yacc[0] = fmaf(sc0, d[0], yacc[0]);
      yacc[2] = fmaf(sc1, d[2], yacc[2]);
      if constexpr (MT > 1) {
        yacc[1] = fmaf(sc0, d[1], yacc[1]);
        yacc[3] = fmaf(sc1, d[3], yacc[3]);
      }
    }
    // release the stage; the last of its 4 slices refills it
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int prev = atomicAdd(&cnt[s], 1);
      if (prev == kSlices - 1) {
        cnt[s] = 0;
        if (j + R < nunits) issue(j + R);
      }
    }
    // partials: rows g8, g8 + 8, tokens 2t, 2t + 1
    float* pp = part + (size_t(j) * kSlices + sl) * 16 * MT;
    if (2 * t < MT) {
      pp[g8 * MT + 2 * t] = yacc[0];
      pp[(g8 + 8) * MT + 2 * t] = yacc[2];
    }
    if (2 * t + 1 < MT) {
      pp[g8 * MT + 2 * t + 1] = yacc[1];
      pp[(g8 + 8) * MT + 2 * t + 1] = yacc[3];
    }
  }
  HTRACE(5);
  __syncthreads();
  // 4. Fixed-order sum over (chunk, slice); super scale and 1 / sigma.
  const int nrows16 = (tile1 - tile0) * 16;
  for (int e = threadIdx.x; e < nrows16 * a.M; e += blockDim.x) {
    const int rl = e / a.M, m = e % a.M;
    const int64_t row = int64_t(tile0) * 16 + rl;
    if (row >= L.rows) continue;
    const int tl = rl / 16, rr = rl % 16;
    float v = 0.f;
    for (int cc = 0; cc < nch; ++cc) {
      const float* pp = part + size_t(tl * nch + cc) * kSlices * 16 * MT;
#pragma unroll
      for (int sl = 0; sl < kSlices; ++sl) v += pp[(sl * 16 + rr) * MT + m];
    }
    v = v * L.super[row] / sigma_of(smax[m]);
    const int64_t yi = int64_t(m) * a.y_stride + row;
    if (a.y_dtype == CCQ_DTYPE_F32) static_cast<float*>(a.y)[yi] = v;
    else static_cast<__nv_bfloat16*>(a.y)[yi] = __float2bfloat16_rn(v);
  }
  HTRACE(6);
#ifdef CCQ_GEMV_TRACE
  if (lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const int gwid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gwid < 8192) g_trace_h[gwid * 8 + 7] = smid;
  }
#endif
}

int half_sm_budget(int dev) {
  static int cached[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int per_sm = 0, reserved = 0;
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    if (per_sm <= 0) per_sm = 233472;
    cached[dev] = per_sm / 2 - reserved - 1024;  // minus the static shared memory
  }
  return cached[dev];
}

template <int FAM, int MT, int XDT>
int launch_t(const ccq_dev_model* m, const void* x, int64_t M0, int Mn, void* y, int y_dtype,
             cudaStream_t s) {
  using F = HF<FAM>;
  constexpr int CGB = (32 * F::PB + 15) & ~15;
  constexpr int REC = CGB + (FAM == kF206 ? 32 : 0);
  constexpr size_t SB = 16 * REC;
  if (m->rec != uint32_t(REC)) return kNotApplicable;
  int dev = 0;
  cudaGetDevice(&dev);
  HmmaArgs a{};
  a.L = layout_of(m);
  a.x = static_cast<const uint16_t*>(x) + size_t(M0) * size_t(m->cols);
  a.y = static_cast<uint8_t*>(y) + size_t(M0) * size_t(m->rows) * (y_dtype == CCQ_DTYPE_F32 ? 4 : 2);
  a.x_dtype = XDT;
  a.y_dtype = y_dtype;
  a.M = Mn;
  a.x_stride = m->cols;
  a.y_stride = m->rows;
  a.ntiles = int((m->rows + 15) / 16);
  a.gpr_pad = m->nch * kChunk;
  const int sms = num_sms(dev);
  const int grid = std::min(sms, a.ntiles);
  a.units_max = ((a.ntiles + grid - 1) / grid) * m->nch;
  const size_t fixed = size_t(MT) * a.gpr_pad * 128 + size_t(a.gpr_pad) * std::max(MT, 4) * 4 +
                       size_t(a.units_max) * kSlices * 16 * MT * 4 + 32 + 256;
  // one CTA of 32 warps per SM (64 registers each): the decode is latency
  // bound below 8 warps per scheduler (profiles/r02_hmma_*)
  // 16 warps and two CTAs per SM (the next layer's CTA is resident and
  // prefetches during this one) for small token counts on K <= 4096; one
  // 32-warp CTA per SM otherwise (profiles/r02_gemv_hmma_warps.txt)
  static const int warps_env = std::getenv("CCQ_HMMA_WARPS") ? std::atoi(std::getenv("CCQ_HMMA_WARPS")) : 0;
  const int warps = warps_env > 0 ? warps_env : (MT <= 4 && m->nch <= 2 ? 16 : 32);
  int64_t budget = warps <= 16 ? half_sm_budget(dev) : int64_t(max_smem_optin(dev)) - 1024;
  int64_t R = (budget - int64_t(fixed) - 256) / int64_t(SB + 16);
  if (R < 4) {
    budget = max_smem_optin(dev) - 1024;
    R = (budget - int64_t(fixed) - 256) / int64_t(SB + 16);
  }
  if (R < 2) return kNotApplicable;
  R = std::min<int64_t>(R, a.units_max);
  a.R = int(R);
  const size_t smem = fixed + 256 + size_t(R) * (SB + 16) + 128;
  auto kern = gemv_hmma<FAM, MT, XDT>;
  if (int st = ensure_smem(reinterpret_cast<const void*>(kern), smem)) return st;
  cudaError_t e = launch_pdl(kern, dim3(unsigned(grid)), dim3(unsigned(warps * 32)), smem, s, a);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemv_hmma launch");
}

template <int FAM, int XDT>
int launch_xdt(const ccq_dev_model* m, const void* x, int64_t M, void* y, int y_dtype, cudaStream_t s) {
  for (int64_t m0 = 0; m0 < M;) {
    const int64_t left = M - m0;
    int st;
    int take;
    if (left == 1) {
      st = launch_t<FAM, 1, XDT>(m, x, m0, 1, y, y_dtype, s);
      take = 1;
    } else if (left == 2) {
      st = launch_t<FAM, 2, XDT>(m, x, m0, 2, y, y_dtype, s);
      take = 2;
    } else if (left <= 4) {
      st = launch_t<FAM, 4, XDT>(m, x, m0, int(left), y, y_dtype, s);
      take = int(left);
    } else {
      take = int(std::min<int64_t>(left, 8));
      st = launch_t<FAM, 8, XDT>(m, x, m0, take, y, y_dtype, s);
    }
    if (st != CCQ_OK) return st;
    m0 += take;
  }
  return CCQ_OK;
}

}  // namespace

bool gemv_hmma_supported(const ccq_dev_model* m, int64_t M, int x_dtype, const void* x) {
  static const int mode = std::getenv("CCQ_GEMV_HMMA") ? std::atoi(std::getenv("CCQ_GEMV_HMMA")) : 1;
  if (mode == 0 || (mode == 1 && M == 1)) return false;  // 2: also M = 1
  if (m->geo.group_size != 64 || !m->fast) return false;
  // 2.75 / 2.5 decode as fast on r01's gemv_mma (profiles/r02_gemv_hmma_families.txt): 2.06 only by default
  static const int fams = std::getenv("CCQ_HMMA_FAMS") ? std::atoi(std::getenv("CCQ_HMMA_FAMS")) : (1 << kF206);
  if (!((fams >> m->family) & 1)) return false;
  if (x_dtype != CCQ_DTYPE_BF16 && x_dtype != CCQ_DTYPE_F16) return false;
  // activations are staged with 16-byte loads of whole 64-weight groups
  if ((reinterpret_cast<uintptr_t>(x) & 15u) != 0 || m->cols % 64 != 0) return false;
  return M >= 1 && M <= 8;
}

int launch_gemv_hmma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                     cudaStream_t s) {
  const bool bf = x_dtype == CCQ_DTYPE_BF16;
  switch (m->family) {
    case kF275: return bf ? launch_xdt<kF275, CCQ_DTYPE_BF16>(m, x, M, y, y_dtype, s)
                          : launch_xdt<kF275, CCQ_DTYPE_F16>(m, x, M, y, y_dtype, s);
    case kF25: return bf ? launch_xdt<kF25, CCQ_DTYPE_BF16>(m, x, M, y, y_dtype, s)
                         : launch_xdt<kF25, CCQ_DTYPE_F16>(m, x, M, y, y_dtype, s);
    default: return bf ? launch_xdt<kF206, CCQ_DTYPE_BF16>(m, x, M, y, y_dtype, s)
                       : launch_xdt<kF206, CCQ_DTYPE_F16>(m, x, M, y, y_dtype, s);
  }
}

}  // namespace ccqb

#ifdef CCQ_GEMV_TRACE
extern "C" int ccq_trace_dump_h(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ccqb::g_trace_h, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif
