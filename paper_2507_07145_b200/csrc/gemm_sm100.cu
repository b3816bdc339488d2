// Kernel (c): prefill / batched GEMM on the 5th-generation tensor cores.
//
// Reference: ccq::gemv_batch (kernels.cpp:152-187), Y = X W^T, computed here
// as a real dense contraction once the batch is large enough to need one.
//
//   D[128 weight rows x BN tokens] (TMEM, f32) =
//       A[128 x K] (decoded weights, f16, TMEM: row = lane, K along columns)
//     * B[BN x K]^T (activations, f16, shared memory, TMA 128-byte swizzle)
//
// Warp roles (512 threads):
//   warps 0-11  decode producers, 3 groups of 4 (K blocks kb % 3): thread r
//               of a group owns weight row r of the tile (= TMEM lane r) and
//               turns one 64-weight group into 32 f16x2 columns of the A
//               stage with one tcgen05.st; afterwards they run the epilogue
//               (tcgen05.ld -> super scale -> y)
//   warp 12     TMA producer: packed-code blocks (128 rows x 8 groups, 2D
//               tensor map, 128B swizzle) + side-band nibbles
//   warp 13     TMA producer: activation tiles (BN x 64 f16, 128B swizzle)
//   warp 14     TMEM allocation; lane 0 issues tcgen05.mma (M=128, N=BN,
//               K=16, A from TMEM) and commits stages back to the producers
//
// Exactness (SURVEY §7 hard part 3): each A value is the exact f16
//     sc * (s - zero_point) * 2^p
// (|.| <= 15*32*8 has <= 9 significant bits), built with one HFMA2 from the
// magic-exponent value 1024 + s*2^p; the matching activation is x * 2^-p,
// exact in f16 for bf16 inputs.  Products are exact in the f32 accumulate,
// so only the accumulation order differs from the reference.
//
// Activations are first converted by a tiny pre-pass to f16 in a per-family
// permuted K order (the order in which the decoder emits weight pairs).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>

#include "ccq_internal.hpp"
#include "ptx.cuh"
#include "tcgen05.cuh"

namespace ccqb {

// ---------------------------------------------------------------------------
// Host side: tensor maps via the driver entry point (no libcuda link).
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_map_2d(CUtensorMap* map, CUtensorMapDataType dt, void* base, uint64_t dim0, uint64_t dim1,
                uint64_t stride1_bytes, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(CCQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {dim0, dim1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(map, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CCQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return CCQ_OK;
}

namespace {

constexpr int kBM = 128;        // weight rows per tile (UMMA M)
constexpr int kBK = 64;         // K per block = one group
constexpr int kStagesC = 5;     // packed-code ring (8 groups per stage)
constexpr int kCodeBox = 128;   // bytes of codes per row per code stage (8 groups x 16 B)
// PAR decode warp groups (K-block stages st % PAR), 4 warps each (one per
// TMEM lane quadrant); then 4 control warps.  Warp roles: decode warps first,
// control warps LAST - the SM warp scheduler prefers the highest warp id among
// eligible warps, and the single MMA issuing thread must not be starved by the
// decode warps on its sub-partition.
//   warp 4 PAR      TMA producer: packed codes
//   warp 4 PAR + 1  TMA producer: activation tiles
//   warp 4 PAR + 2  TMEM alloc + MMA issue
template <int PAR, int RT = 1>
struct Roles {
  static constexpr int kDecWarps = 4 * RT * PAR;
  static constexpr int kThreads = 32 * kDecWarps + 128;
  static constexpr int kWarpCodes = kDecWarps, kWarpB = kDecWarps + 1, kWarpMma = kDecWarps + 2;
};
constexpr int kACols = kBK / 2; // TMEM columns per A stage (two f16 per column)

// ---------------------------------------------------------------------------
// Activation pre-pass: x[M][K] (f32/bf16/f16) -> x16[M*XS][K] f16, permuted,
// one CTA per token.
// 2.06: within each stored byte (4 weights, fields s0..s3 at shifts 9,6,3,0)
// the decoder emits (s3, s2*8, s1, s0*8) as two half2 -> x16 holds
// (x3, x2/8, x1, x0/8) for every 4 consecutive K.
// Each token row is first scaled by a power of two 2^s that puts max|x| in
// [2^14, 2^15) (exact; no f16 overflow, no subnormal loss); the epilogue
// multiplies by inv_scale[token] = 2^-s.  f32 inputs are split into XS = 2
// f16 rows, hi = f16(x) and lo = f16(x - hi) (22+ significant bits), whose
// partial products the epilogue adds; bf16/f16 inputs are exact with XS = 1.
// ---------------------------------------------------------------------------
template <int XDT>
__device__ __forceinline__ void load4(const void* x, int64_t base, float (&v)[4]) {
  if constexpr (XDT == CCQ_DTYPE_F32) {
    const float4 t = *reinterpret_cast<const float4*>(static_cast<const float*>(x) + base);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const uint2 t = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(x) + base);
    const uint16_t h[4] = {uint16_t(t.x & 0xFFFF), uint16_t(t.x >> 16), uint16_t(t.y & 0xFFFF),
                           uint16_t(t.y >> 16)};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      v[i] = XDT == CCQ_DTYPE_BF16 ? __uint_as_float(uint32_t(h[i]) << 16)
                                   : __half2float(__ushort_as_half(h[i]));
  }
}

template <int FAM, int XDT, int XS>
__global__ void __launch_bounds__(256) x_prepass(const void* __restrict__ x, __half* __restrict__ out,
                                                 float* __restrict__ inv_scale, int64_t K) {
  // PDL: the GEMM behind this kernel may start its weight loads and decode
  // now; x belongs to the previous kernel until the wait returns.
  griddep_launch_dependents();
  griddep_wait();
  const int64_t m = blockIdx.x;
  const int64_t nq = K / 4;
  float mx = 0.f;
  // 2.06 with 16-bit activations: the token row is read ONCE with 16-byte
  // loads and kept in registers for the conversion (K <= 8 x 8 x threads);
  // otherwise two passes (the second from L1/L2).
  constexpr bool kCacheable = FAM == kF206 && XDT != CCQ_DTYPE_F32 && XS == 1;
  constexpr int kCache = 8;
  const int64_t n8 = K / 8;
  const bool cached = kCacheable && K % 8 == 0 && n8 <= int64_t(kCache) * blockDim.x &&
                      (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
  uint4 cv[kCacheable ? kCache : 1];
  auto f16b = [](uint32_t h) {
    return XDT == CCQ_DTYPE_BF16 ? __uint_as_float(h << 16) : __half2float(__ushort_as_half(uint16_t(h)));
  };
  if (cached) {
#pragma unroll
    for (int i = 0; i < (kCacheable ? kCache : 1); ++i) {
      const int64_t q = threadIdx.x + int64_t(i) * blockDim.x;
      if (q < n8) {
        cv[i] = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + m * K + q * 8));
        const uint32_t w[4] = {cv[i].x, cv[i].y, cv[i].z, cv[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          mx = fmaxf(mx, fmaxf(fabsf(f16b(w[j] & 0xFFFFu)), fabsf(f16b(w[j] >> 16))));
      }
    }
  } else {
    for (int64_t q = threadIdx.x; q < nq; q += blockDim.x) {
      float v[4];
      load4<XDT>(x, m * K + q * 4, v);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3]))));
    }
  }
  __shared__ float red[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  int ex = 0;
  if (mx > 0.f && mx <= 3.0e38f) frexpf(mx, &ex);  // mx < 2^ex
  int sh = mx > 0.f ? 15 - ex : 0;
  sh = sh > 126 ? 126 : (sh < -126 ? -126 : sh);
  const float scale = __int_as_float((127 + sh) << 23);
  if (threadIdx.x == 0) inv_scale[m] = __int_as_float((127 - sh) << 23);
  if constexpr (kCacheable) {
    if (cached) {
      // same arithmetic as the loop below: (x3, x2/8, x1, x0/8) per 4 K, scaled
#pragma unroll
      for (int i = 0; i < kCache; ++i) {
        const int64_t q = threadIdx.x + int64_t(i) * blockDim.x;
        if (q < n8) {
          const uint32_t w[4] = {cv[i].x, cv[i].y, cv[i].z, cv[i].w};
          uint32_t o[4];
#pragma unroll
          for (int hq = 0; hq < 2; ++hq) {
            const float v0 = f16b(w[2 * hq] & 0xFFFFu), v1 = f16b(w[2 * hq] >> 16);
            const float v2 = f16b(w[2 * hq + 1] & 0xFFFFu), v3 = f16b(w[2 * hq + 1] >> 16);
            const __half2 a = __floats2half2_rn(v3 * scale, v2 * scale * 0.125f);
            const __half2 b = __floats2half2_rn(v1 * scale, v0 * scale * 0.125f);
            o[2 * hq] = *reinterpret_cast<const uint32_t*>(&a);
            o[2 * hq + 1] = *reinterpret_cast<const uint32_t*>(&b);
          }
          *reinterpret_cast<uint4*>(out + m * K + q * 8) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      return;
    }
  }
  if constexpr (FAM != kF206) {
    // 2.75 / 2.5: K position 2U + e of a group holds weight unit_wp(c, u, e)
    // (U = 8c + u) scaled by 2^-p - the order the GEMM decoders emit
    for (int64_t q = threadIdx.x; q < K / 2; q += blockDim.x) {
      const int64_t G = q / 32;
      const int U = int(q % 32), cc = U / 8, u = U % 8;
      const WP w0 = unit_wp(FAM, cc, u, 0), w1 = unit_wp(FAM, cc, u, 1);
      float v0, v1;
      if constexpr (XDT == CCQ_DTYPE_F32) {
        v0 = static_cast<const float*>(x)[m * K + G * 64 + w0.w];
        v1 = static_cast<const float*>(x)[m * K + G * 64 + w1.w];
      } else {
        const uint16_t h0 = static_cast<const uint16_t*>(x)[m * K + G * 64 + w0.w];
        const uint16_t h1 = static_cast<const uint16_t*>(x)[m * K + G * 64 + w1.w];
        v0 = XDT == CCQ_DTYPE_BF16 ? __uint_as_float(uint32_t(h0) << 16) : __half2float(__ushort_as_half(h0));
        v1 = XDT == CCQ_DTYPE_BF16 ? __uint_as_float(uint32_t(h1) << 16) : __half2float(__ushort_as_half(h1));
      }
      const float t0 = v0 * scale * __int_as_float((127 - w0.p) << 23);
      const float t1 = v1 * scale * __int_as_float((127 - w1.p) << 23);
      const __half2 hv = __floats2half2_rn(t0, t1);
      *reinterpret_cast<__half2*>(out + (m * XS) * K + 2 * q) = hv;
      if constexpr (XS == 2) {
        const float2 f = __half22float2(hv);
        *reinterpret_cast<__half2*>(out + (m * XS + 1) * K + 2 * q) = __floats2half2_rn(t0 - f.x, t1 - f.y);
      }
    }
    return;
  }
  for (int64_t q = threadIdx.x; q < nq; q += blockDim.x) {
    const int64_t k0 = q * 4;
    float v[4];
    load4<XDT>(x, m * K + k0, v);
    float t[4];
    if constexpr (FAM == kF206) {
      t[0] = v[3] * scale; t[1] = v[2] * scale * 0.125f; t[2] = v[1] * scale; t[3] = v[0] * scale * 0.125f;
    }
    const __half2 a = __floats2half2_rn(t[0], t[1]);
    const __half2 b = __floats2half2_rn(t[2], t[3]);
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&a);
    o.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(out + (m * XS) * K + k0) = o;
    if constexpr (XS == 2) {
      const float2 fa = __half22float2(a), fb = __half22float2(b);
      const __half2 la = __floats2half2_rn(t[0] - fa.x, t[1] - fa.y);
      const __half2 lb = __floats2half2_rn(t[2] - fb.x, t[3] - fb.y);
      o.x = *reinterpret_cast<const uint32_t*>(&la);
      o.y = *reinterpret_cast<const uint32_t*>(&lb);
      *reinterpret_cast<uint2*>(out + (m * XS + 1) * K + k0) = o;
    }
  }
}

#ifdef CCQ_GEMM_TRACE
}  // namespace
__device__ unsigned long long g_gtrace[4096 * 8];
__device__ unsigned long long g_gtrace2[4096 * 4];  // per decode warp: first code wait, long waits, max wait; producer
__device__ int g_gexp;  // experiment: 1 skip decode math, 2 skip MMAs, 3 skip TMEM stores
namespace {
__device__ __forceinline__ unsigned long long gclk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
#endif

struct GemmArgs {
  const float* super;
  const WidenPlan* plan;
  void* y;
  int y_dtype;
  int64_t M, rows, K, rows_pad;
  int nkb;  // K blocks (= groups per row)
  // grouped-expert mode (offsets != nullptr): rows are E stacked experts of
  // rows_e rows; expert e owns tokens [offsets[e], offsets[e+1]).
  const int32_t* offsets;
  int64_t rows_e;
  int tpe;  // row tiles per expert
  int xs;   // activation rows per token (2 = f32 hi/lo split)
  const float* inv_scale;  // [tokens] power-of-two activation scale
  // split-K (dense only): blockIdx.z owns K blocks [z*kbs, min((z+1)*kbs, nkb)),
  // raw f32 partials go to partial[z][token][row] and a reduce kernel scales them
  int kbs;
  float* partial;
  // grouped tile-list mode (tile_prefix != nullptr): blockIdx.x is a global
  // token-tile index; expert e owns tiles [tile_prefix[e], tile_prefix[e+1])
  // (device-computed, so the launch needs no host copy of the routing)
  const int32_t* tile_prefix;
  int E;
  // dense L2-aware raster (raster_group > 0): a 1-D grid of nt x nr tiles
  // walked as groups of raster_group row tiles, row tile fastest, so one wave
  // of CTAs covers few token tiles (activation tiles, the big operand) and
  // many row tiles: activations are read ~(nr / group) times, not ~(nr / wave_rows)
  int raster_group, raster_nt, raster_nr;
};

__device__ __forceinline__ uint32_t lop_mask_or(uint32_t v, uint32_t mask, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(magic));
  return d;
}

__device__ __forceinline__ uint32_t hfma2_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// A (TMEM) / B (smem) ring depth: deep enough to cover the L2 latency of an
// activation tile; the B stage is BN x 128 B.
//
// Rings: the decoded A tile lives in TMEM (tcgen05.st by the decode warps;
// the MMA reads A from tensor memory, "TS" form - no shared-memory writes or
// proxy fences; measured: same MMA rate as SS at N = 64..256).  A (TMEM
// columns) and B (shared memory) have SEPARATE rings and barriers so the
// activation TMA can run far ahead of the decoders (L2 latency ~1 us).
// One ring: stage s = {A: kACols TMEM columns, B: BN x 128 B of smem}; a
// single `full` barrier per stage completes when the 128 decoders of that K
// block have arrived AND the activation TMA bytes have landed, so the MMA
// issuer waits once per K block (each mbarrier wait costs ~90 cycles).
// A stage holds G groups (K = 64 G): each mbarrier wait + tcgen05 fence on
// the MMA issuing thread costs ~200 cycles (measured, tools/micro/mma_loop.cu)
// while 4 MMAs of N = 64 take ~180, so small-N tiles batch several groups per
// wait; at N = 256 one group (512 MMA cycles) already hides it.
// Family traits of the GEMM: code box bytes per row (8 groups), code ring
// depth, side-band nibbles, and SPLIT = number of f16 operand parts per
// weight (2.5: 13-bit scales do not fit f16 exactly; sc = 64 hi + lo gives
// two exact operands and two accumulators, combined in the epilogue).
template <int FAM>
struct GF;
template <>
struct GF<kF206> {
  static constexpr int BOXB = 128, STAGES_C = 5, NIB = 1, SPLIT = 1;
};
template <>
struct GF<kF275> {
  static constexpr int BOXB = 176, STAGES_C = 4, NIB = 0, SPLIT = 1;
};
template <>
struct GF<kF25> {
  static constexpr int BOXB = 160, STAGES_C = 4, NIB = 0, SPLIT = 2;
};

// Ring shape.  Each stage holds G groups (K = 64 G): the MMA issuer pays one
// mbarrier wait + fence + commit per stage (~250 cycles,
// profiles/r01_micro_tcgen05_issue.txt), so small-N tiles batch several
// groups per stage.  (Measured: a deeper 2*kPar-stage ring with G = 2 did not
// help small M and slowed the grouped MoE GEMM by 15 %.)
// TMEM: SPLIT*BN + SA*G*SPLIT*32 <= 512.
//
// More decode warp groups (PAR > 3): the decode warps are latency-bound at
// three per SM sub-partition (profiles/r02_gemm_bound.txt: decoding one group
// per thread takes ~870 cycles while the ALU pipe is half idle), so wider
// variants run PAR groups over a ring of SA = PAR one-group stages.  A group
// handles every PAR-th stage and waits on its slot's `empty` barrier by
// phase parity, which is only sound while PAR <= SA (otherwise the barrier
// can be two phases behind and the parity test passes early).  The code ring
// shrinks to what shared memory leaves (>= 3 blocks = 24 K blocks ahead).
//
// Two row tiles per CTA (RT = 2, 256 weight rows): both tiles' MMAs read the
// same activation stage, halving the L2 -> SM traffic of the activation
// operand per FLOP (1 B per 128 FLOP at RT = 1, which at the tensor rate is
// ~10-12 TB/s of crossbar reads: profiles/r02_gemm_l2.txt).  Decode groups
// are then 8 warps (2 tiles x 4 lane quadrants); TMEM holds 2 BN accumulator
// columns + SA stages of 2 x 32 A columns, so RT = 2 exists for BN <= 160.
template <int FAM, int BN, int PAR, int RT = 1>
constexpr int groups_per_stage() {
  if constexpr (RT > 1) return 1;
  if constexpr (PAR > 3) return BN <= 64 ? 2 : 1;
  return GF<FAM>::SPLIT == 2 ? (BN <= 64 ? 2 : 1) : (BN <= 64 ? 4 : (BN <= 128 ? 2 : 1));
}
template <int FAM, int BN, int PAR, int RT = 1>
constexpr int stages_a() {
  if constexpr (RT > 1) return (512 - RT * BN) / (RT * 32) < 4 ? (512 - RT * BN) / (RT * 32) : 4;
  return PAR > 3 ? PAR : (BN <= 64 ? 3 : 4);
}

template <int FAM, int BN, int PAR = 3, int RT = 1>
struct GemmSmem {
  static constexpr int SA = stages_a<FAM, BN, PAR, RT>();
  static constexpr int SB = SA;
  static constexpr int G = groups_per_stage<FAM, BN, PAR, RT>();
  static constexpr int B_BLOCK = BN * kBK * 2;               // BN x 128 B per group
  static constexpr int B_BYTES = G * B_BLOCK;
  static constexpr int C_BOX = kBM * GF<FAM>::BOXB;          // 128 rows x 8 groups of codes
  static constexpr int N_BOX = GF<FAM>::NIB ? kBM * 16 : 0;  // side-band nibbles (2.06)
  static constexpr int C_BYTES = RT * C_BOX;                 // one code stage: RT boxes
  static constexpr int N_BYTES = RT * N_BOX;
  static constexpr int SC_FIT = (232448 - 1536 - SB * B_BYTES) / (C_BYTES + N_BYTES);
  static constexpr int SC = SC_FIT < GF<FAM>::STAGES_C ? SC_FIT : GF<FAM>::STAGES_C;
  static constexpr bool OK = SC >= 3 && PAR <= SA && SA >= 2 && (RT == 1 || GF<FAM>::SPLIT == 1) &&
                             RT * GF<FAM>::SPLIT * BN + SA * G * RT * GF<FAM>::SPLIT * kACols <= 512;
  static constexpr int OFF_B = 0;                            // 1024-aligned
  static constexpr int OFF_C = OFF_B + SB * B_BYTES;
  static constexpr int OFF_N = OFF_C + SC * C_BYTES;
  static constexpr int OFF_BAR = OFF_N + SC * N_BYTES;
  static constexpr int TOTAL = OFF_BAR + 512 + 1024;  // + alignment slack
  static constexpr int TMEM_NEED = RT * GF<FAM>::SPLIT * BN + SA * G * RT * GF<FAM>::SPLIT * kACols;
};



// f16 bit pattern of a small non-negative integer (exact below 2048).
__host__ __device__ constexpr uint32_t f16_int(int v) {
  if (v == 0) return 0u;
  int e = 0;
  while ((2 << e) <= v) ++e;
  return uint32_t(((e + 15) << 10) | ((v << (10 - e)) & 0x3FF));
}
__host__ __device__ constexpr uint32_t f16x2_int(int lo, int hi) { return f16_int(lo) | (f16_int(hi) << 16); }

__device__ __forceinline__ uint32_t lop_m(uint32_t v, uint32_t mask) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(v), "r"(mask), "r"(0x64006400u));
  return d;
}
__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// 2.75: one 22-byte group (row base rb, group j of the 8-group code box) ->
// 32 f16x2 columns sc*(s-8)*2^p in the unit order of unit_wp (ccq_internal.hpp).
__device__ __forceinline__ void decode_gemm_275(const uint8_t* rb, int j, uint32_t (&h)[32]) {
  const int off = 22 * j;
  const uint32_t* gp = reinterpret_cast<const uint32_t*>(rb + (off & ~3));
  const uint32_t sh = 8u * uint32_t(off & 3);
  uint32_t w[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) w[i] = gp[i];
  uint32_t B[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) B[i] = __funnelshift_r(w[i], w[i + 1], sh);
  const uint32_t sc = (B[5] >> 8) & 0xFu;  // tail byte 21, low nibble
  const float fs = float(sc);
  const __half2 sc2 = __float2half2_rn(fs);
  const uint32_t scu = *reinterpret_cast<const uint32_t*>(&sc2);
  // bias -(1024 + 8*2^p) * sc, exact in f16 for sc <= 15
  auto bias = [&](int plo, int phi) {
    const __half2 b = __floats2half2_rn(-(1024.f + 8.f * float(1 << plo)) * fs, -(1024.f + 8.f * float(1 << phi)) * fs);
    return *reinterpret_cast<const uint32_t*>(&b);
  };
  const uint32_t b00 = bias(0, 0), b22 = bias(2, 2), b44 = bias(4, 4), b42 = bias(4, 2), b40 = bias(4, 0),
                 b20 = bias(2, 0);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int bb = 5 * c;
    const uint32_t lo = __funnelshift_r(B[bb >> 2], B[(bb >> 2) + 1], 8u * uint32_t(bb & 3));
    const uint32_t hi = B[(bb + 4) >> 2] >> (8u * uint32_t((bb + 4) & 3));
    const uint32_t p0 = prmt(lo, 0u, 0x1100u), p1 = prmt(lo, 0u, 0x3322u);
    h[8 * c + 0] = hfma2_u32(lop_m(p0, 0x000F000Fu), scu, b00);
    h[8 * c + 1] = hfma2_u32(lop_m(p0, 0x003C003Cu), scu, b22);
    h[8 * c + 2] = hfma2_u32(lop_m(p0, 0x00F000F0u), scu, b44);
    h[8 * c + 3] = hfma2_u32(lop_m(p1, 0x000F000Fu), scu, b00);
    h[8 * c + 4] = hfma2_u32(lop_m(p1, 0x003C003Cu), scu, b22);
    h[8 * c + 5] = hfma2_u32(lop_m(p1, 0x00F000F0u), scu, b44);
    const uint32_t eb = 4u + (c == 3 ? 1u : 0u);  // b20 (lanes 0..2) or b21 (lane 3) of B[5]
    const uint32_t me = c == 0 ? 0xF0u : c == 1 ? 0x3Cu : c == 2 ? 0x0Fu : 0xF0u;
    h[8 * c + 6] = hfma2_u32(lop_m(prmt(hi, B[5], (eb << 12) | (eb << 8)), 0x000000F0u | (me << 16)), scu,
                             c == 1 ? b42 : c == 2 ? b40 : b44);
    h[8 * c + 7] = hfma2_u32(lop_m(prmt(hi, 0u, 0x0000u), 0x000F003Cu), scu, b20);
  }
}

// 2.5: one 20-byte group -> 32 f16x2 columns for each of the two exact
// operand parts: lo*(s-4)*2^p and hi*(s-4)*2^p with sc = 64 hi + lo.
__device__ __forceinline__ void decode_gemm_25(const uint8_t* gb, uint32_t (&hl)[32], uint32_t (&hh)[32]) {
  uint32_t W[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) W[i] = reinterpret_cast<const uint32_t*>(gb)[i];
  const uint32_t sc = (W[4] >> 16) & 0x1FFFu;
  const __half2 lo2 = __float2half2_rn(float(sc & 63u)), hi2 = __float2half2_rn(float(sc >> 6));
  const uint32_t lou = *reinterpret_cast<const uint32_t*>(&lo2), hiu = *reinterpret_cast<const uint32_t*>(&hi2);
  auto put = [&](int idx, uint32_t unit, uint32_t magicz) {
    const uint32_t t = hsub2_u32(unit, magicz);  // (s - 4) * 2^p, exact
    hl[idx] = hmul2_u32(t, lou);
    hh[idx] = hmul2_u32(t, hiu);
  };
  constexpr uint32_t z0 = f16x2_int(1028, 1028), z2 = f16x2_int(1040, 1040), z4 = f16x2_int(1088, 1088),
                     z6 = f16x2_int(1280, 1280);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t v = W[c], sv = v >> 9;
    put(8 * c + 0, lop_m(v, 0x00070007u), z0);
    put(8 * c + 1, lop_m(v, 0x001C001Cu), z2);
    put(8 * c + 2, lop_m(v, 0x00700070u), z4);
    put(8 * c + 3, lop_m(v, 0x01C001C0u), z6);
    put(8 * c + 4, lop_m(sv, 0x00070007u), z0);
    put(8 * c + 5, lop_m(sv, 0x001C001Cu), z2);
    put(8 * c + 6, lop_m(sv, 0x00700070u), z4);
    const uint32_t sel = c == 0 ? 0x1010u : c == 1 ? 0x1010u : c == 2 ? 0x1111u : 0x3311u;
    const uint32_t mk = c == 0 ? 0x001C0007u : c == 1 ? 0x01C00070u : c == 2 ? 0x0038000Eu : 0x00E000E0u;
    const uint32_t zz = c == 0 ? f16x2_int(1028, 1040) : c == 1 ? f16x2_int(1088, 1280)
                      : c == 2 ? f16x2_int(1032, 1056) : f16x2_int(1152, 1152);
    put(8 * c + 7, lop_m(prmt(W[4], W[4], sel), mk), zz);
  }
}

template <int FAM, int BN, int PAR, int RT>
__global__ void __launch_bounds__(Roles<PAR, RT>::kThreads, 1)
    gemm_ccq(const __grid_constant__ CUtensorMap tm_codes, const __grid_constant__ CUtensorMap tm_nib,
             const __grid_constant__ CUtensorMap tm_x, GemmArgs a) {
  using SM = GemmSmem<FAM, BN, PAR, RT>;
  using RL = Roles<PAR, RT>;
  static_assert(SM::OK && SM::TMEM_NEED <= 512 && SM::TOTAL <= 232448, "ring does not fit");
  constexpr int kPar = PAR, kDecWarps = RL::kDecWarps, kRows = kBM * RT;
  constexpr int kWarpCodes = RL::kWarpCodes, kWarpB = RL::kWarpB, kWarpMma = RL::kWarpMma;
  constexpr int SA = SM::SA, SB = SM::SB, G = SM::G;
  constexpr int SPLIT = GF<FAM>::SPLIT;
  constexpr int kStagesC = SM::SC;
  constexpr int kCodeBox = GF<FAM>::BOXB;
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offset (not through an integer cast, which would turn
  // every smem access of the decoders into a generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);
  static_assert(SA == SB, "single ring");
  uint64_t* full = bars;                        // [SA], 4 decode warps + 1 TMA arrival (+tx)
  uint64_t* empty = full + SA;                  // [SA], mma commit
  uint64_t* code_full = empty + SA;             // [kStagesC], tx
  uint64_t* code_empty = code_full + kStagesC;  // [kStagesC], one arrival per decode warp
  uint64_t* tmem_full = code_empty + kStagesC;  // 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PDL: the launch behind this one (split-K reduce, the next layer's
  // prepass) waits for this grid's completion itself, so it may be scheduled now.
  griddep_launch_dependents();
  // Weights (codes, nibbles, plans, super scales) are static; the activation
  // tile, inv_scale, y and the routing offsets belong to the previous kernel
  // until griddepcontrol.wait: the B producer and the epilogue wait, and in
  // grouped mode every thread waits before reading the offsets.
  if (a.offsets) griddep_wait();
  // Tile: weight rows [r0, row_end), tokens [n0, tok_end); y row stride y_ld,
  // y column of row r is r - y_col0.
  // The tile covers BN activation rows = BN / xs tokens.
  int64_t r0, row_end, tok_end, y_ld, y_col0;
  int n0;
  const int tb = BN / a.xs;
  if (a.offsets) {
    int e, t, jt;
    if (a.tile_prefix) {
      const int tt = int(blockIdx.x);
      if (tt >= a.tile_prefix[a.E]) return;  // worst-case grid: no tile here
      int lo = 0, hi = a.E;                  // tile_prefix[lo] <= tt < tile_prefix[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.tile_prefix[mid] <= tt) lo = mid;
        else hi = mid;
      }
      e = lo;
      jt = tt - a.tile_prefix[e];
      t = int(blockIdx.y);
    } else {
      e = blockIdx.y / a.tpe;
      t = blockIdx.y % a.tpe;
      jt = int(blockIdx.x);
    }
    r0 = e * a.rows_e + int64_t(t) * kRows;
    row_end = (e + 1) * a.rows_e < r0 + kRows ? (e + 1) * a.rows_e : r0 + kRows;
    n0 = a.offsets[e] + jt * tb;
    tok_end = a.offsets[e + 1];
    if (n0 >= tok_end) return;  // expert without (more) tokens: no work, no bytes
    y_ld = a.rows_e;
    y_col0 = e * a.rows_e;
  } else {
    int bt = int(blockIdx.x), br = int(blockIdx.y);
    if (a.raster_group > 0) {
      const int pid = int(blockIdx.x), per_group = a.raster_group * a.raster_nt;
      const int gid = pid / per_group, first = gid * a.raster_group;
      const int gsz = min(a.raster_nr - first, a.raster_group);
      br = first + (pid % per_group) % gsz;
      bt = (pid % per_group) / gsz;
    }
    r0 = int64_t(br) * kRows;
    row_end = a.rows < r0 + kRows ? a.rows : r0 + kRows;
    n0 = bt * tb;
    tok_end = a.M;
    y_ld = a.rows;
    y_col0 = 0;
  }
  const int kb0 = a.partial ? int(blockIdx.z) * a.kbs : 0;  // first (absolute) K block
  const int nkb = a.partial ? min(a.kbs, a.nkb - kb0) : a.nkb;  // K blocks of this CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&full[s], 4 * RT + 1);  // 4 RT decode warps (one elected lane each) + 1 TMA arrival
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kStagesC; ++s) {
      mbar_init(&code_full[s], 1);
      mbar_init(&code_empty[s], kDecWarps);  // one elected lane per decode warp
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
    prefetch_tmap(&tm_codes);
    prefetch_tmap(&tm_nib);
    prefetch_tmap(&tm_x);
  }
  constexpr int kTmemNeed = SM::TMEM_NEED;
  constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  if (warp == kWarpMma) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;             // accumulator(s): columns [0, RT * SPLIT * BN)
  const uint32_t tmem_a = tmem_d + RT * SPLIT * BN;  // A stages: SA x G x RT x SPLIT x kACols columns
  const int nst = (nkb + G - 1) / G;          // pipeline stages (G groups each)

  if (warp == kWarpB) {
    if (lane == 0) {
      // ---------------- TMA producer: activation tiles ----------------
      griddep_wait();
      for (int st = 0; st < nst; ++st) {
        const int s = st % SB;
        const int ng = nkb - st * G < G ? nkb - st * G : G;
        mbar_wait(&empty[s], ((st / SB) + 1) & 1);
        mbar_arrive_expect_tx(&full[s], uint32_t(ng) * SM::B_BLOCK);
        for (int gg = 0; gg < ng; ++gg)
          tma_load_2d(smem + SM::OFF_B + s * SM::B_BYTES + gg * SM::B_BLOCK, &tm_x,
                      (kb0 + st * G + gg) * kBK, n0 * a.xs, &full[s]);
      }
    }
  } else if (warp == kWarpCodes) {
    if (lane == 0) {
      // ---------------- TMA producer: packed codes (runs ahead on its own ring) ----
#ifdef CCQ_GEMM_TRACE
      unsigned long long pw = 0;
#endif
      for (int cb = 0; cb * 8 < nkb; ++cb) {
        const int kb = kb0 + cb * 8, cs = cb % kStagesC;
#ifdef CCQ_GEMM_TRACE
        const unsigned long long tp = gclk();
#endif
        mbar_wait(&code_empty[cs], ((cb / kStagesC) + 1) & 1);
#ifdef CCQ_GEMM_TRACE
        pw += gclk() - tp;
#endif
        // RT boxes of 128 rows; a second box with no row of this tile is not loaded
        const int nbox = RT > 1 && r0 + kBM >= row_end ? 1 : RT;
        mbar_arrive_expect_tx(&code_full[cs], uint32_t(nbox) * (SM::C_BOX + SM::N_BOX));
        const int c = kb / kChunk, jb = (kb % kChunk) / 8;
        const int y = int(int64_t(c) * a.rows_pad + r0);
        for (int hb = 0; hb < nbox; ++hb) {
          tma_load_2d(smem + SM::OFF_C + cs * SM::C_BYTES + hb * SM::C_BOX, &tm_codes, jb * kCodeBox, y + hb * kBM,
                      &code_full[cs]);
          if constexpr (GF<FAM>::NIB)
            tma_load_2d(smem + SM::OFF_N + cs * SM::N_BYTES + hb * SM::N_BOX, &tm_nib, 0, y + hb * kBM, &code_full[cs]);
        }
      }
#ifdef CCQ_GEMM_TRACE
      if (blockIdx.x == 0 && blockIdx.y < 3840 / kDecWarps) g_gtrace2[(blockIdx.y * kDecWarps) * 4 + 3] = pw;
#endif
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer (whole warp, converged; one elected lane issues) ----
    {
      constexpr uint32_t idesc = idesc_f16_f32(kBM, BN);
#ifdef CCQ_GEMM_TRACE
      unsigned long long wa = 0, wb = 0, t0m = gclk();
#endif
      // B descriptors: one base per stage, + (byte offset >> 4) per group / K step
      const uint64_t db_ring = smem_desc(smem_addr(smem + SM::OFF_B), 16, 1024, 2);
      for (int st = 0; st < nst; ++st) {
        const int s = st % SA;
        const int ng = nkb - st * G < G ? nkb - st * G : G;
#ifdef CCQ_GEMM_TRACE
        unsigned long long ta = gclk();
        mbar_wait(&full[s], (st / SA) & 1);
        wa += gclk() - ta;
#else
        mbar_wait(&full[s], (st / SA) & 1);
#endif
        tc_fence_after();
        const uint64_t db_s = db_ring + uint64_t((s * SM::B_BYTES) >> 4);
        const uint32_t ta_s = tmem_a + (s * G * RT * SPLIT) * kACols;
#ifdef CCQ_GEMM_TRACE
        const unsigned long long tb0 = gclk();
        if (g_gexp != 2)
#endif
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          if (gg < ng) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // A from TMEM (lane = weight row, 8 columns per K = 16);
              // B: 128B-swizzled K-major (TMA layout): 32 B per K step inside the atom.
              // Row tile ht of the CTA: accumulator columns ht * SPLIT * BN.
              const uint64_t db = db_s + uint64_t((gg * SM::B_BLOCK + k * 32) >> 4);
#pragma unroll
              for (int ht = 0; ht < RT; ++ht)
#pragma unroll
                for (int h = 0; h < SPLIT; ++h)
                  mma_f16_ts_warp(tmem_d + (ht * SPLIT + h) * BN, ta_s + ((gg * RT + ht) * SPLIT + h) * kACols + k * 8,
                                  db, idesc, (st | gg | k) != 0);
            }
          }
        }
#ifdef CCQ_GEMM_TRACE
        wb += gclk() - tb0;
#endif
        mma_commit_warp(&empty[s]);
      }
      mma_commit_warp(tmem_full);
#ifdef CCQ_GEMM_TRACE
      if (lane == 0 && blockIdx.x == 0 && blockIdx.y < 3840 / kDecWarps) {
        const int slot = (blockIdx.y * kDecWarps) * 8;
        g_gtrace[slot + 5] = wa; g_gtrace[slot + 6] = wb; g_gtrace[slot + 7] = gclk() - t0m;
      }
#endif
    }
  } else if (warp < kDecWarps) {
    // ---------------- decode producers (+ epilogue) ----------------
    const int quad = warp & 3;              // TMEM lane quadrant this warp may access
    const int ht = (warp >> 2) % RT;        // row tile of the CTA
    const int parity = warp / (4 * RT);     // K blocks kb % kPar == parity
    const int r = quad * 32 + lane;         // row in the tile == TMEM lane
    const int64_t row = r0 + ht * kBM + r;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    // Rows past row_end decode row_end-1's plan (their output is never
    // stored); an unconditional load keeps M a known 32-bit operand, so
    // the widening stays one IMAD.HI (a select here costs 2 more IMADs/byte).
    WidenPlan pl = WidenPlan{0, 0, plan_sel(0)};
    if constexpr (FAM == kF206) pl = a.plan[row < row_end ? row : row_end - 1];
    const uint32_t selb = pl.sel & 0xFFFFu, step = pl.sel >> 16;
    const uint32_t sel[4] = {selb, selb + step, selb + 2 * step, selb + 3 * step};
    uint32_t magic, mask, shift26;
    asm volatile("mov.b32 %0, 0x64006400;" : "=r"(magic));
    asm volatile("mov.b32 %0, 0x01F8003F;" : "=r"(mask));
    asm volatile("mov.b32 %0, 0x04000000;" : "=r"(shift26));
#ifdef CCQ_GEMM_TRACE
    unsigned long long t_code = 0, t_dec = 0, t_empty = 0, t_st = 0, t_prev = gclk(), t0 = t_prev;
    unsigned long long x_first = 0, x_long = 0, x_max = 0;
#define GT(var) { const unsigned long long _t = gclk(); var += _t - t_prev; t_prev = _t; }
#else
#define GT(var)
#endif
    // Code blocks are released by EVERY decode thread, in order: blocks this
    // group never reads are first awaited (so the arrival lands in the right
    // phase of code_empty), then released.
    int next_rel = 0;
    auto release_until = [&](int cb_end) {
      for (; next_rel < cb_end; ++next_rel) {
        const int rs = next_rel % kStagesC;
        mbar_wait(&code_full[rs], (next_rel / kStagesC) & 1);
        // one arrival per warp, not per thread: 384 serialized shared-memory
        // atomics per code block become 12
        __syncwarp();
        if (lane == 0) mbar_arrive(&code_empty[rs]);
      }
    };
    static_assert(8 % G == 0, "a stage must lie inside one 8-group code block");
    for (int st = parity; st < nst; st += kPar) {
      // per stage: one code block, one code_full wait, one nibble word
      const int s = st % SA;
      const int ng = nkb - st * G < G ? nkb - st * G : G;
      const int kbs = st * G;
      const int cb = kbs >> 3, cs = cb % kStagesC;
      release_until(cb);
#ifdef CCQ_GEMM_TRACE
      const unsigned long long tcw = gclk();
#endif
      mbar_wait(&code_full[cs], (cb / kStagesC) & 1);
#ifdef CCQ_GEMM_TRACE
      {
        const unsigned long long d = gclk() - tcw;
        if (kbs == 0) x_first = gclk() - t0;
        if (d > 1000) ++x_long;
        if (d > x_max) x_max = d;
      }
#endif
      GT(t_code);
      const uint8_t* cstage = smem + SM::OFF_C + cs * SM::C_BYTES + ht * SM::C_BOX;
      uint32_t nibword = 0;
      if constexpr (FAM == kF206)
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nibword)
                     : "r"(smem_addr(smem + SM::OFF_N + cs * SM::N_BYTES + ht * SM::N_BOX + r * 16 +
                                     (((kb0 + kbs) % kChunk) / 8) * 4)));
      // two groups in flight per warp for 2.75 / 2.5 (more ILP for their
      // shift/mask decoders: 2-4 % at M <= 64); 2.06 is issue-bound, unchanged
      // (profiles/r01_gemm_unroll2_experiment.txt)
#pragma unroll(FAM == kF206 ? 1 : 2)
      for (int gg = 0; gg < ng; ++gg) {
      const int j = (kbs & 7) + gg;
      uint32_t h[32];
      uint32_t h2[SPLIT == 2 ? 32 : 1];
#ifdef CCQ_GEMM_TRACE
      if (g_gexp == 1) {
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] = magic + i;
        if constexpr (SPLIT == 2)
#pragma unroll
          for (int i = 0; i < 32; ++i) h2[i] = magic + i;
      } else
#endif
      if constexpr (FAM == kF206) {
        const uint4 cw = lds128(cstage + r * kCodeBox + ((j ^ (r & 7)) << 4));
        const uint32_t sc = (nibword >> (4 * j)) & 0xFu;
        // half2 (sc, sc) and bias (-(1024+32) sc, -(1024+256) sc), exact in f16
        const __half2 sc2 = __hsub2(__halves2half2(__ushort_as_half(uint16_t(0x6400u | sc)),
                                                   __ushort_as_half(uint16_t(0x6400u | sc))),
                                    __float2half2_rn(1024.f));
        const __half2 bias2 = __hmul2(sc2, __floats2half2_rn(-1056.f, -1280.f));
        const uint32_t scu = *reinterpret_cast<const uint32_t*>(&sc2);
        const uint32_t biasu = *reinterpret_cast<const uint32_t*>(&bias2);
        const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
  #pragma unroll
        for (int byte = 0; byte < 16; ++byte) {
          const uint32_t qb = prmt(words[byte >> 2], 0u, sel[byte & 3]);
          const uint32_t hi = uint32_t((uint64_t(qb) * pl.M + pl.C) >> 32);  // code at [8,23)
          const uint32_t w2 = prmt(hi, 0u, 0x2121u);                        // code | code << 16
#ifndef CCQ_GEMM_W3
#define CCQ_GEMM_W3 2
#endif
          // w2 >> 6 on the ALU (SHF) or the FMA pipe (IMAD.HI); mixed to balance the two
          const uint32_t w3 = CCQ_GEMM_W3 == 2 || (CCQ_GEMM_W3 == 1 && (byte & 1)) ? (w2 >> 6) : __umulhi(w2, shift26);
          h[2 * byte] = hfma2_u32(lop_mask_or(w2, mask, magic), scu, biasu);     // (s3, 8 s2)
          h[2 * byte + 1] = hfma2_u32(lop_mask_or(w3, mask, magic), scu, biasu); // (s1, 8 s0)
        }
      } else if constexpr (FAM == kF275) {
        decode_gemm_275(cstage + r * kCodeBox, j, h);
      } else {
        decode_gemm_25(cstage + r * kCodeBox + 20 * j, h, h2);
      }
      GT(t_dec);
      if (gg == 0) {
        mbar_wait(&empty[s], ((st / SA) + 1) & 1);
        GT(t_empty);
        tc_fence_after();
      }
#ifdef CCQ_GEMM_TRACE
      if (g_gexp == 3) {
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= h[i];
        if (acc == 0x12345678u) g_gtrace[4095 * 8] = acc;  // keep the decode alive
      } else {
#endif
      tmem_st32(tmem_a + lane_base + (((s * G + gg) * RT + ht) * SPLIT) * kACols, h);
      if constexpr (SPLIT == 2) tmem_st32(tmem_a + lane_base + (((s * G + gg) * RT + ht) * SPLIT + 1) * kACols, h2);
#ifdef CCQ_GEMM_TRACE
      }
#endif
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
      GT(t_st);
    }
    release_until((nkb + 7) >> 3);
#ifdef CCQ_GEMM_TRACE
    if (lane == 0 && blockIdx.x == 0 && blockIdx.y < 3840 / kDecWarps) {
      const int slot = (blockIdx.y * kDecWarps + warp) * 8;
      g_gtrace[slot + 0] = t_code; g_gtrace[slot + 1] = t_dec; g_gtrace[slot + 2] = t_empty;
      g_gtrace[slot + 3] = t_st; g_gtrace[slot + 4] = gclk() - t0;
      const int s2 = (blockIdx.y * kDecWarps + warp) * 4;
      g_gtrace2[s2 + 0] = x_first; g_gtrace2[s2 + 1] = x_long; g_gtrace2[s2 + 2] = x_max;
    }
#endif

    // ---------------- epilogue: 32-column slices round-robin over the groups ----
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    griddep_wait();  // inv_scale and y (long complete by now)
    const float sup = row < row_end ? a.super[row] : 0.f;
#pragma unroll 1
    for (int cc = parity * 32; cc < BN; cc += 32 * kPar) {
      uint32_t v[32];
      tmem_ld32(tmem_d + ht * SPLIT * BN + lane_base + cc, v);
      if constexpr (SPLIT == 2) {
        uint32_t vh[32];
        tmem_ld32(tmem_d + (ht * SPLIT + 1) * BN + lane_base + cc, vh);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(fmaf(64.f, __uint_as_float(vh[i]), __uint_as_float(v[i])));
      }
      tmem_ld_wait();
      // Lanes are consecutive rows: one 128 B (f32) / 64 B (bf16) store per
      // token and warp.  The token scales are loaded once per slice (one per
      // lane) and broadcast by shuffles - a per-element load behind a store
      // to y (which may alias it) serialised one L1 round trip per element
      // (profiles/r02_gemm_epilogue.txt).  f32 inputs: hi + lo columns first.
      if (a.xs == 2) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[2 * i]) + __uint_as_float(v[2 * i + 1]));
      }
      const int per = 32 / a.xs;          // tokens in this slice
      const int64_t nb = n0 + cc / a.xs;  // its first token
      const bool rok = row < row_end;
      float* const pz = a.partial ? a.partial + size_t(blockIdx.z) * size_t(a.M) * size_t(a.rows) + row : nullptr;
      // split-K: raw sums to the partial buffer, scaled by the reduce kernel
      const float isc = a.partial ? 1.f : (lane < per && nb + lane < tok_end ? __ldg(a.inv_scale + nb + lane) : 0.f);
      const float rs = a.partial ? 1.f : sup;
      const int64_t ycol = row - y_col0;
      const bool f32 = a.partial || a.y_dtype == CCQ_DTYPE_F32;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float si = __shfl_sync(0xffffffffu, isc, i) * rs;
        if (i < per && rok && nb + i < tok_end) {
          const float o = __uint_as_float(v[i]) * si;
          if (pz) pz[(nb + i) * a.rows] = o;
          else if (f32) static_cast<float*>(a.y)[(nb + i) * y_ld + ycol] = o;
          else static_cast<__nv_bfloat16*>(a.y)[(nb + i) * y_ld + ycol] = __float2bfloat16_rn(o);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) tmem_dealloc<kTmemCols>(tmem_d);
}

// Split-K epilogue: y[n][r] = (sum_z partial[z][n][r]) * super[r] * inv_scale[n],
// summed in a fixed order (deterministic).
__global__ void __launch_bounds__(256) splitk_reduce(const float* __restrict__ part, int splits, int64_t M,
                                                     int64_t rows, const float* __restrict__ super,
                                                     const float* __restrict__ inv_scale, void* y, int y_dtype) {
  const int64_t total = M * rows;
  griddep_wait();  // the partial sums are the GEMM's
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += part[size_t(z) * size_t(total) + size_t(i)];
    const int64_t n = i / rows, r = i - n * rows;
    v *= super[r] * inv_scale[n];
    if (y_dtype == CCQ_DTYPE_F32)
      static_cast<float*>(y)[i] = v;
    else
      static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(v);
  }
}

template <int FAM, int BN, int PAR, int RT>
int run_gemm_p(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
               cudaStream_t s, const int32_t* offsets_dev, int64_t rows_e, int E,
               int64_t max_tokens, const int32_t* tile_prefix, int64_t max_tiles) {
  using SM = GemmSmem<FAM, BN, PAR, RT>;
  constexpr int kRows = kBM * RT;
  const int64_t K = m->cols;
  const bool grouped = offsets_dev != nullptr;
  const int xs = x_dtype == CCQ_DTYPE_F32 ? 2 : 1;
  const int64_t xrows = M * xs;  // activation rows (TMA zero-fills past the end)
  void* x16 = nullptr;
  // scratch: the library pool outside graph capture (no re-mapping after
  // syncs); graph-owned memory (cudaMallocAsync) while capturing
  int pdev = 0;
  cudaGetDevice(&pdev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  cudaMemPool_t pool = scratch_pool(pdev);
  auto salloc = [&](void** p, size_t bytes) {
    return capturing ? cudaMallocAsync(p, bytes, s) : cudaMallocFromPoolAsync(p, bytes, pool, s);
  };
  CCQ_CUDA_TRY(salloc(&x16, size_t(xrows * K) * 2 + size_t(M) * 4 + 16));
  float* inv_scale = reinterpret_cast<float*>(static_cast<uint8_t*>(x16) + size_t(xrows * K) * 2);
  if (M > 0) {
    const unsigned blocks = unsigned(M);
    __half* xh = static_cast<__half*>(x16);
    cudaError_t pe;
    if (x_dtype == CCQ_DTYPE_F32)
      pe = launch_pdl(x_prepass<FAM, CCQ_DTYPE_F32, 2>, dim3(blocks), dim3(256), 0, s, x, xh, inv_scale, K);
    else if (x_dtype == CCQ_DTYPE_BF16)
      pe = launch_pdl(x_prepass<FAM, CCQ_DTYPE_BF16, 1>, dim3(blocks), dim3(256), 0, s, x, xh, inv_scale, K);
    else
      pe = launch_pdl(x_prepass<FAM, CCQ_DTYPE_F16, 1>, dim3(blocks), dim3(256), 0, s, x, xh, inv_scale, K);
    count_launch();
    if (pe != cudaSuccess) {
      cudaFreeAsync(x16, s);
      return cuda_fail(pe, "gemm prepass launch");
    }
  }
  CUtensorMap tm_codes, tm_nib, tm_x;
  int st = make_map_2d(&tm_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, m->codes, m->rec,
                       uint64_t(m->nch) * m->rows_pad, m->rec, GF<FAM>::BOXB, kBM,
                       FAM == kF206 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st == CCQ_OK && FAM != kF206) tm_nib = tm_codes;
  if (st == CCQ_OK && FAM == kF206)
    st = make_map_2d(&tm_nib, CU_TENSOR_MAP_DATA_TYPE_UINT8, m->codes + m->cgb, 16,
                     uint64_t(m->nch) * m->rows_pad, m->rec, 16, kBM, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st == CCQ_OK)
    st = make_map_2d(&tm_x, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, x16, uint64_t(K),
                     uint64_t(xrows > 0 ? xrows : 1), uint64_t(K) * 2, kBK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != CCQ_OK) {
    cudaFreeAsync(x16, s);
    return st;
  }
  GemmArgs a{m->super, m->plan, y, y_dtype, M, m->rows, K, m->rows_pad, int(m->gpr),
             offsets_dev, rows_e, grouped ? int((rows_e + kRows - 1) / kRows) : 0, xs, inv_scale, 0, nullptr,
             tile_prefix, E, 0, 0, 0};
  auto kern = gemm_ccq<FAM, BN, PAR, RT>;
  if (int st2 = ensure_smem(reinterpret_cast<const void*>(kern), SM::TOTAL)) {
    cudaFreeAsync(x16, s);
    return st2;
  }
  const int tb = BN / xs;
  dim3 grid = grouped ? (tile_prefix ? dim3(unsigned(max_tiles), unsigned(a.tpe))
                                     : dim3(unsigned((max_tokens + tb - 1) / tb), unsigned(E * a.tpe)))
                      : dim3(unsigned((M + tb - 1) / tb), unsigned((m->rows + kRows - 1) / kRows));
  // Split K when the tiles would leave most SMs idle (K-heavy shapes such as
  // 14336 -> 4096: 32 row tiles); splits cover whole 8-group code blocks.
  float* part = nullptr;
  int splits = 1;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = int64_t(grid.x) * grid.y;
    const int cblocks = int((m->gpr + 7) / 8);
    static const int force_splits = std::getenv("CCQ_GEMM_SPLITS") ? std::atoi(std::getenv("CCQ_GEMM_SPLITS")) : 0;
    if (!grouped && tiles > 0 && ((tiles * 2 <= sms && cblocks >= 8) || force_splits > 1)) {
      splits = int(std::min<int64_t>(sms / tiles, cblocks / 4));
      if (force_splits > 1) splits = std::min(force_splits, cblocks);
      if (splits >= 2) {
        const int cb_per = (cblocks + splits - 1) / splits;
        a.kbs = cb_per * 8;
        splits = (cblocks + cb_per - 1) / cb_per;
        CCQ_CUDA_TRY(salloc(reinterpret_cast<void**>(&part), size_t(splits) * size_t(M) * size_t(m->rows) * 4));
        a.partial = part;
        grid.z = unsigned(splits);
      } else {
        splits = 1;
      }
    }
  }
  // L2-aware raster for multi-wave dense grids: a wave of `sms` CTAs covers
  // ~sms / group token tiles x group row tiles (profiles/r02_gemm_raster.txt)
  static const int raster_env = std::getenv("CCQ_GEMM_RASTER") ? std::atoi(std::getenv("CCQ_GEMM_RASTER")) : -1;
  if (!grouped && splits == 1 && grid.x > 1 && raster_env != 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t sms = num_sms(dev);
    const int64_t nt = grid.x, nr = grid.y;
    if (nt * nr > sms) {
      int gsz = raster_env > 0 ? raster_env : int(std::max<int64_t>(1, sms / std::min<int64_t>(nt, 4)));
      a.raster_group = int(std::min<int64_t>(gsz, nr));
      a.raster_nt = int(nt);
      a.raster_nr = int(nr);
      grid = dim3(unsigned(nt * nr), 1, 1);
    }
  }
  if (grid.x && grid.y) {
    cudaError_t le = launch_pdl(kern, grid, dim3(Roles<PAR, RT>::kThreads), SM::TOTAL, s, tm_codes, tm_nib, tm_x, a);
    count_launch();
    if (le == cudaSuccess && part) {
      const int64_t total = M * m->rows;
      const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 8));
      le = launch_pdl(splitk_reduce, dim3(blocks), dim3(256), 0, s, static_cast<const float*>(part), splits, M,
                      m->rows, m->super, static_cast<const float*>(inv_scale), y, y_dtype);
      count_launch();
    }
    if (le != cudaSuccess) {
      if (part) cudaFreeAsync(part, s);
      cudaFreeAsync(x16, s);
      return cuda_fail(le, "gemm launch");
    }
  }
  cudaError_t e = cudaGetLastError();
  if (part) cudaFreeAsync(part, s);
  cudaFreeAsync(x16, s);
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gemm launch");
}

// Decode warp groups per CTA (PAR, see groups_per_stage): CCQ_GEMM_PAR
// overrides the default; variants are compiled where their ring fits and the
// register budget (65536 / threads) holds the decoder without spills.
template <int FAM, int BN, int PAR, int RT = 1>
constexpr bool par_built() {
  if constexpr (RT == 2)  // 2.06 (<= 80 registers) at the DeepSeek-like tile widths
    // (BN = 192 fits only a 2-stage ring: measured slower, profiles/r02_gemm_rt192.txt)
    return ((FAM == kF206 && (BN == 128 || BN == 160)) || (FAM == kF275 && BN == 160)) && (PAR == 2 || PAR == 3) &&
           GemmSmem<FAM, BN, PAR, RT>::OK;
  if constexpr (PAR == 3) return true;
  // (not at 64-column tiles: PAR 4-6 measured 3-10 % slower there, profiles/r02_gemm_par_small.txt)
  if constexpr (!GemmSmem<FAM, BN, PAR>::OK || BN < 128) return false;
  if constexpr (FAM == kF206) return PAR == 4 || PAR == 5 || PAR == 6;
  if constexpr (FAM == kF275) return BN >= 160 && (PAR == 4 || PAR == 6);
  return false;
}
// Measured per family and tile width (profiles/r02_gemm_par.txt: dense
// 4096 -> 14336 at M = 128..256, configs[4] prefill, grouped prefill).
inline int gemm_par_default(int fam, int bn) {
  if (fam == kF206) return bn == 128 ? 4 : bn == 160 ? 5 : bn == 192 ? 6 : bn == 256 ? 4 : 3;
  if (fam == kF275) return bn == 160 || bn == 192 ? 6 : bn == 256 ? 4 : 3;
  return 3;
}
template <int FAM, int BN>
int run_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
             cudaStream_t s, const int32_t* offsets_dev = nullptr, int64_t rows_e = 0, int E = 0,
             int64_t max_tokens = 0, const int32_t* tile_prefix = nullptr, int64_t max_tiles = 0) {
  static const int force_par = std::getenv("CCQ_GEMM_PAR") ? std::atoi(std::getenv("CCQ_GEMM_PAR")) : 0;
  static const int force_rt = std::getenv("CCQ_GEMM_RT") ? std::atoi(std::getenv("CCQ_GEMM_RT")) : 0;
  // Two row tiles per CTA where they still fill the SMs: every grouped launch
  // (many experts x row tiles) and dense grids of >= 0.8 waves at RT = 2
  // (profiles/r02_gemm_rt.txt: DeepSeek grouped prefill 1198 -> 1120 us,
  // 7168 -> 32768 M=128 68.4 -> 63.3 us; a one-wave 4096 -> 14336 grid at
  // RT = 2 leaves half the SMs idle: 24.8 -> 40.0 us).
  int rt = 1;
  if (force_rt > 0) {
    rt = force_rt;
  } else if (par_built<FAM, BN, 2, 2>()) {
    if (offsets_dev) {
      rt = 2;
    } else {
      int dev = 0;
      cudaGetDevice(&dev);
      const int64_t tb = BN / (x_dtype == CCQ_DTYPE_F32 ? 2 : 1);
      const int64_t tiles2 = (m->rows + 2 * kBM - 1) / (2 * kBM) * ((M + tb - 1) / tb);
      if (tiles2 * 5 >= int64_t(num_sms(dev)) * 4) rt = 2;
    }
  }
  const int par = force_par > 0 ? force_par : rt == 2 ? 2 : gemm_par_default(FAM, BN);
#define CCQ_PAR(P, R)                                                                                       \
  if constexpr (par_built<FAM, BN, P, R>())                                                                 \
    if (par == P && rt == R)                                                                                \
      return run_gemm_p<FAM, BN, P, R>(m, x, x_dtype, M, y, y_dtype, s, offsets_dev, rows_e, E, max_tokens, \
                                       tile_prefix, max_tiles);
  CCQ_PAR(4, 1)
  CCQ_PAR(5, 1)
  CCQ_PAR(6, 1)
  CCQ_PAR(2, 2)
  CCQ_PAR(3, 2)
#undef CCQ_PAR
  return run_gemm_p<FAM, BN, 3, 1>(m, x, x_dtype, M, y, y_dtype, s, offsets_dev, rows_e, E, max_tokens, tile_prefix,
                                   max_tiles);
}

}  // namespace

bool gemm_supported(const ccq_dev_model* m, int64_t M) {
  (void)M;
  return m->geo.group_size == 64 && m->cols % 64 == 0 && m->cols > 0;
}

int launch_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                cudaStream_t s) {
  int64_t xr = x_dtype == CCQ_DTYPE_F32 ? 2 * M : M;  // BN is chosen on activation rows
  static const int force_bn = std::getenv("CCQ_GEMM_BN") ? std::atoi(std::getenv("CCQ_GEMM_BN")) : 0;
  if (force_bn) xr = force_bn;
  switch (m->family) {
    case kF275:
      if (xr <= 64) return run_gemm<kF275, 64>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 128) return run_gemm<kF275, 128>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 160) return run_gemm<kF275, 160>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 192) return run_gemm<kF275, 192>(m, x, x_dtype, M, y, y_dtype, s);
      return run_gemm<kF275, 256>(m, x, x_dtype, M, y, y_dtype, s);
    case kF25:  // two accumulators: at most 128 token columns per tile
      if (xr <= 64) return run_gemm<kF25, 64>(m, x, x_dtype, M, y, y_dtype, s);
      return run_gemm<kF25, 128>(m, x, x_dtype, M, y, y_dtype, s);
    default:
      if (xr <= 64) return run_gemm<kF206, 64>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 128) return run_gemm<kF206, 128>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 160) return run_gemm<kF206, 160>(m, x, x_dtype, M, y, y_dtype, s);
      if (xr <= 192) return run_gemm<kF206, 192>(m, x, x_dtype, M, y, y_dtype, s);
      return run_gemm<kF206, 256>(m, x, x_dtype, M, y, y_dtype, s);
  }
}

// Kernel (d): all experts of a stacked model in ONE launch.  T = total tokens
// (expert-major), max_tokens = largest per-expert token count.
// Token-tile width for a grouped launch: with every tile MMA-bound (N >= 96),
// the time is proportional to the padded columns sum_e ceil(n_e / BN) * BN,
// so take the candidate that minimises them (larger on ties).  DeepSeek's
// ~128 tokens per expert fit one 160-column tile (vs half-empty 256-column
// ones); ERNIE's ~512 stay on 256 (profiles/r02_grouped_bn.txt).
int grouped_bn_for(const ccq_dev_model* stack, const int32_t* offsets_host, int E, int x_dtype) {
  const int xs = x_dtype == CCQ_DTYPE_F32 ? 2 : 1;
  static const int cands[4] = {128, 160, 192, 256};
  int best = 256;
  int64_t best_cols = -1;
  int64_t maxn = 0;
  for (int e = 0; e < E; ++e) maxn = std::max<int64_t>(maxn, offsets_host[e + 1] - offsets_host[e]);
  if (maxn * xs <= 64) return 64;
  for (int c : cands) {
    if (stack->family == kF25 && c > 128) break;  // two accumulators: <= 128 columns
    const int tb = c / xs;
    int64_t cols = 0;
    for (int e = 0; e < E; ++e) cols += (int64_t(offsets_host[e + 1] - offsets_host[e]) + tb - 1) / tb * c;
    if (best_cols < 0 || cols <= best_cols) {
      best_cols = cols;
      best = c;
    }
  }
  return best;
}

int launch_grouped_gemm(const ccq_dev_model* stack, int E, int64_t rows_e, const int32_t* offsets_dev,
                        int64_t T, int64_t max_tokens, const void* x, int x_dtype, void* y,
                        int y_dtype, cudaStream_t s, int bn) {
  if (max_tokens <= 0 || T <= 0) return CCQ_OK;
  int64_t xr = x_dtype == CCQ_DTYPE_F32 ? 2 * max_tokens : max_tokens;
  static const int force_bn = std::getenv("CCQ_GROUPED_BN") ? std::atoi(std::getenv("CCQ_GROUPED_BN")) : 0;
  if (force_bn) bn = force_bn;
  if (bn <= 0) bn = xr <= 64 ? 64 : xr <= 128 ? 128 : 256;
#define CCQ_GROUPED(F, B) run_gemm<F, B>(stack, x, x_dtype, T, y, y_dtype, s, offsets_dev, rows_e, E, max_tokens)
  switch (stack->family) {
    case kF275:
      if (bn <= 64) return CCQ_GROUPED(kF275, 64);
      if (bn <= 128) return CCQ_GROUPED(kF275, 128);
      if (bn <= 160) return CCQ_GROUPED(kF275, 160);
      if (bn <= 192) return CCQ_GROUPED(kF275, 192);
      return CCQ_GROUPED(kF275, 256);
    case kF25:
      if (bn <= 64) return CCQ_GROUPED(kF25, 64);
      return CCQ_GROUPED(kF25, 128);
    default:
      if (bn <= 64) return CCQ_GROUPED(kF206, 64);
      if (bn <= 128) return CCQ_GROUPED(kF206, 128);
      if (bn <= 160) return CCQ_GROUPED(kF206, 160);
      if (bn <= 192) return CCQ_GROUPED(kF206, 192);
      return CCQ_GROUPED(kF206, 256);
  }
#undef CCQ_GROUPED
}

// Sync-free grouped GEMM: the routing lives only on the device.  tile_prefix
// (E + 1 entries, written by an earlier kernel) counts token tiles of
// grouped_tile_tokens(...) tokens per expert; the grid is sized for the worst
// case (max_tiles) and CTAs past tile_prefix[E] exit at once.
int grouped_tile_tokens(const ccq_dev_model* stack, int64_t pairs, int E, int x_dtype) {
  // the routing is not on the host: size tiles for ~1.25x the mean tokens per expert
  const int xs = x_dtype == CCQ_DTYPE_F32 ? 2 : 1;
  const int64_t typ = ((pairs + E - 1) / std::max(E, 1)) * 5 / 4 * xs;
  int bn = typ <= 64 ? 64 : typ <= 128 ? 128 : typ <= 160 ? 160 : typ <= 192 ? 192 : 256;
  if (stack->family == kF25 && bn > 128) bn = 128;
  return bn / xs;
}

int launch_grouped_gemm_tiles(const ccq_dev_model* stack, int E, int64_t rows_e, const int32_t* offsets_dev,
                              const int32_t* tile_prefix_dev, int64_t max_tiles, int64_t T, const void* x,
                              int x_dtype, void* y, int y_dtype, cudaStream_t s) {
  if (T <= 0 || max_tiles <= 0) return CCQ_OK;
  const int xs = x_dtype == CCQ_DTYPE_F32 ? 2 : 1;
  const int bn = grouped_tile_tokens(stack, T, E, x_dtype) * xs;
#define CCQ_TILES(F, B) \
  run_gemm<F, B>(stack, x, x_dtype, T, y, y_dtype, s, offsets_dev, rows_e, E, 0, tile_prefix_dev, max_tiles)
  switch (stack->family) {
    case kF275:
      return bn == 64 ? CCQ_TILES(kF275, 64) : bn == 128 ? CCQ_TILES(kF275, 128) : bn == 160 ? CCQ_TILES(kF275, 160)
           : bn == 192 ? CCQ_TILES(kF275, 192) : CCQ_TILES(kF275, 256);
    case kF25:
      return bn == 64 ? CCQ_TILES(kF25, 64) : CCQ_TILES(kF25, 128);
    default:
      return bn == 64 ? CCQ_TILES(kF206, 64) : bn == 128 ? CCQ_TILES(kF206, 128) : bn == 160 ? CCQ_TILES(kF206, 160)
           : bn == 192 ? CCQ_TILES(kF206, 192) : CCQ_TILES(kF206, 256);
  }
#undef CCQ_TILES
}

}  // namespace ccqb

#ifdef CCQ_GEMM_TRACE
extern "C" int ccq_gemm_trace_dump2(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ccqb::g_gtrace2, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
extern "C" int ccq_gemm_trace_exp(int e) { return cudaMemcpyToSymbol(ccqb::g_gexp, &e, sizeof(int)) == cudaSuccess ? 0 : 1; }
extern "C" int ccq_gemm_trace_dump(unsigned long long* host, int n) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(host, ccqb::g_gtrace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif
