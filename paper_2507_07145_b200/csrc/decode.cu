// Kernel (a): standalone decode of packed CCQ groups into integer levels
// and/or f32 weights, bit-exact to the reference dequantize
// (kernels.cpp:60-122; FORMAT.md §7).
//
// One thread decodes one group (64 weights at the default group size).  The
// group's payload is read with the widest aligned loads the family allows
// (16 B for 2.06, 4 B for 2.5, 2 B for 2.75 at group size 64); the per-row
// super scale and widening plan come from the row tables built at upload.
// Arithmetic matches the reference exactly:
//   scale  = float(scale_code) * super            (f32, round to nearest)
//   weight = float(state - zero_point) * scale    (f32, round to nearest)
//   code   = lround(q * alpha + beta)             via the exact fixed-point plan
// The kernel is store-bound (5 B written per weight when both outputs are
// requested, vs 0.26-0.34 B read); outputs are written with 16-byte vector
// stores where the layout allows.
#include "ccq_internal.hpp"

namespace ccqb {
namespace {

struct DecodeArgs {
  DevLayout L;
  int8_t* levels;
  float* weights;
  int64_t groups;
};

template <int FAM>
__device__ __forceinline__ uint32_t load_word(const uint8_t* p) {
  constexpr FamilyConst fc = family_const(FAM);
  if constexpr (fc.word_bytes == 2) return uint32_t(p[0]) | (uint32_t(p[1]) << 8);
  return p[0];
}

// Generic decoder: any group geometry.  Writes directly to global memory.
template <int FAM>
__global__ void __launch_bounds__(256) decode_generic(DecodeArgs a) {
  constexpr FamilyConst fc = family_const(FAM);
  const int64_t gi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gi >= a.groups) return;
  const DevLayout& L = a.L;
  const int64_t r = gi / L.gpr, gj = gi - r * L.gpr;
  const uint8_t* p = L.group(r, gj);
  uint32_t sc;
  if (L.geo.embedded_scale) {
    sc = load_word<FAM>(p + L.geo.full_words * fc.word_bytes) & fc.scale_mask;
  } else {
    sc = L.nibble(r, gj);
  }
  const float scale = __fmul_rn(float(sc), L.super[r]);
  WidenPlan pl{};
  if constexpr (fc.cluster) pl = L.plan[r];
  const int64_t base = r * L.cols + gj * L.geo.group_size;
  int idx = 0;
  for (int w = 0; w < L.geo.words_per_group; ++w) {
    uint32_t code = load_word<FAM>(p + w * fc.word_bytes);
    if constexpr (fc.cluster) code = widen_hi(code, pl) >> 8;
    const int nk = (w < L.geo.full_words) ? fc.wpw : 1;
    for (int k = 0; k < nk; ++k) {
      const int lv = int((code >> fc.shifts[k]) & fc.weight_mask) - fc.zero_point;
      if (a.weights) a.weights[base + idx] = __fmul_rn(float(lv), scale);
      if (a.levels) a.levels[base + idx] = int8_t(lv);
      ++idx;
    }
  }
}

// Group-64 fast path: the 64 decoded values of a group go to registers first
// and leave as 16 float4 / 4 int4 stores.
template <int FAM>
__global__ void __launch_bounds__(128) decode_g64(DecodeArgs a) {
  constexpr FamilyConst fc = family_const(FAM);
  const int64_t gi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gi >= a.groups) return;
  const DevLayout& L = a.L;
  const int64_t r = gi / L.gpr, gj = gi - r * L.gpr;
  const uint8_t* p = L.group(r, gj);

  // Stored words of the group, widened to code values.
  uint32_t code[22];
  uint32_t sc;
  if constexpr (FAM == kF206) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
    const WidenPlan pl = L.plan[r];
#pragma unroll
    for (int i = 0; i < 16; ++i) code[i] = widen_hi((wv[i / 4] >> (8 * (i % 4))) & 0xFF, pl) >> 8;
    sc = L.nibble(r, gj);
  } else if constexpr (FAM == kF25) {
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(p);  // 20 B, 4-B aligned
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint32_t v = p32[i];
      code[2 * i] = v & 0xFFFF;
      code[2 * i + 1] = v >> 16;
    }
    sc = code[9] & fc.scale_mask;
  } else {
    const uint16_t* p16 = reinterpret_cast<const uint16_t*>(p);  // 22 B, 2-B aligned
#pragma unroll
    for (int i = 0; i < 11; ++i) {
      const uint32_t v = p16[i];
      code[2 * i] = v & 0xFF;
      code[2 * i + 1] = v >> 8;
    }
    sc = code[21] & fc.scale_mask;
  }
  const float scale = __fmul_rn(float(sc), L.super[r]);

  int lv[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const int w = i / fc.wpw, k = i % fc.wpw;
    lv[i] = int((code[w] >> fc.shifts[w < (64 / fc.wpw) ? k : 0]) & fc.weight_mask) - fc.zero_point;
  }
  const int64_t base = gi * 64;  // cols == gpr * 64: groups are contiguous in the output
  if (a.weights) {
    float4* o = reinterpret_cast<float4*>(a.weights + base);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      o[i] = make_float4(__fmul_rn(float(lv[4 * i]), scale), __fmul_rn(float(lv[4 * i + 1]), scale),
                         __fmul_rn(float(lv[4 * i + 2]), scale),
                         __fmul_rn(float(lv[4 * i + 3]), scale));
  }
  if (a.levels) {
    int4* o = reinterpret_cast<int4*>(a.levels + base);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[j] = (uint32_t(lv[16 * i + 4 * j]) & 0xFF) | ((uint32_t(lv[16 * i + 4 * j + 1]) & 0xFF) << 8) |
               ((uint32_t(lv[16 * i + 4 * j + 2]) & 0xFF) << 16) |
               ((uint32_t(lv[16 * i + 4 * j + 3]) & 0xFF) << 24);
      o[i] = make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
    }
  }
}

template <int FAM>
int launch_fam(const ccq_dev_model* m, int8_t* levels, float* weights, cudaStream_t s) {
  DecodeArgs a{layout_of(m), levels, weights, m->rows * m->gpr};
  if (a.groups == 0) return CCQ_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(levels) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(weights) % 16 == 0);
  if (m->geo.group_size == 64 && aligned) {
    const unsigned blocks = unsigned((a.groups + 127) / 128);
    decode_g64<FAM><<<blocks, 128, 0, s>>>(a);
  } else {
    const unsigned blocks = unsigned((a.groups + 255) / 256);
    decode_generic<FAM><<<blocks, 256, 0, s>>>(a);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "decode launch");
}

}  // namespace

int launch_decode(const ccq_dev_model* m, int8_t* levels, float* weights, cudaStream_t s) {
  switch (m->family) {
    case kF275: return launch_fam<kF275>(m, levels, weights, s);
    case kF25: return launch_fam<kF25>(m, levels, weights, s);
    default: return launch_fam<kF206>(m, levels, weights, s);
  }
}

}  // namespace ccqb
