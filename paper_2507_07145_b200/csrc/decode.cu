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
#include <algorithm>
#include <cstdlib>

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

// Group-64, record-major variant (the default): one warp per (row, K chunk)
// device record = 32 consecutive groups of one row, lane = group.  Each
// lane decodes its group into registers and stages it in shared memory (row
// stride padded by 16 B so the 8 lanes of a store phase hit distinct banks);
// the warp then writes the record's 8 KB of f32 weights / 2 KB of levels
// back with fully coalesced 16-byte stores (512 contiguous bytes per warp
// instruction) instead of 32 scattered 16-byte pieces.  The kernel is bound
// by HBM writes (4-5 B per weight out vs 0.26-0.34 B in).
constexpr int kDecWarps = 8;
constexpr int kWStride = 64 * 4 + 16;  // bytes per staged group, f32
constexpr int kLStride = 64 + 16;      // bytes per staged group, int8

template <int FAM>
__device__ __forceinline__ void group_levels(const uint8_t* p, const WidenPlan& pl, uint32_t nibble_code,
                                             int (&lv)[64], uint32_t* sc_out) {
  constexpr FamilyConst fc = family_const(FAM);
  uint32_t code[22];
  uint32_t sc;
  if constexpr (FAM == kF206) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) code[i] = widen_hi((wv[i / 4] >> (8 * (i % 4))) & 0xFF, pl) >> 8;
    sc = nibble_code;
  } else if constexpr (FAM == kF25) {
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint32_t v = p32[i];
      code[2 * i] = v & 0xFFFF;
      code[2 * i + 1] = v >> 16;
    }
    sc = code[9] & fc.scale_mask;
  } else {
    const uint16_t* p16 = reinterpret_cast<const uint16_t*>(p);
#pragma unroll
    for (int i = 0; i < 11; ++i) {
      const uint32_t v = p16[i];
      code[2 * i] = v & 0xFF;
      code[2 * i + 1] = v >> 8;
    }
    sc = code[21] & fc.scale_mask;
  }
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const int w = i / fc.wpw, k = i % fc.wpw;
    lv[i] = int((code[w] >> fc.shifts[w < (64 / fc.wpw) ? k : 0]) & fc.weight_mask) - fc.zero_point;
  }
  *sc_out = sc;
}

template <int FAM>
__global__ void __launch_bounds__(kDecWarps * 32) decode_rec(DecodeArgs a) {
  constexpr FamilyConst fc = family_const(FAM);
  extern __shared__ __align__(16) uint8_t dsm[];
  const DevLayout& L = a.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* wst = dsm + size_t(warp) * 32 * (kWStride + kLStride);
  uint8_t* lst = wst + 32 * kWStride;
  const int64_t nrec = L.rows * L.nch;
  for (int64_t w = int64_t(blockIdx.x) * kDecWarps + warp; w < nrec; w += int64_t(gridDim.x) * kDecWarps) {
    const int64_t r = w / L.nch;
    const int c = int(w - r * L.nch);
    const int ng = int(L.gpr - int64_t(c) * kChunk < kChunk ? L.gpr - int64_t(c) * kChunk : kChunk);
    const uint8_t* rec = L.record(c, r);
    if (lane < ng) {
      WidenPlan pl{};
      uint32_t nib = 0;
      if constexpr (fc.cluster) {
        const uint4 pv = *reinterpret_cast<const uint4*>(rec + L.cgb + 16);
        pl.C = uint64_t(pv.x) | (uint64_t(pv.y) << 32);
        pl.M = pv.z;
        pl.sel = pv.w;
        nib = (rec[L.cgb + lane / 2] >> (4 * (lane & 1))) & 0xFu;
      }
      int lv[64];
      uint32_t sc;
      group_levels<FAM>(rec + lane * L.geo.payload_bytes, pl, nib, lv, &sc);
      if (a.weights) {
        const float scale = __fmul_rn(float(sc), L.super[r]);
        float4* o = reinterpret_cast<float4*>(wst + lane * kWStride);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          o[i] = make_float4(__fmul_rn(float(lv[4 * i]), scale), __fmul_rn(float(lv[4 * i + 1]), scale),
                             __fmul_rn(float(lv[4 * i + 2]), scale), __fmul_rn(float(lv[4 * i + 3]), scale));
      }
      if (a.levels) {
        uint4* o = reinterpret_cast<uint4*>(lst + lane * kLStride);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[j] = (uint32_t(lv[16 * i + 4 * j]) & 0xFF) | ((uint32_t(lv[16 * i + 4 * j + 1]) & 0xFF) << 8) |
                   ((uint32_t(lv[16 * i + 4 * j + 2]) & 0xFF) << 16) |
                   ((uint32_t(lv[16 * i + 4 * j + 3]) & 0xFF) << 24);
          o[i] = make_uint4(v[0], v[1], v[2], v[3]);
        }
      }
    }
    __syncwarp();
    const int64_t col0 = int64_t(c) * kChunk * 64;
    if (a.weights) {  // ng * 16 float4s, 32 per instruction, contiguous in the output row
      float4* dst = reinterpret_cast<float4*>(a.weights + r * L.cols + col0);
      for (int f = lane; f < ng * 16; f += 32)
        __stcs(dst + f, *reinterpret_cast<const float4*>(wst + (f >> 4) * kWStride + (f & 15) * 16));
    }
    if (a.levels) {
      uint4* dst = reinterpret_cast<uint4*>(a.levels + r * L.cols + col0);
      for (int f = lane; f < ng * 4; f += 32)
        __stcs(reinterpret_cast<int4*>(dst + f),
               *reinterpret_cast<const int4*>(lst + (f >> 2) * kLStride + (f & 3) * 16));
    }
    __syncwarp();
  }
}

template <int FAM>
int launch_fam(const ccq_dev_model* m, int8_t* levels, float* weights, cudaStream_t s) {
  DecodeArgs a{layout_of(m), levels, weights, m->rows * m->gpr};
  if (a.groups == 0) return CCQ_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(levels) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(weights) % 16 == 0);
  static const bool legacy = std::getenv("CCQ_DECODE_G64") != nullptr;
  // levels alone (1 B per weight) are decode-bound, not store-bound: the
  // thread-per-group kernel's occupancy wins there (profiles/r02_decode.txt)
  if (m->geo.group_size == 64 && aligned && m->cols % 64 == 0 && !legacy && weights) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = size_t(kDecWarps) * 32 * (kWStride + kLStride);
    auto kern = decode_rec<FAM>;
    if (int st = ensure_smem(reinterpret_cast<const void*>(kern), smem)) return st;
    const int64_t nrec = m->rows * m->nch;
    const unsigned blocks = unsigned(std::min<int64_t>((nrec + kDecWarps - 1) / kDecWarps, int64_t(num_sms(dev)) * 2 * 4));
    kern<<<blocks, kDecWarps * 32, smem, s>>>(a);
  } else if (m->geo.group_size == 64 && aligned) {
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
