// Internal definitions shared by the CCQ sm_100a kernels and the C ABI.
//
// Device layout of an uploaded model:
//   codes    rows x code_stride bytes; row r holds its groups exactly as in
//            the reference's group-major code_payload (container.hpp:44),
//            padded to a 16-byte row stride so every row (and every 32-group
//            chunk at group size 64) starts on a 16-byte boundary for
//            cp.async.bulk / 128-bit loads.
//   nibbles  side-band scale nibbles re-laid out per row (row r starts at
//            byte r*nib_stride; group gj of the row in the low nibble of
//            byte gj/2 when gj is even), stride padded to 16 bytes.
//   super    f32[rows]   per-row super scale (FORMAT.md §5)
//   plan     WidenPlan[rows] (2.06 only): the exact fixed-point restatement of
//            clustered_code_value (coding.hpp:142-150), see widen() below.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "ccq_cuda.h"

namespace ccqb {

enum Family : int { kF275 = 0, kF25 = 1, kF206 = 2 };

// Per-family constants (coding.cpp:213-249, FORMAT.md §2).
struct FamilyConst {
  int code_bits, word_bytes, wpw, state_bits, zero_point, scale_bits, cluster, nshift;
  uint32_t weight_mask, scale_mask;
  int shifts[7];
};

__host__ __device__ constexpr FamilyConst family_const(int f) {
  return f == kF275 ? FamilyConst{8, 1, 3, 4, 8, 4, 0, 3, 0xFu, 0xFu, {4, 2, 0, 0, 0, 0, 0}}
         : f == kF25 ? FamilyConst{16, 2, 7, 3, 4, 13, 0, 7, 0x7u, 0x1FFFu, {13, 11, 9, 6, 4, 2, 0}}
                     : FamilyConst{15, 1, 4, 6, 32, 4, 1, 4, 0x3Fu, 0xFu, {9, 6, 3, 0, 0, 0, 0}};
}

// Group geometry (packing.cpp:24-47).
struct Geometry {
  int group_size = 0, full_words = 0, has_tail = 0, words_per_group = 0, embedded_scale = 0,
      payload_bytes = 0;
};

// Exact fixed-point widening plan of one row (2.06).  For every stored byte q
// that can occur,
//     hi = (uint32)(( (uint64)(q << sh) * M + C ) >> 32)
// satisfies  hi >> 8 == lround(double(q)*alpha + double(beta))  and
// hi < 2^23, i.e. hi carries the 15-bit code at bits [8,23) with 8 fraction
// bits below.  M = alpha * 2^(40-sh) is an exact integer (alpha is an f32),
// C = floor((beta + 0.5) * 2^40); the host builder verifies all 256 q
// against the reference double formula (model.cu: build_widen_plan).
struct __align__(16) WidenPlan {
  uint64_t C;
  uint32_t M;
  uint32_t sh;  // 0, 8, 16 or 24
};

__host__ __device__ __forceinline__ uint32_t widen_hi(uint32_t q, const WidenPlan& p) {
  const uint64_t v = uint64_t(q << p.sh) * uint64_t(p.M) + p.C;
  return uint32_t(v >> 32);
}

}  // namespace ccqb

struct ccq_dev_model {
  int device = 0;
  int64_t rows = 0, cols = 0;
  int family = 0, group_size = 0, rounds = 0;
  ccqb::Geometry geo;
  int64_t gpr = 0;  // groups per row

  void* base = nullptr;
  size_t device_bytes = 0;
  uint8_t* codes = nullptr;
  uint64_t code_stride = 0;
  uint8_t* nibbles = nullptr;
  uint64_t nib_stride = 0;
  float* super = nullptr;
  ccqb::WidenPlan* plan = nullptr;

  uint64_t payload_bytes = 0;  // model_payload_bytes of the reference model
  bool fast = false;           // group-64 streaming kernels apply
};

namespace ccqb {

// Thread-local error message + status helpers.
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// Launch accounting (bench "gpu_launches").
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int geometry_for(int family, int group_size, Geometry* g);

// Kernel launchers (decode.cu, gemv.cu, gemm_sm100.cu, grouped.cu).
int launch_decode(const ccq_dev_model* m, int8_t* levels, float* weights, cudaStream_t s);
int launch_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                int y_dtype, cudaStream_t s);
int launch_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                int y_dtype, cudaStream_t s);
bool gemm_supported(const ccq_dev_model* m, int64_t M);
bool gemv_fast_supported(const ccq_dev_model* m, int64_t M);

}  // namespace ccqb

#define CCQ_CUDA_TRY(expr)                                     \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::ccqb::cuda_fail(_e, #expr); \
  } while (0)
