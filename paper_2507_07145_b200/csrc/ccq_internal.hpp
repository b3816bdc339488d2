// Internal definitions shared by the CCQ sm_100a kernels and the C ABI.
//
// Device layout of an uploaded model, "chunk-major records":
//   K is cut into nch chunks of kChunk = 32 groups; rows are padded to a
//   multiple of 16 (rows_pad).  The reference stores codes group-major per
//   row (container.hpp:44); on the device every (chunk c, row r) pair is one
//   self-contained, 16-byte aligned RECORD of `rec` bytes at
//       base + (c * rows_pad + r) * rec :
//     [0, cgb)          codes of groups 32c .. 32c+31 of row r, byte-identical
//                       to the reference payload (cgb = round16(32 * PB));
//     [cgb, cgb+16)     side-band scale nibbles of those groups (group j of
//                       the chunk in the low nibble of byte j/2 when j is
//                       even) - side-band families only;
//     [cgb+16, cgb+32)  the row's WidenPlan - clustered family only.
//   A warp streaming consecutive rows of one chunk therefore fetches ONE
//   contiguous region per tile with a single bulk copy.  Padding (rows, the
//   tail of the last chunk) is zero: zero scale codes contribute nothing.
//     super    f32[rows_pad]       per-row super scale (FORMAT.md §5)
//     plan     WidenPlan[rows_pad] (2.06) - same plans, row-major, for the
//              decode kernel; see WidenPlan below.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <utility>

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
// that can occur, with q placed in byte `pos` of a 32-bit word,
//     hi = (uint32)(( (uint64)(q << 8*pos) * M + C ) >> 32)
// satisfies  hi >> 8 == lround(double(q)*alpha + double(beta))  and
// hi < 2^23, i.e. hi carries the 15-bit code at bits [8,23) with 8 fraction
// bits below.  M = alpha * 2^(40-8*pos) is an exact integer (alpha is an
// f32), C = floor((beta + 0.5) * 2^40); the host builder verifies all 256 q
// against the reference double formula (model.cu: build_widen_plan).
// On the device the 64-bit multiply-add is ONE IMAD.HI.U32 (64-bit addend).
//   sel: bits 0-15  PRMT selector moving byte 0 of a word to byte `pos`
//                   (zeros elsewhere);
//        bits 16-31 1 << (4*pos): adding b * that selects byte b instead.
struct __align__(16) WidenPlan {
  uint64_t C;
  uint32_t M;
  uint32_t sel;
};

__host__ __device__ constexpr uint32_t plan_sel(uint32_t pos) {
  return ((0x4444u & ~(0xFu << (4 * pos))) & 0xFFFFu) | ((1u << (4 * pos)) << 16);
}
__host__ __device__ __forceinline__ uint32_t plan_pos(const WidenPlan& p) {
  const uint32_t step = p.sel >> 16;
  return step == 1 ? 0 : step == 16 ? 1 : step == 256 ? 2 : 3;
}
__host__ __device__ __forceinline__ uint32_t widen_hi(uint32_t q, const WidenPlan& p) {
  const uint64_t v = uint64_t(q << (8 * plan_pos(p))) * uint64_t(p.M) + p.C;
  return uint32_t(v >> 32);
}

constexpr int kChunk = 32;  // groups per K-chunk in the device layout

// Activation order of the tensor-core kernels for the 2.75 / 2.5 families
// (gemv_mma.cu, gemm_sm100.cu): 32 f16x2 "units" per 64-weight group, unit
// U = 8c + u; // (weight index within the group, field power p) of element e (0 = low half,
// 1 = high half) of unit u (0..7) produced by lane c (0..3).
struct WP {
  int w, p;
};
__host__ __device__ constexpr WP unit_wp(int fam, int c, int u, int e) {
  if (fam == kF206) {
    // natural order: unit u of lane c holds weights 16c + 2u + e (p-free magic)
    return WP{16 * c + 2 * u + e, 0};
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

// Read-only view of the device layout, passed to kernels by value.
struct DevLayout {
  const uint8_t* codes;  // record base
  const float* super;
  const WidenPlan* plan;
  const double2* plan64;  // 2.06 FP64 widening plans (may be null)
  int64_t rows, cols, gpr, rows_pad;
  uint32_t cgb;  // code bytes per record
  uint32_t rec;  // bytes per (chunk, row) record
  int nch;
  Geometry geo;

  __host__ __device__ __forceinline__ const uint8_t* record(int64_t c, int64_t r) const {
    return codes + (uint64_t(c) * rows_pad + r) * rec;
  }
  __host__ __device__ __forceinline__ const uint8_t* group(int64_t r, int64_t gj) const {
    return record(gj / kChunk, r) + (gj % kChunk) * geo.payload_bytes;
  }
  __host__ __device__ __forceinline__ uint32_t nibble(int64_t r, int64_t gj) const {
    const uint8_t b = record(gj / kChunk, r)[cgb + (gj % kChunk) / 2];
    return (b >> (4 * (gj & 1))) & 0xFu;
  }
};

}  // namespace ccqb

struct ccq_dev_model {
  int device = 0;
  int64_t rows = 0, cols = 0;
  int family = 0, group_size = 0, rounds = 0;
  ccqb::Geometry geo;
  int64_t gpr = 0;  // groups per row

  void* base = nullptr;
  size_t device_bytes = 0;
  uint8_t* codes = nullptr;  // records
  float* super = nullptr;
  ccqb::WidenPlan* plan = nullptr;
  uint32_t cgb = 0;      // code bytes per record
  uint32_t rec = 0;      // bytes per (chunk, row) record
  int nch = 0;           // K chunks
  int64_t rows_pad = 0;  // rows rounded up to 16

  uint64_t payload_bytes = 0;  // model_payload_bytes of the reference model
  int num_experts = 0;         // > 0: rows are num_experts stacked experts
  int64_t rows_per_expert = 0;
  bool fast = false;           // group-64 streaming kernels apply
  int plan_pos_min = 0;        // 2.06: smallest byte position of any real row's widening plan
  // 2.06: per-row FP64-pipe widening (A = 4096 alpha, B = beta + 1/2 - A as
  // doubles): code = floor(fma.rm(1 + q 2^-12, A, B)); verified at upload for
  // every valid q of every row (w64 = all rows exact).
  double2* plan64 = nullptr;
  bool w64 = false;
};

namespace ccqb {

inline DevLayout layout_of(const ccq_dev_model* m) {
  return DevLayout{m->codes, m->super, m->plan, m->plan64, m->rows, m->cols, m->gpr, m->rows_pad,
                   m->cgb, m->rec, m->nch, m->geo};
}

// Makes `d` the current device for the scope of a call (device-pointer entry
// points run on the model's device whatever the caller's current device is).
struct DeviceScope {
  int prev = 0;
  bool changed = false;
  explicit DeviceScope(int d) {
    cudaGetDevice(&prev);
    if (prev != d) changed = cudaSetDevice(d) == cudaSuccess;
  }
  ~DeviceScope() {
    if (changed) cudaSetDevice(prev);
  }
};

// Thread-local error message + status helpers.
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// Launch accounting (bench "gpu_launches").
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel in the stream is still running and must execute
// griddepcontrol.wait before it touches anything that kernel produces.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int geometry_for(int family, int group_size, Geometry* g);

// Kernel launchers (decode.cu, gemv.cu, gemm_sm100.cu, grouped.cu).
int launch_decode(const ccq_dev_model* m, int8_t* levels, float* weights, cudaStream_t s);
int launch_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                int y_dtype, cudaStream_t s);
int launch_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                int y_dtype, cudaStream_t s);
bool gemm_supported(const ccq_dev_model* m, int64_t M);
// Sync-free grouped GEMM over a device-side token-tile prefix (moe.cu).
int grouped_tile_tokens(const ccq_dev_model* stack, int64_t pairs, int E, int x_dtype);
int launch_grouped_gemm_tiles(const ccq_dev_model* stack, int E, int64_t rows_e, const int32_t* offsets_dev,
                              const int32_t* tile_prefix_dev, int64_t max_tiles, int64_t T, const void* x,
                              int x_dtype, void* y, int y_dtype, cudaStream_t s);
int launch_grouped_gemm(const ccq_dev_model* stack, int E, int64_t rows_e, const int32_t* offsets_dev,
                        int64_t T, int64_t max_tokens, const void* x, int x_dtype, void* y,
                        int y_dtype, cudaStream_t s, int bn = 0);
// token-tile width (64/128/160/192/256) minimising padded columns for the host routing
int grouped_bn_for(const ccq_dev_model* stack, const int32_t* offsets_host, int E, int x_dtype);
bool gemv_fast_supported(const ccq_dev_model* m, int64_t M);
// Kernel (b) on the tensor pipe (gemv_mma.cu): M <= kMmaMaxTokens per launch
// chunk, group size 64, all three families.
constexpr int kMmaMaxTokens = 16;
constexpr int kMmaMinTokens = 2;  // M = 1: CUDA-core streaming GEMV (gemv.cu)
bool gemv_mma_supported(const ccq_dev_model* m, int64_t M);
// smallest batch routed to the tensor-pipe GEMV (env CCQ_FORCE_MMA=1 -> 1, for tests)
int mma_min_tokens();
bool gemv_mma_fits(const ccq_dev_model* m, int64_t M);
int launch_grouped_stream(const ccq_dev_model* st, int E, int64_t rows_e, const int32_t* offsets_dev, int nhit,
                          const void* x, int x_dtype, void* y, int y_dtype, cudaStream_t s);
int launch_grouped_gemv(const ccq_dev_model* st, int E, int64_t rows_e, const int32_t* offsets_dev,
                        const int32_t* offsets_host, int64_t T, const void* x, int x_dtype, void* y,
                        int y_dtype, cudaStream_t s);
// Small-batch (M <= 8) tensor-pipe GEMV over shared-memory-resident weights
// (gemv_hmma.cu); kNotApplicable when the shape does not suit it.
constexpr int kNotApplicable = -1;
bool gemv_hmma_supported(const ccq_dev_model* m, int64_t M, int x_dtype, const void* x);
int launch_gemv_hmma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                     cudaStream_t s);
int launch_gemv_mma(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                    int y_dtype, cudaStream_t s);
int num_sms(int device);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `kern` on the CURRENT
// device, once per (kernel, device) and only when `bytes` grows; thread-safe
// (the attribute is per device, the library may drive several GPUs).
int ensure_smem(const void* kern, size_t bytes);
int max_smem_optin(int device);  // cached cudaDevAttrMaxSharedMemoryPerBlockOptin
// Library-owned stream-ordered memory pool of `device` (release threshold =
// unlimited, so per-call scratch does not re-map memory after every sync).
cudaMemPool_t scratch_pool(int device);

// 2-D tensor map over a row-major byte/half matrix (gemm_sm100.cu).
int make_map_2d(CUtensorMap* map, CUtensorMapDataType dt, void* base, uint64_t dim0, uint64_t dim1,
                uint64_t stride1_bytes, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw);

}  // namespace ccqb

#define CCQ_CUDA_TRY(expr)                                     \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::ccqb::cuda_fail(_e, #expr); \
  } while (0)
