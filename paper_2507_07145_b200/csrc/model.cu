#include <mutex>
// Packed-weight upload, per-row widening plans and the synchronous
// host-buffer entry points of the C ABI (include/ccq_cuda.h).
//
// Reference counterparts:
//   model_from_bytes validation       container.cpp:261-319
//   clustered_code_value              coding.hpp:142-150
//   dequantize / gemv / gemv_batch    kernels.cpp:103-187 (signatures kernels.hpp:36-43)
//   model_payload_bytes               kernels.cpp:203-207
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ccq_internal.hpp"

namespace ccqb {

namespace {
thread_local std::string g_err;
}

std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")";
  return CCQ_ERR_CUDA;
}

int geometry_for(int family, int group_size, Geometry* g) {
  if (family < 0 || family > 2) return fail(CCQ_ERR_CONFIG, "unknown family");
  const FamilyConst fc = family_const(family);
  if (group_size <= 0) return fail(CCQ_ERR_CONFIG, "group_size must be positive");
  const int rem = group_size % fc.wpw;
  if (rem > 1) {
    return fail(CCQ_ERR_CONFIG, "group_size " + std::to_string(group_size) + " leaves " +
                                    std::to_string(rem) +
                                    " weights in the last word; only remainders 0 and 1 have "
                                    "a layout");
  }
  if (family == kF25 && rem == 0)
    return fail(CCQ_ERR_CONFIG, "family 2.5 requires group_size % 7 == 1");
  g->group_size = group_size;
  g->full_words = group_size / fc.wpw;
  g->has_tail = rem == 1;
  g->words_per_group = g->full_words + g->has_tail;
  g->embedded_scale = g->has_tail && !fc.cluster;
  g->payload_bytes = g->words_per_group * fc.word_bytes;
  return CCQ_OK;
}

namespace {

// Reference widening (coding.hpp:144): lround in double.
inline long ref_widen(int q, float a, float b) {
  return std::lround(double(q) * double(a) + double(b));
}

// Builds the exact fixed-point plan of one row and marks the q values the
// reference would reject (result outside [0, 2^15)).  Returns false if no
// plan reproduces the reference for every valid q.
bool build_widen_plan(float alpha, float beta, WidenPlan* out, bool invalid[256]) {
  long ref[256];
  for (int q = 0; q < 256; ++q) {
    ref[q] = ref_widen(q, alpha, beta);
    invalid[q] = ref[q] < 0 || ref[q] >= 32768;
  }
  if (!std::isfinite(alpha) || !std::isfinite(beta)) {
    bool all_invalid = true;
    for (int q = 0; q < 256; ++q) all_invalid &= invalid[q];
    if (all_invalid) {
      *out = WidenPlan{0, 0, plan_sel(0)};
      return true;
    }
    return false;
  }
  // C = floor((beta + 1/2) * 2^40).  beta*2^40 is exact in double; floor is
  // exact below 2^53 and a no-op above.
  const int64_t C0 = int64_t(std::floor(std::ldexp(double(beta), 40))) + (int64_t(1) << 39);

  auto verify = [&](uint32_t M, uint32_t pos, int64_t C) {
    WidenPlan p{uint64_t(C), M, plan_sel(pos)};
    for (int q = 0; q < 256; ++q) {
      if (invalid[q]) continue;
      const uint32_t hi = widen_hi(uint32_t(q), p);
      if (long(hi >> 8) != ref[q] || hi >= (1u << 23)) return false;
    }
    *out = p;
    return true;
  };

  // Exact M: alpha * 2^(40 - 8*pos) integral and below 2^32.
  std::vector<std::pair<uint32_t, uint32_t>> cands;  // (M, pos)
  for (uint32_t pos : {2u, 1u, 3u, 0u}) {
    const double Md = std::ldexp(double(alpha), 40 - 8 * int(pos));
    if (Md >= 0.0 && Md < 4294967296.0 && Md == std::floor(Md)) cands.push_back({uint32_t(Md), pos});
  }
  // Approximate M (tiny or huge alpha): rounded, still verified exhaustively.
  for (uint32_t pos : {0u, 1u, 2u, 3u}) {
    const double Md = std::ldexp(double(alpha), 40 - 8 * int(pos));
    if (Md >= 0.0 && Md < 4294967295.5) cands.push_back({uint32_t(std::llround(Md)), pos});
  }
  static const int64_t nudges[] = {0,       1,        -1,        256,        -256,
                                   65536,   -65536,   1 << 24,   -(1 << 24), int64_t(1) << 30,
                                   -(int64_t(1) << 30), int64_t(1) << 34, -(int64_t(1) << 34)};
  for (const auto& [M, pos] : cands)
    for (int64_t d : nudges)
      if (verify(M, pos, C0 + d)) return true;
  return false;
}

size_t align_up(size_t n, size_t a) { return (n + a - 1) / a * a; }

}  // namespace

}  // namespace ccqb

namespace ccqb {

cudaMemPool_t scratch_pool(int device) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  if (device < 0 || device >= 64) device = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaDeviceGetDefaultMemPool(&pool, device);  // fall back to the default pool
    } else {
      uint64_t threshold = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    pools[device] = pool;
  }
  return pools[device];
}

}  // namespace ccqb

using namespace ccqb;

extern "C" {

const char* ccq_cuda_last_error(void) { return g_err.c_str(); }

const char* ccq_cuda_version(void) { return "ccq-b200 0.1 (sm_100a)"; }

uint64_t ccq_cuda_launch_count(void) { return g_launches.load(); }

int ccq_group_geometry(int32_t family, int32_t group_size, int32_t out6[6]) {
  Geometry g;
  const int st = geometry_for(family, group_size, &g);
  if (st != CCQ_OK) return st;
  out6[0] = g.group_size;
  out6[1] = g.full_words;
  out6[2] = g.has_tail;
  out6[3] = g.words_per_group;
  out6[4] = g.embedded_scale;
  out6[5] = g.payload_bytes;
  return CCQ_OK;
}

int ccq_clustered_code_value(uint8_t q, float alpha, float beta, int32_t code_bits,
                             uint16_t* out) {
  const long v = ref_widen(q, alpha, beta);
  if (v < 0 || v >= (1l << code_bits)) {
    return fail(CCQ_ERR_DOMAIN, "clustered code reconstructs outside [0, 2^" +
                                    std::to_string(code_bits) + "): q=" + std::to_string(int(q)));
  }
  *out = uint16_t(v);
  return CCQ_OK;
}

int ccq_cuda_model_upload_rows(const ccq_packed_view* v, int64_t r0, int64_t r1, int device,
                               ccq_dev_model** out) {
  if (!v || !out) return fail(CCQ_ERR_INVALID, "null view or output handle");
  *out = nullptr;
  Geometry geo;
  int st = geometry_for(v->family, v->group_size, &geo);
  if (st != CCQ_OK) return st;
  const FamilyConst fc = family_const(v->family);
  if (v->rows < 0 || v->cols < 0) return fail(CCQ_ERR_SHAPE, "negative shape");
  if (v->cols % v->group_size != 0)
    return fail(CCQ_ERR_FORMAT, "shape is not a whole number of groups");
  const int64_t gpr = v->cols / v->group_size;
  const uint64_t groups = uint64_t(v->rows) * uint64_t(gpr);
  if (v->code_bytes != groups * uint64_t(geo.payload_bytes) || (groups && !v->code_payload))
    return fail(CCQ_ERR_FORMAT, "codes section length does not match the geometry");
  if (!geo.embedded_scale) {
    if (v->scale_bytes != (groups + 1) / 2 || (groups && !v->scale_payload))
      return fail(CCQ_ERR_FORMAT, "group_scales section length does not match the group count");
  } else if (v->scale_bytes != 0) {
    return fail(CCQ_ERR_FORMAT, "embedded-scale family carries a side-band section");
  }
  if (v->n_super_scales != uint64_t(v->rows) || (v->rows && !v->super_scales))
    return fail(CCQ_ERR_FORMAT, "super_scales section length does not match the row count");
  if (fc.cluster) {
    if (v->n_cluster_scales != uint64_t(v->rows) || v->n_cluster_zero_points != uint64_t(v->rows) ||
        (v->rows && (!v->cluster_scales || !v->cluster_zero_points)))
      return fail(CCQ_ERR_FORMAT, "cluster_params section length does not match the row count");
  }
  if (r0 < 0 || r1 < r0 || r1 > v->rows) return fail(CCQ_ERR_SHAPE, "row range out of bounds");

  auto* m = new ccq_dev_model();
  m->device = device;
  m->rows = r1 - r0;
  m->cols = v->cols;
  m->family = v->family;
  m->group_size = v->group_size;
  m->rounds = v->rounds;
  m->geo = geo;
  m->gpr = gpr;
  const int64_t rows = m->rows;
  const uint64_t row_bytes = uint64_t(gpr) * geo.payload_bytes;
  m->nch = int((gpr + kChunk - 1) / kChunk);
  m->rows_pad = (rows + 15) / 16 * 16;
  m->cgb = uint32_t(align_up(size_t(kChunk) * geo.payload_bytes, 16));
  m->rec = m->cgb + (geo.embedded_scale ? 0u : 16u) + (fc.cluster ? 16u : 0u);
  m->payload_bytes = uint64_t(rows) * row_bytes +
                     (geo.embedded_scale ? 0 : (uint64_t(rows) * gpr + 1) / 2) + uint64_t(rows) * 4 +
                     (fc.cluster ? uint64_t(rows) * 8 : 0);

  // Host staging in the chunk-major record layout (ccq_internal.hpp).
  const int64_t rp = m->rows_pad;
  const size_t off_codes = 0;
  const size_t off_super = align_up(off_codes + size_t(m->nch) * size_t(rp) * m->rec, 256);
  const size_t off_plan = align_up(off_super + size_t(rp) * 4, 256);
  const size_t total = align_up(off_plan + (fc.cluster ? size_t(rp) * sizeof(WidenPlan) : 0), 256) + 256;
  std::vector<uint8_t> host(total, 0);
  auto rec_at = [&](int c, int64_t r) { return &host[off_codes + (size_t(c) * rp + r) * m->rec]; };
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t src = r0 + r;
    for (int c = 0; c < m->nch; ++c) {
      const int64_t g0 = int64_t(c) * kChunk;
      const int64_t ng = std::min<int64_t>(kChunk, gpr - g0);
      uint8_t* rec = rec_at(c, r);
      std::memcpy(rec, v->code_payload + uint64_t(src) * row_bytes + uint64_t(g0) * geo.payload_bytes,
                  size_t(ng) * geo.payload_bytes);
      if (!geo.embedded_scale) {
        uint8_t* dst = rec + m->cgb;
        for (int64_t j = 0; j < ng; ++j) {
          const uint64_t gi = uint64_t(src) * gpr + g0 + j;
          const uint8_t nib = (v->scale_payload[gi / 2] >> (4 * (gi % 2))) & 0xF;
          dst[j / 2] |= uint8_t(nib << (4 * (j % 2)));
        }
      }
    }
  }
  if (rows) std::memcpy(&host[off_super], v->super_scales + r0, size_t(rows) * 4);
  if (fc.cluster) {
    auto* plans = reinterpret_cast<WidenPlan*>(&host[off_plan]);
    for (int64_t r = rows; r < rp; ++r) plans[r] = WidenPlan{0, 0, plan_sel(0)};
    for (int64_t r = 0; r < rows; ++r) {
      bool invalid[256];
      const int64_t src = r0 + r;
      if (!build_widen_plan(v->cluster_scales[src], v->cluster_zero_points[src], &plans[r],
                            invalid)) {
        delete m;
        return fail(CCQ_ERR_DOMAIN, "row " + std::to_string(src) +
                                        ": cluster parameters have no exact fixed-point "
                                        "widening plan");
      }
      // The reference raises DomainError when it decodes such a byte
      // (coding.hpp:145-148); we raise it at upload for any stored byte.
      const uint8_t* row = v->code_payload + uint64_t(src) * row_bytes;
      for (uint64_t i = 0; i < row_bytes; ++i) {
        if (invalid[row[i]]) {
          delete m;
          return fail(CCQ_ERR_DOMAIN,
                      "clustered code reconstructs outside [0, 2^15): q=" +
                          std::to_string(int(row[i])) + " (row " + std::to_string(src) + ")");
        }
      }
    }
    for (int64_t r = 0; r < rp; ++r)
      for (int c = 0; c < m->nch; ++c)
        std::memcpy(rec_at(c, r) + m->cgb + 16, &plans[r], sizeof(WidenPlan));
    m->plan_pos_min = 3;
    for (int64_t r = 0; r < rows; ++r) m->plan_pos_min = std::min(m->plan_pos_min, int(plan_pos(plans[r])));
  }

  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&m->base, total);
  if (e == cudaSuccess) e = cudaMemcpy(m->base, host.data(), total, cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (m->base) cudaFree(m->base);
    delete m;
    return cuda_fail(e, "model upload");
  }
  auto* b = static_cast<uint8_t*>(m->base);
  m->device_bytes = total;
  m->codes = b + off_codes;
  m->super = reinterpret_cast<float*>(b + off_super);
  m->plan = fc.cluster ? reinterpret_cast<WidenPlan*>(b + off_plan) : nullptr;
  m->fast = geo.group_size == 64;
  *out = m;
  return CCQ_OK;
}

int ccq_cuda_model_upload(const ccq_packed_view* v, int device, ccq_dev_model** out) {
  if (!v) return fail(CCQ_ERR_INVALID, "null view");
  return ccq_cuda_model_upload_rows(v, 0, v->rows, device, out);
}

int ccq_cuda_model_free(ccq_dev_model* m) {
  if (!m) return CCQ_OK;
  if (m->base) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaFree(m->base);
    cudaSetDevice(prev);
  }
  delete m;
  return CCQ_OK;
}

int ccq_cuda_model_info(const ccq_dev_model* m, ccq_model_info* info) {
  if (!m || !info) return fail(CCQ_ERR_INVALID, "null model or info");
  std::memset(info, 0, sizeof(*info));
  info->rows = m->rows;
  info->cols = m->cols;
  info->family = m->family;
  info->group_size = m->group_size;
  info->rounds = m->rounds;
  info->device = m->device;
  info->payload_bytes_per_group = m->geo.payload_bytes;
  info->embedded_scale = m->geo.embedded_scale;
  info->payload_bytes = m->payload_bytes;
  info->device_bytes = m->device_bytes;
  info->code_row_stride = m->cgb;
  info->fast_path = m->fast ? 1 : 0;
  return CCQ_OK;
}

int ccq_model_payload_bytes(const ccq_dev_model* m, uint64_t* out) {
  if (!m || !out) return fail(CCQ_ERR_INVALID, "null model or output");
  *out = m->payload_bytes;
  return CCQ_OK;
}

int ccq_cuda_decode(const ccq_dev_model* m, int8_t* levels, float* weights, void* stream) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  if (!levels && !weights) return CCQ_OK;
  return launch_decode(m, levels, weights, static_cast<cudaStream_t>(stream));
}

static int check_dtypes(int x_dtype, int y_dtype) {
  if (x_dtype < 0 || x_dtype > 2) return fail(CCQ_ERR_CONFIG, "unsupported activation dtype");
  if (y_dtype != CCQ_DTYPE_F32 && y_dtype != CCQ_DTYPE_BF16)
    return fail(CCQ_ERR_CONFIG, "unsupported output dtype");
  return CCQ_OK;
}

int ccq_cuda_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  return launch_gemv(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

int ccq_cuda_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  if (!gemm_supported(m, M))
    return fail(CCQ_ERR_CONFIG, "tcgen05 GEMM needs group_size 64 and cols % 64 == 0");
  return launch_gemm(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

int ccq_cuda_matmul(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                    int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  // Dispatch by batch (measured, profiles/r01_sweep.json): M = 1 on the
  // CUDA-core streaming GEMV; 2 <= M <= 8 (2.06: see below; bf16/f16 activations) on the
  // tensor-pipe GEMV when all tokens fit one launch; the tcgen05 GEMM above
  // that, or when the activations would not fit; f32 activations (the
  // reference's own f32 API) take the streaming GEMV at M = 1 and the GEMM's
  // exact hi/lo split otherwise.
  const bool mma = x_dtype != CCQ_DTYPE_F32 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                   gemv_mma_supported(m, M);
  // 2.06 hands over to the GEMM earlier when the GEMM fills the SMs (>= 3/4
  // of them with 128-row tiles x split-K): at M = 8, and at M >= 3 on
  // K-heavy layers (cols > rows: few 16-row tiles but long x staging for the
  // tensor-pipe GEMV) (profiles/r01_dispatch_thresholds.txt).
  bool gemm_earlier = false;
  if (m->family == kF206 && (M >= 8 || (m->cols > m->rows && M >= 3))) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = num_sms(dev);
    const int64_t tiles = (m->rows + 127) / 128, cblocks = (m->gpr + 7) / 8;
    const int64_t splits = tiles * 2 <= sms && cblocks >= 8 ? std::min<int64_t>(sms / tiles, cblocks / 4) : 1;
    gemm_earlier = tiles * std::max<int64_t>(splits, 1) * 4 >= int64_t(sms) * 3;
  }
  if (mma && M >= mma_min_tokens() &&
      ((gemv_mma_fits(m, M) && !(gemm_earlier && gemm_supported(m, M))) || !gemm_supported(m, M)))
    return launch_gemv_mma(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
  if (!gemv_fast_supported(m, M) && gemm_supported(m, M))
    return launch_gemm(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
  return launch_gemv(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

// ---- synchronous host-buffer entry points ----

namespace {

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

// Scratch for the synchronous host entry points: stream-ordered allocations
// from the library pool on the legacy stream (no cudaMalloc per call).
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, nullptr);
  }
};

cudaError_t scratch_alloc(void** p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  return cudaMallocFromPoolAsync(p, bytes, ccqb::scratch_pool(dev), nullptr);
}

}  // namespace

int ccq_dequantize_host(const ccq_dev_model* m, float* out) {
  if (!m || (!out && m->rows * m->cols)) return fail(CCQ_ERR_INVALID, "null model or output");
  const size_t n = size_t(m->rows) * size_t(m->cols);
  if (n == 0) return CCQ_OK;
  DeviceScope ds(m->device);
  DevBuf w;
  CCQ_CUDA_TRY(scratch_alloc(&w.p, n * 4));
  int st = launch_decode(m, nullptr, static_cast<float*>(w.p), nullptr);
  if (st != CCQ_OK) return st;
  CCQ_CUDA_TRY(cudaMemcpy(out, w.p, n * 4, cudaMemcpyDeviceToHost));
  return CCQ_OK;
}

int ccq_gemv_batch_host(const ccq_dev_model* m, const float* x, int64_t x_rows, int64_t x_cols,
                        float* y, int64_t y_rows, int64_t y_cols) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  // kernels.cpp:153-155
  if (x_cols != m->cols || y_cols != m->rows || y_rows != x_rows)
    return fail(CCQ_ERR_SHAPE, "gemv_batch operand shapes do not match the model shape");
  if (x_rows == 0 || m->rows == 0) return CCQ_OK;
  if (m->cols == 0) {
    std::memset(y, 0, sizeof(float) * size_t(y_rows * y_cols));
    return CCQ_OK;
  }
  DeviceScope ds(m->device);
  DevBuf dx, dy;
  CCQ_CUDA_TRY(scratch_alloc(&dx.p, size_t(x_rows * x_cols) * 4));
  CCQ_CUDA_TRY(scratch_alloc(&dy.p, size_t(y_rows * y_cols) * 4));
  CCQ_CUDA_TRY(cudaMemcpy(dx.p, x, size_t(x_rows * x_cols) * 4, cudaMemcpyHostToDevice));
  int st = ccq_cuda_matmul(m, dx.p, CCQ_DTYPE_F32, x_rows, dy.p, CCQ_DTYPE_F32, nullptr);
  if (st != CCQ_OK) return st;
  CCQ_CUDA_TRY(cudaMemcpy(y, dy.p, size_t(y_rows * y_cols) * 4, cudaMemcpyDeviceToHost));
  return CCQ_OK;
}

int ccq_gemv_host(const ccq_dev_model* m, const float* x, uint64_t x_len, float* y,
                  uint64_t y_len) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  // kernels.cpp:125-127
  if (int64_t(x_len) != m->cols || int64_t(y_len) != m->rows)
    return fail(CCQ_ERR_SHAPE, "gemv operand sizes do not match the model shape");
  return ccq_gemv_batch_host(m, x, 1, m->cols, y, 1, m->rows);
}

}  // extern "C"
