// The reference's C++ API (include/ccq/*.hpp) implemented on top of the C ABI
// (include/ccq_cuda.h).  Signatures follow kernels.hpp:36-51,
// container.hpp:37-83, coding.hpp:115-150, packing.hpp:38-49 of the reference.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "ccq/coding.hpp"
#include "ccq/container.hpp"
#include "ccq/cuda.hpp"
#include "ccq/error.hpp"
#include "ccq/kernels.hpp"
#include "ccq/packing.hpp"
#include "ccq_cuda.h"

namespace ccq {

void throw_status(int st) {
  if (st == CCQ_OK) return;
  const std::string msg = ccq_cuda_last_error();
  switch (st) {
    case CCQ_ERR_CONFIG: throw ConfigError(msg);
    case CCQ_ERR_DOMAIN: throw DomainError(msg);
    case CCQ_ERR_SHAPE: throw ShapeError(msg);
    case CCQ_ERR_ENCODING: throw EncodingError(msg);
    case CCQ_ERR_FORMAT: throw FormatError(msg);
    case CCQ_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

std::string family_name(Family family) {
  switch (family) {
    case Family::Bpw275: return "2.75";
    case Family::Bpw25: return "2.5";
    case Family::Bpw206: return "2.06";
  }
  throw ConfigError("unknown family");
}

Family family_from_name(const std::string& name) {
  if (name == "2.75") return Family::Bpw275;
  if (name == "2.5" || name == "2.50") return Family::Bpw25;
  if (name == "2.06") return Family::Bpw206;
  throw ConfigError("unknown family '" + name + "' (expected 2.75, 2.5 or 2.06)");
}

std::uint16_t clustered_code_value(std::uint8_t q, float a, float b, int code_bits) {
  std::uint16_t out = 0;
  throw_status(ccq_clustered_code_value(q, a, b, code_bits, &out));
  return out;
}

GroupGeometry group_geometry(Family family, int group_size) {
  int32_t g[6];
  throw_status(ccq_group_geometry(int32_t(family), group_size, g));
  return GroupGeometry{g[0], g[1], g[2] != 0, g[3], g[4] != 0, g[5]};
}

namespace {

ccq_packed_view view_of(const PackedModel& m) {
  ccq_packed_view v{};
  v.rows = m.rows;
  v.cols = m.cols;
  v.family = int32_t(m.family);
  v.group_size = m.group_size;
  v.rounds = m.rounds;
  v.code_payload = m.code_payload.data();
  v.code_bytes = m.code_payload.size();
  v.scale_payload = m.scale_payload.empty() ? nullptr : m.scale_payload.data();
  v.scale_bytes = m.scale_payload.size();
  v.super_scales = m.super_scales.data();
  v.n_super_scales = m.super_scales.size();
  v.cluster_scales = m.cluster_scales.empty() ? nullptr : m.cluster_scales.data();
  v.n_cluster_scales = m.cluster_scales.size();
  v.cluster_zero_points = m.cluster_zero_points.empty() ? nullptr : m.cluster_zero_points.data();
  v.n_cluster_zero_points = m.cluster_zero_points.size();
  return v;
}

// Upload cache for the synchronous reference-signature calls.  PackedModel
// is immutable after load by contract; the key also covers the
// section pointers and sizes so a reallocated model re-uploads.
using Key = std::tuple<const PackedModel*, const void*, size_t, const void*, size_t, const void*,
                       int64_t, int64_t, int, int, int>;
std::mutex g_mu;
std::map<Key, ccq_dev_model*> g_cache;

const ccq_dev_model* device_copy(const PackedModel& m) {
  int dev = 0;
  cudaGetDevice(&dev);
  Key k{&m, m.code_payload.data(), m.code_payload.size(), m.scale_payload.data(),
        m.scale_payload.size(), m.super_scales.data(), m.rows, m.cols, int(m.family),
        m.group_size, dev};
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(k);
  if (it != g_cache.end()) return it->second;
  const ccq_packed_view v = view_of(m);
  ccq_dev_model* h = nullptr;
  throw_status(ccq_cuda_model_upload(&v, dev, &h));
  g_cache.emplace(k, h);
  return h;
}

}  // namespace

PackedModel load_model(const std::string& path) {
  ccq_packed_view v{};
  void* owner = nullptr;
  throw_status(ccq_container_open(path.c_str(), &v, &owner));
  PackedModel m;
  m.rows = v.rows;
  m.cols = v.cols;
  m.family = Family(v.family);
  m.group_size = v.group_size;
  m.rounds = v.rounds;
  m.code_payload.assign(v.code_payload, v.code_payload + v.code_bytes);
  if (v.scale_bytes) m.scale_payload.assign(v.scale_payload, v.scale_payload + v.scale_bytes);
  m.super_scales.assign(v.super_scales, v.super_scales + v.n_super_scales);
  if (v.n_cluster_scales) {
    m.cluster_scales.assign(v.cluster_scales, v.cluster_scales + v.n_cluster_scales);
    m.cluster_zero_points.assign(v.cluster_zero_points,
                                 v.cluster_zero_points + v.n_cluster_zero_points);
  }
  ccq_container_close(owner);
  return m;
}

Matrix dequantize(const PackedModel& model) {
  Matrix out(model.rows, model.cols);
  throw_status(ccq_dequantize_host(device_copy(model), out.data.data()));
  return out;
}

void gemv(const PackedModel& model, std::span<const float> x, std::span<float> y) {
  if (std::int64_t(x.size()) != model.cols || std::int64_t(y.size()) != model.rows)
    throw ShapeError("gemv operand sizes do not match the model shape");
  throw_status(ccq_gemv_host(device_copy(model), x.data(), x.size(), y.data(), y.size()));
}

void gemv_batch(const PackedModel& model, const Matrix& x, Matrix& y) {
  if (x.cols != model.cols || y.cols != model.rows || y.rows != x.rows)
    throw ShapeError("gemv_batch operand shapes do not match the model shape");
  throw_status(ccq_gemv_batch_host(device_copy(model), x.data.data(), x.rows, x.cols,
                                   y.data.data(), y.rows, y.cols));
}

void dense_gemv(const Matrix& weights, std::span<const float> x, std::span<float> y) {
  if (std::int64_t(x.size()) != weights.cols || std::int64_t(y.size()) != weights.rows)
    throw ShapeError("dense_gemv operand sizes do not match the matrix shape");
  for (std::int64_t r = 0; r < weights.rows; ++r) {
    const float* row = weights.row(r).data();
    double acc = 0.0;
    for (std::int64_t c = 0; c < weights.cols; ++c) acc += double(row[c]) * double(x[std::size_t(c)]);
    y[std::size_t(r)] = float(acc);
  }
}

std::uint64_t model_payload_bytes(const PackedModel& model) {
  return std::uint64_t(model.code_payload.size()) + model.scale_payload.size() +
         model.super_scales.size() * 4 + model.cluster_scales.size() * 4 +
         model.cluster_zero_points.size() * 4;
}

namespace cuda {

DeviceModel::DeviceModel(const PackedModel& model, int device, std::int64_t row_begin,
                         std::int64_t row_end) {
  const ccq_packed_view v = view_of(model);
  throw_status(ccq_cuda_model_upload_rows(&v, row_begin, row_end < 0 ? model.rows : row_end,
                                          device, &h_));
}

DeviceModel DeviceModel::load(const std::string& path, int device) {
  ccq_dev_model* h = nullptr;
  throw_status(ccq_cuda_model_load(path.c_str(), device, &h));
  return DeviceModel(h);
}

DeviceModel::~DeviceModel() {
  if (h_) ccq_cuda_model_free(h_);
}

DeviceModel& DeviceModel::operator=(DeviceModel&& o) noexcept {
  if (this != &o) {
    if (h_) ccq_cuda_model_free(h_);
    h_ = o.h_;
    o.h_ = nullptr;
  }
  return *this;
}

ccq_model_info DeviceModel::info() const {
  ccq_model_info i{};
  throw_status(ccq_cuda_model_info(h_, &i));
  return i;
}

void DeviceModel::decode(std::int8_t* levels, float* weights, void* stream) const {
  throw_status(ccq_cuda_decode(h_, levels, weights, stream));
}

void DeviceModel::matmul(const void* x, DType xd, std::int64_t M, void* y, DType yd,
                         void* stream) const {
  throw_status(ccq_cuda_matmul(h_, x, int(xd), M, y, int(yd), stream));
}

PackedModel quantize(const Matrix& weights, Family family, int group_size, int rounds, int device) {
  std::int32_t g[6];
  throw_status(ccq_group_geometry(std::int32_t(family), group_size, g));
  PackedModel m;
  m.rows = weights.rows;
  m.cols = weights.cols;
  m.family = family;
  m.group_size = group_size;
  m.rounds = rounds;
  const std::int64_t groups = group_size > 0 ? weights.rows * (weights.cols / group_size) : 0;
  m.code_payload.resize(std::size_t(groups) * std::size_t(g[5]));
  if (!g[4]) m.scale_payload.resize(std::size_t((groups + 1) / 2));
  m.super_scales.resize(std::size_t(weights.rows));
  if (family == Family::Bpw206) {
    m.cluster_scales.resize(std::size_t(weights.rows));
    m.cluster_zero_points.resize(std::size_t(weights.rows));
  }
  throw_status(ccq_quantize_host(weights.data.data(), weights.rows, weights.cols, std::int32_t(family), group_size,
                                 rounds, device, m.code_payload.data(),
                                 m.scale_payload.empty() ? nullptr : m.scale_payload.data(), m.super_scales.data(),
                                 m.cluster_scales.empty() ? nullptr : m.cluster_scales.data(),
                                 m.cluster_zero_points.empty() ? nullptr : m.cluster_zero_points.data()));
  return m;
}

}  // namespace cuda

}  // namespace ccq
