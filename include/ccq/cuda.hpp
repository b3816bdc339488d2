// Device-resident extension of the ccq API: explicit upload, device
// pointers, streams.  Thin RAII wrapper over ccq_cuda.h.
#ifndef CCQ_CUDA_HPP_
#define CCQ_CUDA_HPP_

#include <cstdint>
#include <string>

#include "ccq/container.hpp"
#include "ccq/tensor.hpp"
#include "ccq_cuda.h"

namespace ccq::cuda {

enum class DType { F32 = CCQ_DTYPE_F32, BF16 = CCQ_DTYPE_BF16, F16 = CCQ_DTYPE_F16 };

class DeviceModel {
 public:
  // Upload (optionally only output rows [row_begin, row_end)) to `device`.
  explicit DeviceModel(const PackedModel& model, int device = 0, std::int64_t row_begin = 0,
                       std::int64_t row_end = -1);
  static DeviceModel load(const std::string& path, int device = 0);
  ~DeviceModel();
  DeviceModel(DeviceModel&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceModel& operator=(DeviceModel&& o) noexcept;
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;

  ccq_model_info info() const;
  const ccq_dev_model* handle() const { return h_; }

  // Kernel (a): levels (int8) and/or f32 weights, device pointers, async.
  void decode(std::int8_t* levels, float* weights, void* stream = nullptr) const;
  // y[M x rows] = x[M x cols] W^T; device pointers, async on `stream`.
  void matmul(const void* x, DType x_dtype, std::int64_t M, void* y, DType y_dtype,
              void* stream = nullptr) const;

 private:
  explicit DeviceModel(ccq_dev_model* h) : h_(h) {}
  ccq_dev_model* h_ = nullptr;
};

// pack_model(quantize_tensor(weights, {family, group_size, rounds})) with the
// search, refinement, scale snapping, clustering and packing on `device`
// (quantizer.cpp:319-425, container.cpp:323-358); the sections are
// bit-identical to the reference's.  group_size <= 256.
PackedModel quantize(const Matrix& weights, Family family, int group_size = 64, int rounds = 2,
                     int device = 0);

}  // namespace ccq::cuda

#endif  // CCQ_CUDA_HPP_
