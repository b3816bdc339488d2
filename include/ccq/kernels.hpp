// The inference kernels - same signatures as the reference's kernels.hpp
// (kernels.hpp:36-51).  Implemented on the GPU (libccq_b200.so): the first
// call with a given PackedModel uploads it to the current CUDA device (cached
// per model object), every call is synchronous like the reference's.
// dequantize is bit-exact; gemv / gemv_batch accumulate in f32 (relative
// Frobenius error vs the reference's double accumulation <= 1e-3, measured
// <= 5e-5).
#ifndef CCQ_KERNELS_HPP_
#define CCQ_KERNELS_HPP_

#include <cstdint>
#include <span>

#include "ccq/container.hpp"
#include "ccq/tensor.hpp"

namespace ccq {

Matrix dequantize(const PackedModel& model);
void gemv(const PackedModel& model, std::span<const float> x, std::span<float> y);
void gemv_batch(const PackedModel& model, const Matrix& x, Matrix& y);
// Reference dense product (double accumulation, left to right) - host code,
// kept for drop-in completeness (kernels.cpp:189-201).
void dense_gemv(const Matrix& weights, std::span<const float> x, std::span<float> y);
std::uint64_t model_payload_bytes(const PackedModel& model);

}  // namespace ccq

#endif  // CCQ_KERNELS_HPP_
