// The inference kernels and the bench report - same signatures as the
// reference's kernels.hpp (kernels.hpp:33-76).  Implemented on the GPU
// (libccq_b200.so): a call uploads the PackedModel to the current CUDA device
// (a bounded cache keyed by a hash of the section CONTENTS, so a changed or
// re-created model is never served stale bytes), and every call is
// synchronous like the reference's.
// dequantize is bit-exact; gemv / gemv_batch accumulate in f32 (relative
// Frobenius error vs the reference's double accumulation <= 1e-3, measured
// <= 5e-5).
#ifndef CCQ_KERNELS_HPP_
#define CCQ_KERNELS_HPP_

#include <cstdint>
#include <span>
#include <string>
#include <vector>

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

// One timing row of the reference's bench report (kernels.hpp:53-64).
// bytes_read counts weight-stream bytes only: dense variants rows*cols*4,
// the fused variants model_payload_bytes, dequantize-then-dense both.
struct BenchRow {
  std::int64_t d_in = 0;   // cols
  std::int64_t d_out = 0;  // rows
  int batch = 1;
  std::string variant;
  double median_ms = 0.0;
  std::uint64_t bytes_read = 0;
};

// The reference's three variants, same meaning and byte accounting
// (kernels.cpp:228-279): dense_f32 (dense_gemv on the dequantized matrix,
// host), dequant_then_dense (GPU dequantize + host dense_gemv) and ccq_fused
// (gemv_batch: host buffers in and out, decode + matmul on the GPU) - plus
// ccq_gpu_fused: the same product on device-resident activations, CUDA-event
// timed.  ConfigError for iterations < 1 or a batch < 1.
std::vector<BenchRow> bench_model(const PackedModel& model, const std::vector<int>& batches,
                                  int iterations, std::uint64_t seed);
std::string bench_csv(const std::vector<BenchRow>& rows);  // shape,M,variant,median_ms,bytes_read
std::vector<BenchRow> parse_bench_csv(const std::string& csv);  // FormatError

}  // namespace ccq

#endif  // CCQ_KERNELS_HPP_
