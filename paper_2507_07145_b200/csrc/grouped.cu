// Kernel (d) entry: grouped experts (MoE).
//
// No reference counterpart ships (SPEC.md:13, :395 put grouped-expert
// orchestration out of the reference's scope); the paper's Table 5 operator
// is a vLLM wna16 port.  Semantics: for each expert e, the
// token rows [offsets[e], offsets[e+1]) of x are multiplied by expert e's
// packed weights exactly as ccq::gemv_batch would (kernels.cpp:152-187).
#include <vector>

#include "ccq_internal.hpp"

using namespace ccqb;

extern "C" int ccq_cuda_grouped(const ccq_dev_model* const* models, int32_t E,
                                const int32_t* offsets_device, const int32_t* offsets_host,
                                const void* x, int x_dtype, void* y, int y_dtype, void* stream) {
  (void)offsets_device;
  if (!models || E < 0 || !offsets_host) return fail(CCQ_ERR_INVALID, "null experts or offsets");
  if (E == 0) return CCQ_OK;
  const ccq_dev_model* m0 = models[0];
  if (!m0) return fail(CCQ_ERR_INVALID, "null expert model");
  for (int e = 0; e < E; ++e) {
    const ccq_dev_model* m = models[e];
    if (!m || m->rows != m0->rows || m->cols != m0->cols || m->family != m0->family ||
        m->group_size != m0->group_size)
      return fail(CCQ_ERR_SHAPE, "experts must share shape, family and group size");
    if (offsets_host[e + 1] < offsets_host[e]) return fail(CCQ_ERR_SHAPE, "offsets must be non-decreasing");
  }
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  const size_t yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  for (int e = 0; e < E; ++e) {
    const int64_t n = offsets_host[e + 1] - offsets_host[e];
    if (n == 0) continue;
    const auto* xe = static_cast<const uint8_t*>(x) + size_t(offsets_host[e]) * m0->cols * xb;
    auto* ye = static_cast<uint8_t*>(y) + size_t(offsets_host[e]) * m0->rows * yb;
    const int st = ccq_cuda_matmul(models[e], xe, x_dtype, n, ye, y_dtype, stream);
    if (st != CCQ_OK) return st;
  }
  return CCQ_OK;
}
