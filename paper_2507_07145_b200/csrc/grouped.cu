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

// ---------------------------------------------------------------------------
// Stacked experts: one device allocation, one launch (tcgen05 grouped GEMM).
// ---------------------------------------------------------------------------
extern "C" int ccq_cuda_experts_upload(const ccq_packed_view* views, int32_t E, int device,
                                       ccq_dev_model** out) {
  if (!views || !out || E <= 0) return fail(CCQ_ERR_INVALID, "null experts or E <= 0");
  const ccq_packed_view& v0 = views[0];
  for (int e = 0; e < E; ++e) {
    const ccq_packed_view& v = views[e];
    if (v.rows != v0.rows || v.cols != v0.cols || v.family != v0.family || v.group_size != v0.group_size)
      return fail(CCQ_ERR_SHAPE, "experts must share shape, family and group size");
  }
  // Concatenate the experts' sections (rows of expert e follow expert e-1);
  // side-band nibbles are concatenated at nibble granularity.
  std::vector<uint8_t> code, scale;
  std::vector<float> sup, cs, czp;
  const uint64_t groups_e = v0.group_size > 0 ? uint64_t(v0.rows) * uint64_t(v0.cols / v0.group_size) : 0;
  for (int e = 0; e < E; ++e) {
    const ccq_packed_view& v = views[e];
    code.insert(code.end(), v.code_payload, v.code_payload + v.code_bytes);
    sup.insert(sup.end(), v.super_scales, v.super_scales + v.n_super_scales);
    if (v.n_cluster_scales) {
      cs.insert(cs.end(), v.cluster_scales, v.cluster_scales + v.n_cluster_scales);
      czp.insert(czp.end(), v.cluster_zero_points, v.cluster_zero_points + v.n_cluster_zero_points);
    }
  }
  if (v0.scale_bytes) {
    scale.assign((groups_e * E + 1) / 2, 0);
    for (int e = 0; e < E; ++e) {
      if (views[e].scale_bytes != (groups_e + 1) / 2)
        return fail(CCQ_ERR_FORMAT, "group_scales section length does not match the group count");
      for (uint64_t i = 0; i < groups_e; ++i) {
        const uint8_t nib = (views[e].scale_payload[i / 2] >> (4 * (i % 2))) & 0xF;
        const uint64_t gi = uint64_t(e) * groups_e + i;
        scale[gi / 2] |= uint8_t(nib << (4 * (gi % 2)));
      }
    }
  }
  ccq_packed_view all = v0;
  all.rows = v0.rows * E;
  all.code_payload = code.data();
  all.code_bytes = code.size();
  all.scale_payload = scale.empty() ? nullptr : scale.data();
  all.scale_bytes = scale.size();
  all.super_scales = sup.data();
  all.n_super_scales = sup.size();
  all.cluster_scales = cs.empty() ? nullptr : cs.data();
  all.n_cluster_scales = cs.size();
  all.cluster_zero_points = czp.empty() ? nullptr : czp.data();
  all.n_cluster_zero_points = czp.size();
  const int st = ccq_cuda_model_upload(&all, device, out);
  if (st != CCQ_OK) return st;
  (*out)->num_experts = E;
  (*out)->rows_per_expert = v0.rows;
  return CCQ_OK;
}

extern "C" int ccq_cuda_experts_matmul(const ccq_dev_model* stack, const int32_t* offsets_device,
                                       const int32_t* offsets_host, const void* x, int x_dtype,
                                       void* y, int y_dtype, void* stream) {
  if (!stack || !offsets_host || stack->num_experts <= 0)
    return fail(CCQ_ERR_INVALID, "not a stacked-expert model or null offsets");
  DeviceScope ds(stack->device);
  const int E = stack->num_experts;
  const int64_t re = stack->rows_per_expert;
  int64_t max_tokens = 0;
  for (int e = 0; e < E; ++e) {
    const int64_t n = int64_t(offsets_host[e + 1]) - offsets_host[e];
    if (n < 0 || offsets_host[0] != 0) return fail(CCQ_ERR_SHAPE, "offsets must start at 0 and be non-decreasing");
    max_tokens = n > max_tokens ? n : max_tokens;
  }
  const int64_t T = offsets_host[E];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (max_tokens == 1) {  // one token per routed expert: the CUDA-core streaming GEMV, one launch
    int nhit = 0;
    for (int e = 0; e < E; ++e) nhit += offsets_host[e + 1] > offsets_host[e];
    const int st = launch_grouped_stream(stack, E, re, offsets_device, nhit, x, x_dtype, y, y_dtype, s);
    if (st != 1) return st;
  }
  {  // decode batches: one tensor-pipe GEMV launch over the routed experts' tiles
    const int st = launch_grouped_gemv(stack, E, re, offsets_device, offsets_host, T, x, x_dtype, y, y_dtype, s);
    if (st != 1) return st;
  }
  if (offsets_device && gemm_supported(stack, max_tokens))
    return launch_grouped_gemm(stack, E, re, offsets_device, T, max_tokens, x, x_dtype, y, y_dtype, s,
                               grouped_bn_for(stack, offsets_host, E, x_dtype));
  // Other families: one fused decode-matmul per expert with tokens, on a
  // shallow per-expert view of the stacked device layout.
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  const size_t yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  for (int e = 0; e < E; ++e) {
    const int64_t n = int64_t(offsets_host[e + 1]) - offsets_host[e];
    if (n == 0) continue;
    ccq_dev_model view = *stack;
    view.rows = re;
    view.codes = stack->codes + uint64_t(e) * re * stack->rec;  // same chunk stride (rows_pad)
    view.super = stack->super + e * re;
    view.plan = stack->plan ? stack->plan + e * re : nullptr;
    view.plan64 = stack->plan64 ? stack->plan64 + e * re : nullptr;
    view.num_experts = 0;
    const auto* xe = static_cast<const uint8_t*>(x) + size_t(offsets_host[e]) * stack->cols * xb;
    auto* ye = static_cast<uint8_t*>(y) + size_t(offsets_host[e]) * re * yb;
    const int st = ccq_cuda_matmul(&view, xe, x_dtype, n, ye, y_dtype, stream);
    if (st != CCQ_OK) return st;
  }
  return CCQ_OK;
}
