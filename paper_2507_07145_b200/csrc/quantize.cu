// Exhaustive trellis code search on the GPU - the inner step of the CCQ
// quantizer: ccq::search_codes (quantizer.cpp:36-103)
// for a batch of subvectors, bit-identical to the reference.
//
// For every subvector the reference walks all 2^(L + (valid-1)S) leaves of
// the code trellis (first window: L bits, every further window: S fresh
// bits), costs each leaf as  sum_j (x_j - (state_j - zp) * scale)^2  in
// double, added left to right, and keeps the first minimum in ascending code
// order.  Here one warp owns a subvector: its per-position cost tables
// (valid x 2^L doubles, the reference's `tables`) sit in shared memory, lanes
// take leaves lane, lane+32, ... (ascending, strict <), and a warp reduction
// picks the minimum cost, ties to the smaller code - the same answer as the
// sequential scan.  Products and sums are rounded separately
// (__dmul_rn/__dsub_rn/__dadd_rn): no FMA contraction, as in the reference's
// x86-64 build.
#include <algorithm>
#include <string>

#include "ccq_internal.hpp"

namespace ccqb {
namespace {

__global__ void __launch_bounds__(256) search_codes_kernel(const float* __restrict__ targets, int64_t n,
                                                           int valid, int stride, const double* __restrict__ scales,
                                                           int zp, int L, int N, int S,
                                                           uint32_t* __restrict__ codes) {
  extern __shared__ double tabs[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int nst = 1 << L;
  double* t = tabs + size_t(wib) * valid * nst;
  const uint32_t smask = uint32_t(nst - 1), fmask = (1u << S) - 1u;
  const int lbits = L + (valid - 1) * S;
  const uint32_t nleaf = 1u << lbits;
  for (int64_t i = int64_t(blockIdx.x) * wpb + wib; i < n; i += int64_t(gridDim.x) * wpb) {
    const double scale = scales[i];
    for (int e = lane; e < valid * nst; e += 32) {
      const int j = e / nst, s = e - j * nst;
      const double d = __dsub_rn(double(targets[i * stride + j]), __dmul_rn(double(s - zp), scale));
      t[e] = __dmul_rn(d, d);
    }
    __syncwarp();
    double best = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    uint32_t bcode = 0;
    for (uint32_t leaf = lane; leaf < nleaf; leaf += 32) {
      uint32_t st = leaf >> ((valid - 1) * S);
      double acc = t[st];
      for (int j = 1; j < valid; ++j) {
        const uint32_t f = (leaf >> ((valid - 1 - j) * S)) & fmask;
        st = ((st << S) | f) & smask;
        acc = __dadd_rn(acc, t[j * nst + st]);
      }
      if (acc < best) {
        best = acc;
        bcode = leaf;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcode, off);
      if (ob < best || (ob == best && oc < bcode)) {
        best = ob;
        bcode = oc;
      }
    }
    if (lane == 0) codes[i] = bcode << ((N - valid) * S);
    __syncwarp();  // the table is rewritten for the next subvector
  }
}

}  // namespace
}  // namespace ccqb

using namespace ccqb;

extern "C" int ccq_cuda_search_codes(const float* targets, int64_t n, int32_t valid, int32_t stride,
                                     const double* scales, int32_t zero_point, int32_t state_bits,
                                     int32_t states_per_code, int32_t transition_bits, uint32_t* codes,
                                     void* stream) {
  // EncodingConfig::validate (coding.cpp:38-57) and search_codes' shape check
  const int L = state_bits, N = states_per_code, S = transition_bits;
  if (N < 1 || S < 1 || S > L || L > 8 || L + (N - 1) * S > 16)
    return fail(CCQ_ERR_CONFIG, "encoding config needs 1 <= S <= L <= 8, N >= 1 and L + (N-1)S <= 16");
  if (valid < 1 || valid > N)
    return fail(CCQ_ERR_SHAPE, "search target must hold 1.." + std::to_string(N) + " values, got " +
                                   std::to_string(valid));
  if (n < 0 || stride < valid) return fail(CCQ_ERR_SHAPE, "bad subvector count or stride");
  if (n == 0) return CCQ_OK;
  if (!targets || !scales || !codes) return fail(CCQ_ERR_INVALID, "null pointer");
  const size_t per_warp = size_t(valid) * size_t(1 << L) * sizeof(double);  // <= 16 x 256 x 8 B
  const int wpb = int(std::min<size_t>(8, (200 * 1024) / per_warp));
  const size_t smem = size_t(wpb) * per_warp;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t blocks = std::min<int64_t>((n + wpb - 1) / wpb, int64_t(num_sms(dev)) * 16);
  static size_t configured = 0;
  if (smem > 48 * 1024 && configured < smem) {
    CCQ_CUDA_TRY(cudaFuncSetAttribute(search_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    configured = smem;
  }
  search_codes_kernel<<<unsigned(blocks), wpb * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      targets, n, valid, stride, scales, zero_point, L, N, S, codes);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "search_codes launch");
}
