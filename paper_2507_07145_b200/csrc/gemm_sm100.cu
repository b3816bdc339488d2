// Kernel (c): tcgen05 GEMM with in-shared-memory tile decode (placeholder
// until the tcgen05 path lands).
#include "ccq_internal.hpp"

namespace ccqb {

bool gemm_supported(const ccq_dev_model*, int64_t) { return false; }

int launch_gemm(const ccq_dev_model*, const void*, int, int64_t, void*, int, cudaStream_t) {
  return fail(CCQ_ERR_CONFIG, "tcgen05 GEMM not available");
}

}  // namespace ccqb
