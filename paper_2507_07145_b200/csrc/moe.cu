// MoE token routing around kernel (d): natural-order
// tokens + router top-k -> expert-major permutation -> grouped decode-matmul
// -> weighted combine back to token order.
//
//   y[t] = sum_j w[t, j] * W_{e(t, j)} x[t]        (j = 0..k-1, fixed order)
//
// Steps (all on `stream`):
//   1. per-expert counts of the T*k routed pairs (atomics), exclusive scan;
//   2. scatter: each pair gets a slot in its expert's contiguous row range and
//      its token's activation row is copied there (slot order inside an expert
//      is arbitrary - every routed row is computed independently, so the
//      result does not depend on it);
//   3. the grouped kernel (one launch) on the expert-major rows;
//   4. combine: per token, the k weighted expert outputs summed in j order
//      (f32, deterministic).
// Nothing comes back to the host: the scan also writes a per-expert token-tile
// prefix and the grouped tcgen05 GEMM reads its work list from the device
// (grid sized for the worst case), so the call is stream-ordered end to end
// and can be captured in a CUDA graph.  Router ids outside [0, E) are
// dropped (their pairs contribute zero); callers that want an error check
// the ids themselves (the Python wrapper does by default).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "ccq_internal.hpp"

namespace ccqb {
namespace {

__global__ void moe_count(const int32_t* __restrict__ ids, int64_t pairs, int E, int32_t* __restrict__ counts) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < pairs; i += int64_t(gridDim.x) * blockDim.x) {
    const int e = ids[i];
    if (e >= 0 && e < E) atomicAdd(&counts[e], 1);
  }
}

// offsets[e] = sum of counts[<e]; cursor = offsets; tiles[e] = sum of
// ceil(counts[<e] / tb) (single CTA, E <= 4096)
__global__ void moe_scan(const int32_t* __restrict__ counts, int E, int tb, int32_t* __restrict__ offsets,
                         int32_t* __restrict__ cursor, int32_t* __restrict__ tiles) {
  __shared__ int32_t buf[4096], tbuf[4096];
  for (int e = threadIdx.x; e < E; e += blockDim.x) buf[e] = counts[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0, tacc = 0;
    for (int e = 0; e < E; ++e) {
      const int32_t c = buf[e];
      buf[e] = acc;
      tbuf[e] = tacc;
      acc += c;
      tacc += (c + tb - 1) / tb;
    }
    offsets[E] = acc;
    tiles[E] = tacc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    offsets[e] = buf[e];
    cursor[e] = buf[e];
    tiles[e] = tbuf[e];
  }
}

// One warp per routed pair: claim a slot, record it, copy the token's row.
__global__ void moe_scatter(const int32_t* __restrict__ ids, int64_t pairs, int k, int E,
                            int32_t* __restrict__ cursor, int32_t* __restrict__ slot_of,
                            const uint8_t* __restrict__ x, int64_t row_bytes, uint8_t* __restrict__ xe) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = wid; i < pairs; i += nwarps) {
    int32_t slot = 0;
    if (lane == 0) {
      const int e = ids[i];
      slot = (e >= 0 && e < E) ? atomicAdd(&cursor[e], 1) : -1;
      slot_of[i] = slot;
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (slot < 0) continue;  // dropped pair (expert id out of range)
    const uint4* src = reinterpret_cast<const uint4*>(x + (i / k) * row_bytes);
    uint4* dst = reinterpret_cast<uint4*>(xe + int64_t(slot) * row_bytes);
    for (int64_t c = lane; c < row_bytes / 16; c += 32) dst[c] = src[c];
  }
}

template <int YDT>
__global__ void moe_combine(const float* __restrict__ ye, const int32_t* __restrict__ slot_of,
                            const float* __restrict__ w, int64_t T, int k, int64_t N, void* __restrict__ y) {
  const int64_t total = T * N;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, n = i - t * N;
    float acc = 0.f;
    for (int j = 0; j < k; ++j) {
      const int32_t sl = slot_of[t * k + j];
      if (sl >= 0) acc = fmaf(w[t * k + j], ye[int64_t(sl) * N + n], acc);
    }
    if constexpr (YDT == CCQ_DTYPE_F32)
      static_cast<float*>(y)[i] = acc;
    else
      static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(acc);
  }
}

}  // namespace
}  // namespace ccqb

using namespace ccqb;

extern "C" int ccq_cuda_moe_forward(const ccq_dev_model* stack, const int32_t* topk_ids, const float* topk_w,
                                    int64_t T, int32_t k, const void* x, int x_dtype, void* y, int y_dtype,
                                    void* stream) {
  if (!stack || stack->num_experts <= 0) return fail(CCQ_ERR_INVALID, "not a stacked-expert model");
  if (T < 0 || k < 1) return fail(CCQ_ERR_SHAPE, "T must be >= 0 and k >= 1");
  if (T == 0) return CCQ_OK;
  if (!topk_ids || !topk_w || !x || !y) return fail(CCQ_ERR_INVALID, "null routing, activation or output pointer");
  if (x_dtype != CCQ_DTYPE_F32 && x_dtype != CCQ_DTYPE_BF16 && x_dtype != CCQ_DTYPE_F16)
    return fail(CCQ_ERR_CONFIG, "unsupported activation dtype");
  if (y_dtype != CCQ_DTYPE_F32 && y_dtype != CCQ_DTYPE_BF16) return fail(CCQ_ERR_CONFIG, "unsupported output dtype");
  const int E = stack->num_experts;
  if (E > 4096) return fail(CCQ_ERR_CONFIG, "more than 4096 experts");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t K = stack->cols, N = stack->rows_per_expert, pairs = T * k;
  const int64_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  if ((K * xb) % 16 != 0) return fail(CCQ_ERR_SHAPE, "activation rows must be a multiple of 16 bytes");
  if (reinterpret_cast<uintptr_t>(x) & 15u) return fail(CCQ_ERR_CONFIG, "activations must be 16-byte aligned");
  DeviceScope ds(stack->device);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  cudaMemPool_t pool = scratch_pool(dev);
  // workspace: counts[E] cursor[E] offsets[E+1] tiles[E+1] slot_of[pairs] | xe[pairs][K] | ye[pairs][N] f32
  const size_t ints = size_t(4 * E + 2) + size_t(pairs);
  const size_t off_xe = (ints * 4 + 255) & ~size_t(255);
  const size_t off_ye = (off_xe + size_t(pairs * K * xb) + 255) & ~size_t(255);
  const size_t bytes = off_ye + size_t(pairs * N) * 4;
  uint8_t* ws = nullptr;
  CCQ_CUDA_TRY(capturing ? cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, s)
                         : cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ws), bytes, pool, s));
  int32_t* counts = reinterpret_cast<int32_t*>(ws);
  int32_t* cursor = counts + E;
  int32_t* offsets = cursor + E;
  int32_t* tiles = offsets + E + 1;
  int32_t* slot_of = tiles + E + 1;
  uint8_t* xe = ws + off_xe;
  float* ye = reinterpret_cast<float*>(ws + off_ye);
  const int tb = grouped_tile_tokens(stack, pairs, E, x_dtype);
  const int64_t max_tiles = std::min<int64_t>((pairs + tb - 1) / tb + E, int64_t(E) * ((pairs + tb - 1) / tb));
  int st = CCQ_OK;
  cudaError_t e = cudaMemsetAsync(counts, 0, size_t(E) * 4, s);
  if (e == cudaSuccess) {
    const unsigned blocks = unsigned(std::min<int64_t>((pairs + 255) / 256, 1184));
    moe_count<<<blocks, 256, 0, s>>>(topk_ids, pairs, E, counts);
    moe_scan<<<1, 256, 0, s>>>(counts, E, tb, offsets, cursor, tiles);
    const unsigned sblocks = unsigned(std::min<int64_t>((pairs * 32 + 255) / 256, 1184));
    moe_scatter<<<sblocks, 256, 0, s>>>(topk_ids, pairs, k, E, cursor, slot_of, static_cast<const uint8_t*>(x),
                                        K * xb, xe);
    count_launch(3);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    cudaFreeAsync(ws, s);
    return cuda_fail(e, "moe routing");
  }
  if (!gemm_supported(stack, pairs)) {
    cudaFreeAsync(ws, s);
    return fail(CCQ_ERR_CONFIG, "moe_forward needs group_size 64 and cols % 64 == 0 (tcgen05 grouped GEMM)");
  }
  st = launch_grouped_gemm_tiles(stack, E, N, offsets, tiles, max_tiles, pairs, xe, x_dtype, ye, CCQ_DTYPE_F32, s);
  if (st == CCQ_OK) {
    const unsigned cblocks = unsigned(std::min<int64_t>((T * N + 255) / 256, 148 * 16));
    if (y_dtype == CCQ_DTYPE_F32)
      moe_combine<CCQ_DTYPE_F32><<<cblocks, 256, 0, s>>>(ye, slot_of, topk_w, T, k, N, y);
    else
      moe_combine<CCQ_DTYPE_BF16><<<cblocks, 256, 0, s>>>(ye, slot_of, topk_w, T, k, N, y);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "moe combine");
  }
  cudaFreeAsync(ws, s);
  return st;
}
