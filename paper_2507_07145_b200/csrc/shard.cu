// Multi-GPU path: output rows of a large linear split across the
// ranks of one node, ONE all-gather of the output blocks over NVLink (NCCL).
//
// The reference is single-process CPU code with no collective; this is the
// north star's "output columns of large linears ... split across GPUs, with
// an NCCL all-gather over NVLink only for the output gather".
//
//   * rank p holds rows [p*N/P, (p+1)*N/P) (ccq_cuda_model_upload_rows: a
//     contiguous slice of the group-major payload);
//   * tokens are processed in chunks: chunk c's decode-matmul writes its
//     [Mc][n_p] block on the caller's stream, then on a communication stream
//     the all-gather of chunk c and the column interleave into y[M][N] run
//     while chunk c+1 computes (double-buffered, event-ordered: no host sync,
//     CUDA-graph capturable);
//   * M = 1 with equal blocks gathers in place into y (no copies at all).
//
// NCCL is not linked: its entry points are resolved at run time from the
// libnccl.so.2 already mapped into the process (torch's) or loaded by name,
// so the library never pulls a second NCCL into a torch process.
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "ccq_internal.hpp"

namespace ccqb {
namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather && n.error_string;
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const Nccl& n = nccl();
  return fail(CCQ_ERR_CUDA, std::string(what) + ": " + (n.error_string ? n.error_string(r) : "NCCL error"));
}

inline void block_range(int64_t n, int r, int world, int64_t* lo, int64_t* hi) {
  *lo = n * r / world;
  *hi = n * (r + 1) / world;
}

// y[m0 + t][lo_r + j] = gath[r][t * n_r + j] for every rank r (blocks padded
// to Mc * n_max elements in the gather buffer).
template <typename T>
__global__ void interleave(const T* __restrict__ gath, int64_t slot_elems, int world, int64_t rows_total,
                           int64_t Mc, T* __restrict__ y, int64_t m0) {
  const int64_t total = Mc * rows_total;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / rows_total, col = i - t * rows_total;
    // rank owning `col`: largest r with r * N / P <= col
    int r = int((col * world + world - 1) / rows_total);
    if (r >= world) r = world - 1;
    while (r > 0 && rows_total * r / world > col) --r;
    while (r + 1 < world && rows_total * (r + 1) / world <= col) ++r;
    const int64_t lo = rows_total * r / world, hi = rows_total * (r + 1) / world;
    y[(m0 + t) * rows_total + col] = gath[int64_t(r) * slot_elems + t * (hi - lo) + (col - lo)];
  }
}

struct CommStreams {
  std::mutex mu;
  cudaStream_t s[64] = {};
};
CommStreams& comm_streams() {
  static CommStreams c;
  return c;
}

}  // namespace
}  // namespace ccqb

using namespace ccqb;

extern "C" int ccq_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(CCQ_ERR_INVALID, "null id buffer");
  const Nccl& n = nccl();
  if (!n.ok) return fail(CCQ_ERR_CONFIG, "libnccl.so.2 not found in the process or on the library path");
  ncclUniqueId id;
  const ncclResult_t r = n.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return CCQ_OK;
}

extern "C" int ccq_nccl_comm_init(int world, int rank, const uint8_t* id128, int device, void** comm) {
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) return fail(CCQ_ERR_INVALID, "bad communicator args");
  const Nccl& n = nccl();
  if (!n.ok) return fail(CCQ_ERR_CONFIG, "libnccl.so.2 not found in the process or on the library path");
  DeviceScope ds(device);
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.comm_init_rank(&c, world, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return CCQ_OK;
}

extern "C" int ccq_nccl_comm_destroy(void* comm) {
  if (!comm) return CCQ_OK;
  const Nccl& n = nccl();
  if (!n.ok) return fail(CCQ_ERR_CONFIG, "libnccl.so.2 not loaded");
  const ncclResult_t r = n.comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? CCQ_OK : nccl_fail(r, "ncclCommDestroy");
}

extern "C" int ccq_cuda_shard_allgather(const ccq_dev_model* shard, int64_t rows_total, int world, int rank,
                                        const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                                        int64_t chunk_tokens, void* comm, void* stream) {
  if (!shard || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !comm))
    return fail(CCQ_ERR_INVALID, "bad rank / world / communicator");
  if (M < 0 || rows_total < world) return fail(CCQ_ERR_SHAPE, "bad token count or row split");
  if (y_dtype != CCQ_DTYPE_F32 && y_dtype != CCQ_DTYPE_BF16) return fail(CCQ_ERR_CONFIG, "unsupported output dtype");
  int64_t lo = 0, hi = 0;
  block_range(rows_total, rank, world, &lo, &hi);
  if (shard->rows != hi - lo)
    return fail(CCQ_ERR_SHAPE, "shard rows do not match this rank's block of rows_total");
  if (M == 0) return CCQ_OK;
  DeviceScope ds(shard->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t yb = y_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  const ncclDataType_t dt = y_dtype == CCQ_DTYPE_F32 ? ncclFloat32 : ncclBfloat16;
  if (world == 1 && !comm) return ccq_cuda_matmul(shard, x, x_dtype, M, y, y_dtype, stream);
  const Nccl& n = nccl();
  if (!n.ok) return fail(CCQ_ERR_CONFIG, "libnccl.so.2 not loaded");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const bool equal = rows_total % world == 0;
  if (M == 1 && equal) {  // [1][N] is contiguous: compute into place, gather in place
    uint8_t* own = static_cast<uint8_t*>(y) + size_t(lo) * yb;
    int st = ccq_cuda_matmul(shard, x, x_dtype, 1, own, y_dtype, stream);
    if (st != CCQ_OK) return st;
    const ncclResult_t r = n.all_gather(own, y, size_t(hi - lo), dt, c, s);
    return r == ncclSuccess ? CCQ_OK : nccl_fail(r, "ncclAllGather");
  }
  int64_t nmax = 0;
  for (int r = 0; r < world; ++r) {
    int64_t a = 0, b = 0;
    block_range(rows_total, r, world, &a, &b);
    nmax = std::max(nmax, b - a);
  }
  const int64_t Mc = std::max<int64_t>(1, std::min<int64_t>(chunk_tokens > 0 ? chunk_tokens : M, M));
  const int64_t nchunks = (M + Mc - 1) / Mc;
  const int64_t slot = Mc * nmax;  // elements per rank block in the gather buffer
  const size_t xb = x_dtype == CCQ_DTYPE_F32 ? 4 : 2;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  // workspace: send[2][slot] | gather[2][world][slot]
  const size_t bytes = size_t(2) * slot * yb + size_t(2) * world * slot * yb;
  uint8_t* ws = nullptr;
  CCQ_CUDA_TRY(capturing ? cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, s)
                         : cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ws), bytes, scratch_pool(dev), s));
  uint8_t* send = ws;
  uint8_t* gath = ws + size_t(2) * slot * yb;
  cudaStream_t cs;
  {
    CommStreams& css = comm_streams();
    std::lock_guard<std::mutex> lock(css.mu);
    if (!css.s[dev]) CCQ_CUDA_TRY(cudaStreamCreateWithFlags(&css.s[dev], cudaStreamNonBlocking));
    cs = css.s[dev];
  }
  cudaEvent_t ev[5];
  for (auto& e : ev) CCQ_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t &comp0 = ev[0], &comp1 = ev[1], &comm0 = ev[2], &comm1 = ev[3], &fork = ev[4];
  int st = CCQ_OK;
  cudaError_t ce = cudaEventRecord(fork, s);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs, fork, 0);  // comm stream joins the caller's order
  for (int64_t ci = 0; ci < nchunks && st == CCQ_OK && ce == cudaSuccess; ++ci) {
    const int b = int(ci & 1);
    const int64_t m0 = ci * Mc, mc = std::min(Mc, M - m0);
    if (ci >= 2) ce = cudaStreamWaitEvent(s, b ? comm1 : comm0, 0);  // slot b drained
    if (ce != cudaSuccess) break;
    st = ccq_cuda_matmul(shard, static_cast<const uint8_t*>(x) + size_t(m0) * shard->cols * xb, x_dtype, mc,
                         send + size_t(b) * slot * yb, y_dtype, stream);
    if (st != CCQ_OK) break;
    ce = cudaEventRecord(b ? comp1 : comp0, s);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(cs, b ? comp1 : comp0, 0);
    if (ce != cudaSuccess) break;
    const ncclResult_t r = n.all_gather(send + size_t(b) * slot * yb, gath + size_t(b) * world * slot * yb,
                                        size_t(slot), dt, c, cs);
    if (r != ncclSuccess) {
      st = nccl_fail(r, "ncclAllGather");
      break;
    }
    const unsigned blocks = unsigned(std::min<int64_t>((mc * rows_total + 255) / 256, 148 * 8));
    if (y_dtype == CCQ_DTYPE_F32)
      interleave<float><<<blocks, 256, 0, cs>>>(reinterpret_cast<const float*>(gath) + size_t(b) * world * slot, slot,
                                                world, rows_total, mc, static_cast<float*>(y), m0);
    else
      interleave<__nv_bfloat16><<<blocks, 256, 0, cs>>>(
          reinterpret_cast<const __nv_bfloat16*>(gath) + size_t(b) * world * slot, slot, world, rows_total, mc,
          static_cast<__nv_bfloat16*>(y), m0);
    count_launch();
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaEventRecord(b ? comm1 : comm0, cs);
  }
  // join: the caller's stream waits for the last gathers
  if (ce == cudaSuccess) ce = cudaEventRecord(fork, cs);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, fork, 0);
  cudaFreeAsync(ws, s);
  for (auto& e : ev) cudaEventDestroy(e);
  if (st != CCQ_OK) return st;
  return ce == cudaSuccess ? CCQ_OK : cuda_fail(ce, "shard all-gather");
}
