/*
 * ccq_cuda.h — the C ABI of the B200-native CCQ hot path (libccq_b200.so).
 *
 * This is the drop-in boundary for the reference's inference path
 * (/root/reference/proj/core/include/ccq/kernels.hpp:36-76 and
 * container.hpp:37-99).  The reference has no FFI of its own; its operator
 * boundary is the C++ library API, which the headers in include/ccq/ re-declare on top
 * of these entry points.  Plain pointers and sizes only: no C++ or torch
 * types cross this boundary.
 *
 * Conventions
 *   - Every function returns a ccq_status; on failure a thread-local message
 *     is available from ccq_cuda_last_error().
 *   - Status values map 1:1 onto the reference exception hierarchy
 *     (error.hpp:25-68) plus CCQ_ERR_CUDA for device failures.
 *   - Device-pointer entry points are asynchronous on the given stream
 *     (cudaStream_t passed as void*, NULL = legacy default stream) and never
 *     synchronize.  "_host" entry points take host buffers and are
 *     synchronous, mirroring the reference's blocking C++ calls.
 *   - A ccq_dev_model is immutable after upload and may be used from several
 *     streams/threads concurrently (the reference's reentrancy contract,
 *     SPEC.md:391).
 *
 * Family numbering follows ccq::Family (coding.hpp:115):
 *   0 = "2.75" (4,3,2) embedded 4-bit scale
 *   1 = "2.5"  hybrid (3,3,2)+(3,4,2) 16-bit word, embedded 13-bit scale
 *   2 = "2.06" (6,4,3) clustered to 8 bits, side-band 4-bit scale nibbles
 */
#ifndef CCQ_CUDA_H_
#define CCQ_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ccq_status {
  CCQ_OK = 0,
  CCQ_ERR_CONFIG = 1,   /* ccq::ConfigError   (error.hpp:31) */
  CCQ_ERR_DOMAIN = 2,   /* ccq::DomainError   (error.hpp:38) */
  CCQ_ERR_SHAPE = 3,    /* ccq::ShapeError    (error.hpp:44) */
  CCQ_ERR_ENCODING = 4, /* ccq::EncodingError (error.hpp:51) */
  CCQ_ERR_FORMAT = 5,   /* ccq::FormatError   (error.hpp:58) */
  CCQ_ERR_CUDA = 6,     /* device / runtime failure (new) */
  CCQ_ERR_INVALID = 7   /* null handle or pointer misuse (new) */
} ccq_status;

typedef enum ccq_dtype {
  CCQ_DTYPE_F32 = 0,
  CCQ_DTYPE_BF16 = 1,
  CCQ_DTYPE_F16 = 2
} ccq_dtype;

/* Borrowed host view of ccq::PackedModel (container.hpp:37-52): the five
 * sections exactly as stored in a .ccq container (FORMAT.md §6), with
 * cluster_params already de-interleaved as the reference loader does
 * (container.cpp:308-316).  Lengths are in elements of each pointer type. */
typedef struct ccq_packed_view {
  int64_t rows;       /* d_out (output channels) */
  int64_t cols;       /* d_in */
  int32_t family;     /* 0 "2.75", 1 "2.5", 2 "2.06" */
  int32_t group_size; /* FORMAT.md §3; 64 by default */
  int32_t rounds;     /* quantizer refinement rounds (metadata) */
  int32_t reserved;
  const uint8_t* code_payload;  /* payload_bytes per group, group-major */
  uint64_t code_bytes;
  const uint8_t* scale_payload; /* side-band nibbles, NULL when embedded */
  uint64_t scale_bytes;
  const float* super_scales; /* rows */
  uint64_t n_super_scales;
  const float* cluster_scales; /* rows (2.06) or NULL */
  uint64_t n_cluster_scales;
  const float* cluster_zero_points; /* rows (2.06) or NULL */
  uint64_t n_cluster_zero_points;
} ccq_packed_view;

typedef struct ccq_dev_model ccq_dev_model;

/* Shape and accounting of an uploaded model. */
typedef struct ccq_model_info {
  int64_t rows, cols;
  int32_t family, group_size, rounds, device;
  int32_t payload_bytes_per_group; /* GroupGeometry::payload_bytes */
  int32_t embedded_scale;
  uint64_t payload_bytes; /* model_payload_bytes (kernels.cpp:203-207) */
  uint64_t device_bytes;  /* HBM held by the device copy */
  uint64_t code_row_stride; /* bytes between rows of codes on the device */
  int32_t fast_path;       /* 1 when the group-64 streaming kernels apply */
  int32_t reserved;
} ccq_model_info;

const char* ccq_cuda_last_error(void);
const char* ccq_cuda_version(void);

/* ---- packed-weight loader / upload (container.cpp:261-319, 428-432) ---- */

/* Validates the sections against the group geometry (FormatError, as
 * model_from_bytes does), builds the per-row exact fixed-point widening plan
 * for the clustered family (coding.hpp:142-150; every q in [0,256) is checked
 * against the reference formula), raises DomainError when a stored byte
 * would widen outside [0, 2^15) (the reference throws the same error lazily
 * at decode time), and copies the sections to `device` in the device layout
 * (DESIGN.md §3).  Synchronous. */
int ccq_cuda_model_upload(const ccq_packed_view* view, int device, ccq_dev_model** out);

/* Upload straight from a .ccq container file (load_model, container.cpp:428). */
int ccq_cuda_model_load(const char* path, int device, ccq_dev_model** out);

/* Host-only container read (load_model + model_from_bytes,
 * container.cpp:261-319, 428-432): fills `view` with pointers into a
 * library-owned image released by ccq_container_close(owner).  Same
 * FormatError checks and byte offsets as the reference parse_info. */
int ccq_container_open(const char* path, ccq_packed_view* view, void** owner);
void ccq_container_close(void* owner);

/* A contiguous block of output rows [row_begin, row_end) of a host model as
 * its own device model (N-column sharding). */
int ccq_cuda_model_upload_rows(const ccq_packed_view* view, int64_t row_begin, int64_t row_end,
                               int device, ccq_dev_model** out);

int ccq_cuda_model_free(ccq_dev_model* model);
int ccq_cuda_model_info(const ccq_dev_model* model, ccq_model_info* info);

/* ---- kernel (a): standalone decode (kernels.cpp:60-122) ---- */

/* levels (rows x cols int8, state - zero_point) and/or weights (rows x cols
 * f32, bit-exact to ccq::dequantize).  Either pointer may be NULL.  Device
 * pointers, asynchronous on `stream`. */
int ccq_cuda_decode(const ccq_dev_model* model, int8_t* levels, float* weights, void* stream);

/* ---- kernels (b)/(c): fused decode + matmul (kernels.cpp:124-187) ----
 *
 * y[M x rows] = x[M x cols] . W^T with W decoded on the fly.
 * x: f32, bf16 or f16 (x_dtype); y: f32 or bf16 (y_dtype).  Device pointers.
 * ccq_cuda_matmul picks the kernel by M: the CUDA-core streaming GEMV for
 * small M, the tcgen05 GEMM otherwise.  The explicit entry points force one. */
int ccq_cuda_matmul(const ccq_dev_model* model, const void* x, int x_dtype, int64_t M, void* y,
                    int y_dtype, void* stream);
int ccq_cuda_gemv(const ccq_dev_model* model, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream);
int ccq_cuda_gemm(const ccq_dev_model* model, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream);

/* ---- kernel (d): grouped experts (MoE) ----
 *
 * models[E] share (rows, cols, family, group_size).  Tokens are laid out
 * expert-major: expert e owns rows [offsets[e], offsets[e+1]) of x and y
 * (offsets has E+1 entries, device int32).  Experts with no rows cost
 * nothing.  x: bf16/f16/f32 [offsets[E] x cols]; y: f32/bf16
 * [offsets[E] x rows]. */
int ccq_cuda_grouped(const ccq_dev_model* const* models, int32_t num_experts,
                     const int32_t* offsets_device, const int32_t* offsets_host,
                     const void* x, int x_dtype, void* y, int y_dtype, void* stream);

/* Stacked experts (the MoE path): E experts with identical shape/family
 * uploaded into ONE device model (rows = E x rows_per_expert) so that all of
 * them run in a single launch. */
int ccq_cuda_experts_upload(const ccq_packed_view* views, int32_t num_experts, int device,
                            ccq_dev_model** out);
/* y[T x rows_per_expert] for x[T x cols], T = offsets[E] tokens laid out
 * expert-major.  2.06: one tcgen05 grouped-GEMM launch over (expert, row tile,
 * token tile); experts with no tokens exit at once (their weights are never
 * read).  offsets_device/offsets_host hold the same E+1 int32 values. */
int ccq_cuda_experts_matmul(const ccq_dev_model* stack, const int32_t* offsets_device,
                            const int32_t* offsets_host, const void* x, int x_dtype, void* y,
                            int y_dtype, void* stream);

/* MoE layer with routing: tokens x[T x cols] in natural
 * order, router top-k expert ids topk_ids[T x k] (device int32) and weights
 * topk_w[T x k] (device f32) -> y[T x rows_per_expert] =
 * sum_j topk_w[t,j] * (expert topk_ids[t,j]) x[t], summed in j order.
 * Permutes the routed rows expert-major, runs the grouped tcgen05 GEMM over a
 * device-side token-tile list, and combines.  Never synchronises: the whole
 * call is stream-ordered and CUDA-graph capturable.  Expert ids outside
 * [0, E) are dropped (those pairs contribute zero); validate ids upstream
 * if they are untrusted. */
int ccq_cuda_moe_forward(const ccq_dev_model* stack, const int32_t* topk_ids, const float* topk_w,
                         int64_t T, int32_t k, const void* x, int x_dtype, void* y, int y_dtype,
                         void* stream);

/* ---- multi-GPU: output rows split across the ranks of a node ---- */

/* NCCL is resolved at run time from the libnccl.so.2 already loaded in the
 * process (e.g. torch's) or on the library path; no link-time dependency.
 * ccq_nccl_unique_id: rank 0 creates the 128-byte id and shares it (any
 * side channel); every rank then calls ccq_nccl_comm_init on its device. */
int ccq_nccl_unique_id(uint8_t* out128);
int ccq_nccl_comm_init(int world, int rank, const uint8_t* id128, int device, void** comm);
int ccq_nccl_comm_destroy(void* comm);

/* Row-sharded linear + output all-gather (the ccq_cuda_shard_allgather of
 * SURVEY §8b).  `shard` holds this rank's block [rank*N/world,
 * (rank+1)*N/world) of an N = rows_total row layer (ccq_cuda_model_upload_rows);
 * y is the FULL output [M x rows_total] on every rank.  Tokens run in chunks of
 * chunk_tokens (0 = all): chunk c's all-gather (NCCL, `comm` = ncclComm_t) and
 * column interleave overlap chunk c+1's decode-matmul on a second stream;
 * M = 1 with N % world == 0 gathers in place.  No host synchronisation (graph
 * capturable).  world == 1 with comm == NULL is a plain ccq_cuda_matmul. */
int ccq_cuda_shard_allgather(const ccq_dev_model* shard, int64_t rows_total, int world, int rank,
                             const void* x, int x_dtype, int64_t M, void* y, int y_dtype,
                             int64_t chunk_tokens, void* comm, void* stream);

/* ---- synthetic models (bench harness) ---- */

/* pack_model(random_quantized(rows, cols, family, group_size, seed)) of the
 * reference bench generator (synthetic.cpp:25-103, container.cpp:323-358),
 * draw for draw (std::mt19937_64): the reference's exact bytes for a seed.
 * Host only (no device).  Buffers: code_payload rows*(cols/g)*payload_bytes,
 * scale_payload (groups+1)/2 (side-band families), super_scales rows,
 * cluster_scales / cluster_zero_points rows (2.06). */
int ccq_synthetic_packed(int64_t rows, int64_t cols, int32_t family, int32_t group_size, uint64_t seed,
                         uint8_t* code_payload, uint8_t* scale_payload, float* super_scales,
                         float* cluster_scales, float* cluster_zero_points);

/* random_matrix (tensor.cpp:37-69), the reference's generator draw for draw:
 * dist 0 = Gaussian, 1 = uniform [-1, 1).  out: rows*cols f32, row-major. */
int ccq_synthetic_matrix(int64_t rows, int64_t cols, int32_t dist, uint64_t seed, float* out);

/* ---- synchronous host-buffer entry points (the reference signatures) ---- */

/* ccq::dequantize (kernels.hpp:36). out: host rows x cols f32. */
int ccq_dequantize_host(const ccq_dev_model* model, float* out);
/* ccq::gemv (kernels.hpp:39). x: host cols f32; y: host rows f32. */
int ccq_gemv_host(const ccq_dev_model* model, const float* x, uint64_t x_len, float* y,
                  uint64_t y_len);
/* ccq::gemv_batch (kernels.hpp:43). x: host M x cols; y: host M x rows. */
int ccq_gemv_batch_host(const ccq_dev_model* model, const float* x, int64_t x_rows,
                        int64_t x_cols, float* y, int64_t y_rows, int64_t y_cols);

/* ccq::model_payload_bytes (kernels.hpp:51). */
int ccq_model_payload_bytes(const ccq_dev_model* model, uint64_t* out);

/* Host-side geometry helpers (packing.hpp:49, coding.hpp:142-150). */
int ccq_group_geometry(int32_t family, int32_t group_size, int32_t out6[6]);
int ccq_clustered_code_value(uint8_t q, float alpha, float beta, int32_t code_bits,
                             uint16_t* out);

/* Number of kernels this library launched since load (bench accounting). */
uint64_t ccq_cuda_launch_count(void);

/* Exhaustive trellis code search of the CCQ quantizer for n subvectors
 * (replaces ccq::search_codes, core/src/quantizer.cpp:36-103, one call per
 * subvector; bit-identical codes).  Device pointers: targets[n][stride] f32
 * (the first `valid` values of each row are the subvector), scales[n] f64,
 * codes[n] out.  Config = EncodingConfig (state_bits L, states_per_code N,
 * transition_bits S), validated like EncodingConfig::validate
 * (CCQ_ERR_CONFIG); valid outside 1..N is CCQ_ERR_SHAPE as in the reference. */
int ccq_cuda_search_codes(const float* targets, int64_t n, int32_t valid, int32_t stride,
                          const double* scales, int32_t zero_point, int32_t state_bits,
                          int32_t states_per_code, int32_t transition_bits, uint32_t* codes,
                          void* stream);

/* The CCQ quantizer on the GPU: pack_model(quantize_tensor(W)) (replaces
 * ccq::quantize_tensor, core/src/quantizer.cpp:319-425, + ccq::pack_model,
 * container.cpp:323-358), bit-identical sections.  Host buffers: w[rows][cols]
 * f32 in; out: code_payload (groups x payload_bytes), scale_payload
 * ((groups+1)/2 bytes, families with side-band scales, else may be NULL),
 * super_scales[rows], cluster_scales / cluster_zero_points [rows] (2.06,
 * else may be NULL).  Per-group search + refinement and the 2.06 cluster
 * re-search run on `device`.  group_size <= 256. */
int ccq_quantize_host(const float* w, int64_t rows, int64_t cols, int32_t family, int32_t group_size,
                      int32_t rounds, int32_t device, uint8_t* code_payload, uint8_t* scale_payload,
                      float* super_scales, float* cluster_scales, float* cluster_zero_points);

/* Quantize weights already in device memory (w: rows x cols f32, device
 * pointer) and upload the result as a device model, with no host round trip
 * (the packed sections go from the quantizer's workspace into the device
 * re-layout).  Same sections as ccq_quantize_host. */
int ccq_cuda_quantize_model(const float* w, int64_t rows, int64_t cols, int32_t family, int32_t group_size,
                            int32_t rounds, int32_t device, ccq_dev_model** out);

#ifdef __cplusplus
}
#endif

#endif /* CCQ_CUDA_H_ */
