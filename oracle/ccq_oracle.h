/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the CCQ decode / GEMV hot path.
 *
 * A plain-C restatement of the reference CCQ codec's inference path
 * (/root/reference/proj/core, FORMAT.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the
 * checker.  The product path (paper_2507_07145_b200/) never links it.
 *
 * Parity is pinned two ways (see tests/test_oracle_golden.py):
 *   1. the reference's own golden vectors (test_coding.cpp, test_packing.cpp,
 *      test_kernels.cpp, acceptance criteria 6/8) ported as data;
 *   2. byte-for-byte agreement with the reference library itself, compiled
 *      from /root/reference by oracle/Makefile into oracle/_ref/.
 *
 * Family numbering follows ccq::Family (coding.hpp:115): 0 = "2.75",
 * 1 = "2.5", 2 = "2.06".
 *
 * Status codes follow the reference exception hierarchy (error.hpp:25-68).
 */
#ifndef CCQ_ORACLE_H_
#define CCQ_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CCQO_OK = 0,
  CCQO_CONFIG = 1,   /* ccq::ConfigError */
  CCQO_DOMAIN = 2,   /* ccq::DomainError */
  CCQO_SHAPE = 3,    /* ccq::ShapeError */
  CCQO_ENCODING = 4, /* ccq::EncodingError */
  CCQO_FORMAT = 5    /* ccq::FormatError */
};

/* ccq::Scheme + LayoutSpec (coding.hpp:101-135, coding.cpp:213-249). */
typedef struct {
  int family;
  int code_bits;         /* 8, 16, 15 */
  int stored_word_bytes; /* 1, 2, 1 */
  int weights_per_word;  /* 3, 7, 4 */
  int state_bits;        /* 4, 3, 6 */
  int zero_point;        /* 8, 4, 32 */
  int scale_bits;        /* 4, 13, 4 */
  int uses_cluster;      /* 0, 0, 1 */
  int word_bits;         /* 8, 16, 16 */
  uint32_t weight_mask;  /* 0xF, 0x7, 0x3F */
  uint32_t scale_mask;   /* 0xF, 0x1FFF, 0xF */
  int shifts[7];         /* MSB-first window shifts */
} ccqo_scheme;

/* ccq::GroupGeometry (packing.hpp:38-49). */
typedef struct {
  int group_size;
  int full_words;
  int has_tail;
  int words_per_group;
  int embedded_scale;
  int payload_bytes;
} ccqo_geometry;

/* A borrowed view of ccq::PackedModel (container.hpp:37-52). */
typedef struct {
  int64_t rows;
  int64_t cols;
  int family;
  int group_size;
  const uint8_t* code_payload;
  size_t code_bytes;
  const uint8_t* scale_payload;
  size_t scale_bytes;
  const float* super_scales;        /* rows */
  const float* cluster_scales;      /* rows, 2.06 only */
  const float* cluster_zero_points; /* rows, 2.06 only */
} ccqo_model;

int ccqo_scheme_for(int family, ccqo_scheme* out);
int ccqo_group_geometry(int family, int group_size, ccqo_geometry* out);

/* clustered_code_value (coding.hpp:142-150). */
int ccqo_clustered_code_value(uint8_t q, float alpha, float beta, int code_bits,
                              uint16_t* out);

/* Sizes of the packed sections for a (rows, cols, family, group_size). */
int ccqo_section_sizes(int64_t rows, int64_t cols, int family, int group_size,
                       size_t* code_bytes, size_t* scale_bytes, size_t* cluster_rows);

/* Validates a model view exactly as the reference loader does
 * (container.cpp:261-319): sizes against the geometry. */
int ccqo_validate(const ccqo_model* m);

/* dequantize (kernels.cpp:103-122): rows x cols f32, row-major. */
int ccqo_dequantize(const ccqo_model* m, float* out);

/* Centered integer levels, state - zero_point (quantizer.cpp:120-134
 * decode_group_states, minus Scheme::zero_point as reconstruct does at
 * quantizer.cpp:441-443). */
int ccqo_levels(const ccqo_model* m, int8_t* out);

/* Per-group f32 scale = float(scale_code) * super (kernels.cpp:65-71). */
int ccqo_group_scales(const ccqo_model* m, float* out);

/* gemv_batch (kernels.cpp:152-187): y[M x rows] = x[M x cols] W^T with
 * double accumulation, left to right within a row. */
int ccqo_gemv_batch(const ccqo_model* m, const float* x, int64_t batch, float* y);

/* Same arithmetic, rows sharded over `threads` POSIX threads (the survey's
 * all-cores CPU baseline; each output element is computed exactly as in the
 * single-threaded version). */
int ccqo_gemv_batch_mt(const ccqo_model* m, const float* x, int64_t batch, float* y,
                       int threads);

/* model_payload_bytes (kernels.cpp:203-207). */
uint64_t ccqo_payload_bytes(const ccqo_model* m);

/* random_matrix (tensor.cpp:48-69): dist 0 = Gaussian, 1 = Uniform. */
void ccqo_random_matrix(int64_t rows, int64_t cols, int dist, uint64_t seed, float* out);

/* pack_model(random_quantized(rows, cols, family, group_size, seed))
 * (synthetic.cpp:25-103, container.cpp:323-358): fills caller buffers sized
 * by ccqo_section_sizes.  cluster_* may be NULL for non-clustered families. */
int ccqo_random_packed(int64_t rows, int64_t cols, int family, int group_size, uint64_t seed,
                       uint8_t* code_payload, uint8_t* scale_payload, float* super_scales,
                       float* cluster_scales, float* cluster_zero_points);

/* Side-band nibbles (packing.cpp:160-184). */
int ccqo_pack_cluster_scales(const uint16_t* codes, size_t n, uint8_t* out);
int ccqo_unpack_cluster_scales(const uint8_t* bytes, size_t nbytes, size_t group_count,
                               uint16_t* out);

/* pack_group (packing.cpp:71-114): payload bytes of one group, side-band
 * scale returned through *sideband (0 when embedded). */
int ccqo_pack_group(const uint16_t* codes, size_t n_codes, uint16_t scale_code, int family,
                    int group_size, uint8_t* payload, uint16_t* sideband);

#ifdef __cplusplus
}
#endif

#endif /* CCQ_ORACLE_H_ */
