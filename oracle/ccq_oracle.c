/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the CCQ decode / GEMV hot path.
 * See ccq_oracle.h for scope and the rules on who may call this.
 *
 * Every function restates the reference algorithm it cites
 * (/root/reference/proj/core/...).  Arithmetic is kept identical: the decode
 * multiplies in f32, the widening runs in double with lround semantics, and
 * the GEMV accumulates in double left to right, so outputs are bit-identical
 * to the reference library (checked against oracle/_ref in the tests).
 *
 * Build: gcc -O2 -fPIC -shared (no -march / -ffast-math: the reference is
 * built the same way so libm and FP contraction behave identically).
 */
#include "ccq_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Families: coding.cpp:145-193 (word_shifts / layout_for), 213-249    */
/* (make_scheme).                                                      */
/* ------------------------------------------------------------------ */

int ccqo_scheme_for(int family, ccqo_scheme* s) {
  memset(s, 0, sizeof(*s));
  s->family = family;
  switch (family) {
    case 0: /* "2.75": (4,3,2), T = 8, embedded 4-bit scale */
      s->code_bits = 8;
      s->stored_word_bytes = 1;
      s->weights_per_word = 3;
      s->state_bits = 4;
      s->scale_bits = 4;
      s->word_bits = 8;
      s->weight_mask = 0xF;
      s->scale_mask = 0xF;
      s->shifts[0] = 4; s->shifts[1] = 2; s->shifts[2] = 0;
      break;
    case 1: /* "2.5": hybrid (3,3,2)+(3,4,2) in a 16-bit word, 13-bit scale */
      s->code_bits = 16;
      s->stored_word_bytes = 2;
      s->weights_per_word = 7;
      s->state_bits = 3;
      s->scale_bits = 13;
      s->word_bits = 16;
      s->weight_mask = 0x7;
      s->scale_mask = 0x1FFF;
      {
        const int sh[7] = {13, 11, 9, 6, 4, 2, 0};
        memcpy(s->shifts, sh, sizeof(sh));
      }
      break;
    case 2: /* "2.06": (6,4,3), T = 15, clustered to one byte, side-band scale */
      s->code_bits = 15;
      s->stored_word_bytes = 1;
      s->weights_per_word = 4;
      s->state_bits = 6;
      s->scale_bits = 4;
      s->uses_cluster = 1;
      s->word_bits = 16;
      s->weight_mask = 0x3F;
      s->scale_mask = 0xF;
      s->shifts[0] = 9; s->shifts[1] = 6; s->shifts[2] = 3; s->shifts[3] = 0;
      break;
    default:
      return CCQO_CONFIG;
  }
  s->zero_point = 1 << (s->state_bits - 1);
  return CCQO_OK;
}

/* group_geometry (packing.cpp:24-47). */
int ccqo_group_geometry(int family, int group_size, ccqo_geometry* g) {
  ccqo_scheme s;
  if (ccqo_scheme_for(family, &s) != CCQO_OK) return CCQO_CONFIG;
  if (group_size <= 0) return CCQO_CONFIG;
  const int rem = group_size % s.weights_per_word;
  if (rem > 1) return CCQO_CONFIG;
  if (family == 1 && rem == 0) return CCQO_CONFIG;
  g->group_size = group_size;
  g->full_words = group_size / s.weights_per_word;
  g->has_tail = rem == 1;
  g->words_per_group = g->full_words + g->has_tail;
  g->embedded_scale = g->has_tail && !s.uses_cluster;
  g->payload_bytes = g->words_per_group * s.stored_word_bytes;
  return CCQO_OK;
}

/* clustered_code_value (coding.hpp:142-150): lround in double, half away
 * from zero; DomainError outside [0, 2^code_bits). */
int ccqo_clustered_code_value(uint8_t q, float alpha, float beta, int code_bits,
                              uint16_t* out) {
  const long v = lround((double)q * (double)alpha + (double)beta);
  if (v < 0 || v >= (1l << code_bits)) return CCQO_DOMAIN;
  *out = (uint16_t)v;
  return CCQO_OK;
}

int ccqo_section_sizes(int64_t rows, int64_t cols, int family, int group_size,
                       size_t* code_bytes, size_t* scale_bytes, size_t* cluster_rows) {
  ccqo_scheme s;
  ccqo_geometry g;
  if (ccqo_scheme_for(family, &s) != CCQO_OK) return CCQO_CONFIG;
  if (ccqo_group_geometry(family, group_size, &g) != CCQO_OK) return CCQO_CONFIG;
  if (rows < 0 || cols < 0 || cols % group_size != 0) return CCQO_SHAPE;
  const uint64_t groups = (uint64_t)rows * (uint64_t)(cols / group_size);
  if (code_bytes) *code_bytes = (size_t)(groups * (uint64_t)g.payload_bytes);
  if (scale_bytes) *scale_bytes = g.embedded_scale ? 0 : (size_t)((groups + 1) / 2);
  if (cluster_rows) *cluster_rows = s.uses_cluster ? (size_t)rows : 0;
  return CCQO_OK;
}

/* Section-size checks of model_from_bytes (container.cpp:273-316). */
int ccqo_validate(const ccqo_model* m) {
  size_t cb, sb, cr;
  const int st = ccqo_section_sizes(m->rows, m->cols, m->family, m->group_size, &cb, &sb, &cr);
  if (st != CCQO_OK) return st;
  if (m->code_bytes != cb) return CCQO_FORMAT;
  if (m->scale_bytes != sb) return CCQO_FORMAT;
  if (m->rows > 0 && !m->super_scales) return CCQO_FORMAT;
  if (cr && (!m->cluster_scales || !m->cluster_zero_points)) return CCQO_FORMAT;
  return CCQO_OK;
}

/* ------------------------------------------------------------------ */
/* Decode: kernels.cpp:29-99                                           */
/* ------------------------------------------------------------------ */

typedef struct {
  ccqo_scheme s;
  ccqo_geometry g;
} plan_t;

static int make_plan(const ccqo_model* m, plan_t* p) {
  int st = ccqo_validate(m);
  if (st != CCQO_OK) return st;
  ccqo_scheme_for(m->family, &p->s);
  ccqo_group_geometry(m->family, m->group_size, &p->g);
  return CCQO_OK;
}

/* load_word (kernels.cpp:53-55). */
static inline uint32_t load_word(const uint8_t* p, int wide) {
  return wide ? ((uint32_t)p[0] | ((uint32_t)p[1] << 8)) : (uint32_t)p[0];
}

/* Side-band nibble of group gi (packing.cpp:172-184, FORMAT.md §3). */
static inline uint32_t sideband_code(const ccqo_model* m, int64_t gi) {
  return (m->scale_payload[gi / 2] >> (4 * (gi % 2))) & 0xF;
}

/* decode_group (kernels.cpp:60-93).  Writes f32 weights to out (if non-null)
 * and centered levels to lv (if non-null). */
static int decode_group(const plan_t* p, const uint8_t* payload, uint32_t sideband,
                        float super, float cs, float czp, float* out, int8_t* lv) {
  const ccqo_scheme* s = &p->s;
  const int bpw = s->stored_word_bytes;
  const int wide = bpw == 2;
  uint32_t scale_code = sideband;
  if (p->g.embedded_scale) {
    const uint8_t* tail = payload + p->g.full_words * bpw;
    scale_code = load_word(tail, wide) & s->scale_mask;
  }
  const float scale = (float)scale_code * super;

  int idx = 0;
  const uint8_t* q = payload;
  for (int w = 0; w < p->g.full_words; ++w, q += bpw) {
    uint32_t code = load_word(q, wide);
    if (s->uses_cluster) {
      uint16_t c;
      if (ccqo_clustered_code_value((uint8_t)code, cs, czp, s->code_bits, &c) != CCQO_OK)
        return CCQO_DOMAIN;
      code = c;
    }
    for (int k = 0; k < s->weights_per_word; ++k) {
      const int state = (int)((code >> s->shifts[k]) & s->weight_mask);
      if (out) out[idx] = (float)(state - s->zero_point) * scale;
      if (lv) lv[idx] = (int8_t)(state - s->zero_point);
      ++idx;
    }
  }
  if (p->g.has_tail) {
    uint32_t code = load_word(q, wide);
    if (s->uses_cluster) {
      uint16_t c;
      if (ccqo_clustered_code_value((uint8_t)code, cs, czp, s->code_bits, &c) != CCQO_OK)
        return CCQO_DOMAIN;
      code = c;
    }
    const int state = (int)((code >> s->shifts[0]) & s->weight_mask);
    if (out) out[idx] = (float)(state - s->zero_point) * scale;
    if (lv) lv[idx] = (int8_t)(state - s->zero_point);
  }
  return CCQO_OK;
}

static int decode_all(const ccqo_model* m, float* out, int8_t* lv) {
  plan_t p;
  int st = make_plan(m, &p);
  if (st != CCQO_OK) return st;
  const int64_t gpr = m->cols / m->group_size;
  for (int64_t r = 0; r < m->rows; ++r) {
    const float super = m->super_scales[r];
    const float cs = p.s.uses_cluster ? m->cluster_scales[r] : 0.0f;
    const float czp = p.s.uses_cluster ? m->cluster_zero_points[r] : 0.0f;
    for (int64_t gj = 0; gj < gpr; ++gj) {
      const int64_t gi = r * gpr + gj;
      const size_t off = (size_t)(r * m->cols + gj * m->group_size);
      st = decode_group(&p, m->code_payload + gi * p.g.payload_bytes,
                        p.g.embedded_scale ? 0 : sideband_code(m, gi), super, cs, czp,
                        out ? out + off : NULL, lv ? lv + off : NULL);
      if (st != CCQO_OK) return st;
    }
  }
  return CCQO_OK;
}

int ccqo_dequantize(const ccqo_model* m, float* out) { return decode_all(m, out, NULL); }

int ccqo_levels(const ccqo_model* m, int8_t* out) { return decode_all(m, NULL, out); }

int ccqo_group_scales(const ccqo_model* m, float* out) {
  plan_t p;
  int st = make_plan(m, &p);
  if (st != CCQO_OK) return st;
  const int64_t gpr = m->cols / m->group_size;
  const int wide = p.s.stored_word_bytes == 2;
  for (int64_t gi = 0; gi < m->rows * gpr; ++gi) {
    uint32_t code;
    if (p.g.embedded_scale) {
      const uint8_t* tail =
          m->code_payload + gi * p.g.payload_bytes + p.g.full_words * p.s.stored_word_bytes;
      code = load_word(tail, wide) & p.s.scale_mask;
    } else {
      code = sideband_code(m, gi);
    }
    out[gi] = (float)code * m->super_scales[gi / gpr];
  }
  return CCQO_OK;
}

/* gemv_batch (kernels.cpp:152-187) over a contiguous row range. */
static int gemv_rows(const ccqo_model* m, const plan_t* p, const float* x, int64_t batch,
                     float* y, int64_t r0, int64_t r1) {
  const int64_t gpr = m->cols / m->group_size;
  float* decoded = (float*)malloc(sizeof(float) * (size_t)m->group_size);
  double* acc = (double*)malloc(sizeof(double) * (size_t)(batch > 0 ? batch : 1));
  if (!decoded || !acc) {
    free(decoded);
    free(acc);
    return CCQO_DOMAIN;
  }
  int st = CCQO_OK;
  for (int64_t r = r0; r < r1 && st == CCQO_OK; ++r) {
    const float super = m->super_scales[r];
    const float cs = p->s.uses_cluster ? m->cluster_scales[r] : 0.0f;
    const float czp = p->s.uses_cluster ? m->cluster_zero_points[r] : 0.0f;
    for (int64_t b = 0; b < batch; ++b) acc[b] = 0.0;
    for (int64_t gj = 0; gj < gpr; ++gj) {
      const int64_t gi = r * gpr + gj;
      st = decode_group(p, m->code_payload + gi * p->g.payload_bytes,
                        p->g.embedded_scale ? 0 : sideband_code(m, gi), super, cs, czp,
                        decoded, NULL);
      if (st != CCQO_OK) break;
      const int64_t col0 = gj * m->group_size;
      for (int64_t b = 0; b < batch; ++b) {
        const float* xg = x + b * m->cols + col0;
        double a = acc[b];
        for (int i = 0; i < m->group_size; ++i) a += (double)decoded[i] * (double)xg[i];
        acc[b] = a;
      }
    }
    for (int64_t b = 0; b < batch; ++b) y[b * m->rows + r] = (float)acc[b];
  }
  free(decoded);
  free(acc);
  return st;
}

int ccqo_gemv_batch(const ccqo_model* m, const float* x, int64_t batch, float* y) {
  plan_t p;
  int st = make_plan(m, &p);
  if (st != CCQO_OK) return st;
  if (batch < 0) return CCQO_SHAPE;
  return gemv_rows(m, &p, x, batch, y, 0, m->rows);
}

typedef struct {
  const ccqo_model* m;
  const plan_t* p;
  const float* x;
  int64_t batch;
  float* y;
  int64_t r0, r1;
  int status;
} shard_t;

static void* shard_main(void* arg) {
  shard_t* s = (shard_t*)arg;
  s->status = gemv_rows(s->m, s->p, s->x, s->batch, s->y, s->r0, s->r1);
  return NULL;
}

int ccqo_gemv_batch_mt(const ccqo_model* m, const float* x, int64_t batch, float* y,
                       int threads) {
  plan_t p;
  int st = make_plan(m, &p);
  if (st != CCQO_OK) return st;
  if (threads <= 1 || m->rows < 2) return gemv_rows(m, &p, x, batch, y, 0, m->rows);
  if (threads > m->rows) threads = (int)m->rows;
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  shard_t* sh = (shard_t*)calloc((size_t)threads, sizeof(shard_t));
  for (int t = 0; t < threads; ++t) {
    sh[t].m = m;
    sh[t].p = &p;
    sh[t].x = x;
    sh[t].batch = batch;
    sh[t].y = y;
    sh[t].r0 = m->rows * t / threads;
    sh[t].r1 = m->rows * (t + 1) / threads;
    pthread_create(&tid[t], NULL, shard_main, &sh[t]);
  }
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    if (sh[t].status != CCQO_OK) st = sh[t].status;
  }
  free(tid);
  free(sh);
  return st;
}

/* model_payload_bytes (kernels.cpp:203-207). */
uint64_t ccqo_payload_bytes(const ccqo_model* m) {
  ccqo_scheme s;
  ccqo_scheme_for(m->family, &s);
  return (uint64_t)m->code_bytes + m->scale_bytes + (uint64_t)m->rows * 4 +
         (s.uses_cluster ? (uint64_t)m->rows * 8 : 0);
}

/* ------------------------------------------------------------------ */
/* Deterministic generators: tensor.cpp:37-69, synthetic.cpp:25-103    */
/* ------------------------------------------------------------------ */

/* std::mt19937_64 (the C++ standard's parameters). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64_t* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* unit_double (tensor.cpp:37-41): 53 random bits in [0, 1). */
static inline double unit_double(mt64_t* g) {
  return (double)(mt64_next(g) >> 11) * 0x1.0p-53;
}

void ccqo_random_matrix(int64_t rows, int64_t cols, int dist, uint64_t seed, float* out) {
  mt64_t* g = (mt64_t*)malloc(sizeof(mt64_t));
  mt64_seed(g, seed);
  const size_t n = (size_t)(rows * cols);
  if (dist == 1) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)(2.0 * unit_double(g) - 1.0);
    free(g);
    return;
  }
  const double pi = 3.141592653589793; /* std::numbers::pi */
  size_t i = 0;
  while (i < n) {
    double u1 = unit_double(g);
    while (u1 <= 0.0) u1 = unit_double(g);
    const double u2 = unit_double(g);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * pi * u2;
    out[i++] = (float)(r * cos(a));
    if (i < n) out[i++] = (float)(r * sin(a));
  }
  free(g);
}

/* pack_cluster_scales / unpack_cluster_scales (packing.cpp:160-184). */
int ccqo_pack_cluster_scales(const uint16_t* codes, size_t n, uint8_t* out) {
  memset(out, 0, (n + 1) / 2);
  for (size_t i = 0; i < n; ++i) {
    if (codes[i] > 0xF) return CCQO_ENCODING;
    out[i / 2] |= (uint8_t)(codes[i] << (4 * (i % 2)));
  }
  return CCQO_OK;
}

int ccqo_unpack_cluster_scales(const uint8_t* bytes, size_t nbytes, size_t group_count,
                               uint16_t* out) {
  if (nbytes != (group_count + 1) / 2) return CCQO_ENCODING;
  for (size_t i = 0; i < group_count; ++i) out[i] = (bytes[i / 2] >> (4 * (i % 2))) & 0xF;
  return CCQO_OK;
}

/* pack_group (packing.cpp:71-114). */
int ccqo_pack_group(const uint16_t* codes, size_t n_codes, uint16_t scale_code, int family,
                    int group_size, uint8_t* payload, uint16_t* sideband) {
  ccqo_scheme s;
  ccqo_geometry g;
  if (ccqo_scheme_for(family, &s) != CCQO_OK) return CCQO_CONFIG;
  if (ccqo_group_geometry(family, group_size, &g) != CCQO_OK) return CCQO_CONFIG;
  if (n_codes != (size_t)g.words_per_group) return CCQO_ENCODING;
  if (scale_code >= (1u << s.scale_bits)) return CCQO_ENCODING;
  const uint32_t limit = s.uses_cluster ? 0x100u : (1u << s.code_bits);
  for (int w = 0; w < g.full_words; ++w)
    if (codes[w] >= limit) return CCQO_ENCODING;
  const int wb = s.stored_word_bytes * 8;
  const uint16_t tail_mask = (uint16_t)(s.weight_mask << (wb - s.state_bits));
  uint8_t* o = payload;
  for (int w = 0; w < g.words_per_group; ++w) {
    uint16_t word = codes[w];
    if (w == g.full_words) { /* tail */
      if (s.uses_cluster) {
        if (word >= limit) return CCQO_ENCODING;
      } else {
        if ((word & ~tail_mask) != 0) return CCQO_ENCODING;
        word = (uint16_t)(word | scale_code);
      }
    }
    *o++ = (uint8_t)(word & 0xFF);
    if (s.stored_word_bytes == 2) *o++ = (uint8_t)(word >> 8);
  }
  *sideband = g.embedded_scale ? 0 : scale_code;
  return CCQO_OK;
}

/* pack_model(random_quantized(...)): synthetic.cpp:25-103 draws, then
 * container.cpp:323-358 packs.  The draw order is reproduced exactly:
 * all per-row reals first, then per group its words and its scale code. */
int ccqo_random_packed(int64_t rows, int64_t cols, int family, int group_size, uint64_t seed,
                       uint8_t* code_payload, uint8_t* scale_payload, float* super_scales,
                       float* cluster_scales, float* cluster_zero_points) {
  ccqo_scheme s;
  ccqo_geometry g;
  if (rows < 0 || cols < 0) return CCQO_SHAPE;
  if (group_size <= 0 || cols % group_size != 0) return CCQO_SHAPE;
  if (ccqo_scheme_for(family, &s) != CCQO_OK) return CCQO_CONFIG;
  if (ccqo_group_geometry(family, group_size, &g) != CCQO_OK) return CCQO_CONFIG;

  mt64_t* rng = (mt64_t*)malloc(sizeof(mt64_t));
  mt64_seed(rng, seed);
  for (int64_t r = 0; r < rows; ++r) {
    super_scales[r] = (float)(0.001 + 0.05 * unit_double(rng));
    if (s.uses_cluster) {
      const double limit = (double)((1u << s.code_bits) - 1u);
      const double alpha = 1.0 + unit_double(rng) * (limit / 512.0);
      const double beta = unit_double(rng) * (limit - 255.0 * alpha);
      cluster_scales[r] = (float)alpha;
      cluster_zero_points[r] = (float)beta;
    }
  }

  const int64_t gpr = cols / group_size;
  const int64_t groups = rows * gpr;
  const int wpg = g.words_per_group;
  const uint32_t full_mask = s.uses_cluster ? 0xFFu : (s.word_bits == 8 ? 0xFFu : 0xFFFFu);
  const uint32_t state_mask = (1u << s.state_bits) - 1u;
  const int tail_shift = s.word_bits - s.state_bits;
  const uint32_t scale_limit = 1u << s.scale_bits;
  uint16_t words[64 + 1];
  uint16_t* scale_codes = g.embedded_scale ? NULL : (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(groups ? groups : 1));
  int st = CCQO_OK;
  for (int64_t gi = 0; gi < groups && st == CCQO_OK; ++gi) {
    const int64_t row = gi / gpr;
    uint16_t* w = wpg <= 65 ? words : NULL;
    uint16_t* heap = NULL;
    if (!w) w = heap = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)wpg);
    for (int k = 0; k < g.full_words; ++k) w[k] = (uint16_t)(mt64_next(rng) & full_mask);
    if (g.has_tail) {
      w[wpg - 1] = s.uses_cluster ? (uint16_t)(mt64_next(rng) & 0xFF)
                                  : (uint16_t)((mt64_next(rng) & state_mask) << tail_shift);
    }
    if (s.uses_cluster) {
      /* random_quantized widens each byte (synthetic.cpp:89-96) and throws on
       * an out-of-range reconstruction; the stored bytes are the q's. */
      for (int k = 0; k < wpg; ++k) {
        uint16_t c;
        if (ccqo_clustered_code_value((uint8_t)w[k], cluster_scales[row],
                                      cluster_zero_points[row], s.code_bits,
                                      &c) != CCQO_OK) {
          st = CCQO_DOMAIN;
          break;
        }
      }
    }
    const uint16_t sc = (uint16_t)(mt64_next(rng) % scale_limit);
    uint16_t side = 0;
    if (st == CCQO_OK)
      st = ccqo_pack_group(w, (size_t)wpg, sc, family, group_size,
                           code_payload + gi * g.payload_bytes, &side);
    if (scale_codes) scale_codes[gi] = sc;
    free(heap);
  }
  if (st == CCQO_OK && scale_codes)
    st = ccqo_pack_cluster_scales(scale_codes, (size_t)groups, scale_payload);
  free(scale_codes);
  free(rng);
  return st;
}
