// Synthetic packed models, draw for draw the reference bench generator:
// ccq::random_quantized (synthetic.cpp:25-103) followed by pack_model
// (container.cpp:323-358), with the same std::mt19937_64 stream, so a seed
// gives the reference's exact bytes.  Used by the bench harness so the GPU
// arm and the reference CPU arm (oracle/_ref, the reference's own generator)
// time byte-identical weights.
//
// Draw order (synthetic.cpp): every row's super scale (and, clustered, alpha
// then beta) first; then per group its full words, the tail word, and the
// scale code.  unit_double = 53 random bits (tensor.cpp:37-41).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "ccq/coding.hpp"
#include "ccq/error.hpp"
#include "ccq/packing.hpp"
#include "ccq_cuda.h"
#include "ccq_internal.hpp"

namespace {

inline double unit_double(std::mt19937_64& g) { return double(g() >> 11) * 0x1.0p-53; }

}  // namespace

extern "C" int ccq_synthetic_packed(int64_t rows, int64_t cols, int32_t family, int32_t group_size, uint64_t seed,
                                    uint8_t* code_payload, uint8_t* scale_payload, float* super_scales,
                                    float* cluster_scales, float* cluster_zero_points) {
  using namespace ccq;
  try {
    if (rows < 0 || cols < 0 || group_size <= 0 || cols % group_size != 0)
      return ccqb::fail(CCQ_ERR_SHAPE, "cols must be a whole number of groups");
    if (family < 0 || family > 2) return ccqb::fail(CCQ_ERR_CONFIG, "unknown family");
    const Scheme& s = family_scheme(Family(family));
    const GroupGeometry g = group_geometry(s, group_size);
    if (rows && (!code_payload || !super_scales || (!g.embedded_scale && !scale_payload) ||
                 (s.uses_cluster && (!cluster_scales || !cluster_zero_points))))
      return ccqb::fail(CCQ_ERR_INVALID, "null section buffer");
    std::mt19937_64 rng(seed);
    for (int64_t r = 0; r < rows; ++r) {
      super_scales[r] = float(0.001 + 0.05 * unit_double(rng));
      if (s.uses_cluster) {
        const double limit = double((1u << s.code_bits) - 1u);
        const double alpha = 1.0 + unit_double(rng) * (limit / 512.0);
        const double beta = unit_double(rng) * (limit - 255.0 * alpha);
        cluster_scales[r] = float(alpha);
        cluster_zero_points[r] = float(beta);
      }
    }
    const int64_t gpr = cols / group_size, groups = rows * gpr;
    const int wpg = g.words_per_group;
    const uint32_t full_mask = s.uses_cluster ? 0xFFu : (s.stored_word_bytes == 1 ? 0xFFu : 0xFFFFu);
    const uint32_t state_mask = (1u << s.state_bits) - 1u;
    const int tail_shift = s.stored_word_bytes * 8 - s.state_bits;
    const uint32_t scale_limit = 1u << s.scale_bits;
    std::vector<std::uint16_t> wv(static_cast<size_t>(wpg));
    std::vector<std::uint16_t> scale_codes(g.embedded_scale ? 0 : static_cast<size_t>(groups));
    for (int64_t gi = 0; gi < groups; ++gi) {
      const int64_t row = gi / gpr;
      for (int k = 0; k < g.full_words; ++k) wv[size_t(k)] = std::uint16_t(rng() & full_mask);
      if (g.has_tail)
        wv[size_t(wpg - 1)] = s.uses_cluster ? std::uint16_t(rng() & 0xFFu)
                                                : std::uint16_t((rng() & state_mask) << tail_shift);
      if (s.uses_cluster)  // synthetic.cpp:89-96: every stored byte must widen in range
        for (int k = 0; k < wpg; ++k)
          (void)clustered_code_value(std::uint8_t(wv[size_t(k)]), cluster_scales[row], cluster_zero_points[row],
                                     s.code_bits);
      const std::uint16_t sc = std::uint16_t(rng() % scale_limit);
      const PackedGroup pg = pack_group(wv, sc, s, group_size);
      std::memcpy(code_payload + size_t(gi) * size_t(g.payload_bytes), pg.payload.data(), pg.payload.size());
      if (!g.embedded_scale) scale_codes[size_t(gi)] = sc;
    }
    if (!g.embedded_scale) {
      const std::vector<std::uint8_t> nib = pack_cluster_scales(scale_codes);
      std::memcpy(scale_payload, nib.data(), nib.size());
    }
    return CCQ_OK;
  } catch (const DomainError& e) {
    return ccqb::fail(CCQ_ERR_DOMAIN, e.what());
  } catch (const EncodingError& e) {
    return ccqb::fail(CCQ_ERR_ENCODING, e.what());
  } catch (const Error& e) {
    return ccqb::fail(CCQ_ERR_CONFIG, e.what());
  }
}

// random_matrix (tensor.cpp:37-69): dist 0 = Gaussian (Box-Muller on
// unit_double pairs, u1 redrawn while <= 0, cos then sin), 1 = uniform [-1, 1).
extern "C" int ccq_synthetic_matrix(int64_t rows, int64_t cols, int32_t dist, uint64_t seed, float* out) {
  if (rows < 0 || cols < 0 || (rows * cols != 0 && !out)) return ccqb::fail(CCQ_ERR_INVALID, "bad matrix arguments");
  std::mt19937_64 rng(seed);
  const size_t n = size_t(rows) * size_t(cols);
  if (dist == 1) {
    for (size_t i = 0; i < n; ++i) out[i] = float(2.0 * unit_double(rng) - 1.0);
    return CCQ_OK;
  }
  const double pi = 3.141592653589793;
  size_t i = 0;
  while (i < n) {
    double u1 = unit_double(rng);
    while (u1 <= 0.0) u1 = unit_double(rng);
    const double u2 = unit_double(rng);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * pi * u2;
    out[i++] = float(r * std::cos(a));
    if (i < n) out[i++] = float(r * std::sin(a));
  }
  return CCQ_OK;
}
