// TEST INFRASTRUCTURE ONLY — C entry points over the UNMODIFIED reference
// CCQ library, compiled from /root/reference/proj/core/src by
// oracle/Makefile (namespace-isolated with -Dccq=ccq_ref) into
// oracle/_ref/libccq_ref.so.  Used by tests/ to pin the C oracle and by
// bench.py --impl reference / cpu_baseline as the reference CPU path.
// No reference source is copied here: this file only calls its public API
// (kernels.hpp:36-76, container.hpp:37-99, synthetic.hpp:30-31,
// quantizer.hpp:138-147, tensor.hpp:56-63).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "ccq/coding.hpp"
#include "ccq/container.hpp"
#include "ccq/error.hpp"
#include "ccq/kernels.hpp"
#include "ccq/quantizer.hpp"
#include "ccq/synthetic.hpp"
#include "ccq/tensor.hpp"

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ccq::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const ccq::DomainError& e) {
    g_err = e.what();
    return 2;
  } catch (const ccq::ShapeError& e) {
    g_err = e.what();
    return 3;
  } catch (const ccq::EncodingError& e) {
    g_err = e.what();
    return 4;
  } catch (const ccq::FormatError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

ccq::Family fam(int f) {
  switch (f) {
    case 0: return ccq::Family::Bpw275;
    case 1: return ccq::Family::Bpw25;
    case 2: return ccq::Family::Bpw206;
  }
  throw ccq::ConfigError("unknown family index");
}

int fam_index(ccq::Family f) {
  switch (f) {
    case ccq::Family::Bpw275: return 0;
    case ccq::Family::Bpw25: return 1;
    case ccq::Family::Bpw206: return 2;
  }
  return -1;
}

ccq::PackedModel* M(void* h) { return static_cast<ccq::PackedModel*>(h); }

// Contiguous row slice [r0, r1) of a packed model (groups_per_row even for
// side-band families so nibbles stay byte aligned; checked by the caller).
ccq::PackedModel slice_rows(const ccq::PackedModel& m, std::int64_t r0, std::int64_t r1) {
  const ccq::Scheme& s = ccq::family_scheme(m.family);
  const ccq::GroupGeometry g = ccq::group_geometry(s, m.group_size);
  const std::int64_t gpr = m.groups_per_row();
  ccq::PackedModel out;
  out.rows = r1 - r0;
  out.cols = m.cols;
  out.family = m.family;
  out.group_size = m.group_size;
  out.rounds = m.rounds;
  out.code_payload.assign(m.code_payload.begin() + r0 * gpr * g.payload_bytes,
                          m.code_payload.begin() + r1 * gpr * g.payload_bytes);
  if (!g.embedded_scale) {
    const std::int64_t g0 = r0 * gpr, g1 = r1 * gpr;
    out.scale_payload.resize(std::size_t((g1 - g0 + 1) / 2));
    for (std::int64_t gi = g0; gi < g1; ++gi) {
      const std::uint8_t nib = (m.scale_payload[std::size_t(gi / 2)] >> (4 * (gi % 2))) & 0xF;
      out.scale_payload[std::size_t((gi - g0) / 2)] |= std::uint8_t(nib << (4 * ((gi - g0) % 2)));
    }
  }
  out.super_scales.assign(m.super_scales.begin() + r0, m.super_scales.begin() + r1);
  if (s.uses_cluster) {
    out.cluster_scales.assign(m.cluster_scales.begin() + r0, m.cluster_scales.begin() + r1);
    out.cluster_zero_points.assign(m.cluster_zero_points.begin() + r0,
                                   m.cluster_zero_points.begin() + r1);
  }
  return out;
}

}  // namespace

extern "C" {

const char* ccqref_last_error() { return g_err.c_str(); }

void ccqref_free(void* h) { delete M(h); }

// pack_model(random_quantized(rows, cols, family, group_size, seed)).
int ccqref_model_random(std::int64_t rows, std::int64_t cols, int family, int group_size,
                        std::uint64_t seed, void** out) {
  return guard([&] {
    *out = new ccq::PackedModel(
        ccq::pack_model(ccq::random_quantized(rows, cols, fam(family), group_size, seed)));
  });
}

// pack_model(quantize_tensor(W)) for a caller-provided dense W; optionally
// returns the quantizer-side reconstruction (quantizer.cpp:427-447).
int ccqref_model_quantize(const float* w, std::int64_t rows, std::int64_t cols, int family,
                          int group_size, int rounds, int threads, float* recon_or_null,
                          void** out) {
  return guard([&] {
    ccq::Matrix m(rows, cols);
    std::memcpy(m.data.data(), w, sizeof(float) * std::size_t(rows * cols));
    ccq::QuantizerOptions opt;
    opt.family = fam(family);
    opt.group_size = group_size;
    opt.refinement_rounds = rounds;
    opt.threads = threads;
    const ccq::QuantizeResult r = ccq::quantize_tensor(m, opt);
    if (recon_or_null) {
      const ccq::Matrix rec = ccq::reconstruct(r.tensor);
      std::memcpy(recon_or_null, rec.data.data(), sizeof(float) * rec.data.size());
    }
    *out = new ccq::PackedModel(ccq::pack_model(r.tensor));
  });
}

int ccqref_model_from_sections(std::int64_t rows, std::int64_t cols, int family, int group_size,
                               int rounds, const std::uint8_t* code, std::size_t code_len,
                               const std::uint8_t* scale, std::size_t scale_len,
                               const float* super, const float* cs, const float* czp,
                               void** out) {
  return guard([&] {
    auto* m = new ccq::PackedModel();
    m->rows = rows;
    m->cols = cols;
    m->family = fam(family);
    m->group_size = group_size;
    m->rounds = rounds;
    m->code_payload.assign(code, code + code_len);
    if (scale_len) m->scale_payload.assign(scale, scale + scale_len);
    m->super_scales.assign(super, super + rows);
    if (ccq::family_scheme(m->family).uses_cluster) {
      m->cluster_scales.assign(cs, cs + rows);
      m->cluster_zero_points.assign(czp, czp + rows);
    }
    *out = m;
  });
}

// ccq::search_codes (quantizer.cpp:36-103) over n subvectors: targets[i] holds
// `valid` floats (row stride `stride`), scales[i] the group scale.
int ccqref_search_codes(const float* targets, std::int64_t n, int valid, int stride, const double* scales,
                        int zero_point, int state_bits, int states_per_code, int transition_bits,
                        std::uint32_t* codes) {
  return guard([&] {
    ccq::EncodingConfig cfg;
    cfg.state_bits = state_bits;
    cfg.states_per_code = states_per_code;
    cfg.transition_bits = transition_bits;
    for (std::int64_t i = 0; i < n; ++i)
      codes[i] = ccq::search_codes(std::span<const float>(targets + i * stride, std::size_t(valid)), scales[i],
                                   zero_point, cfg);
  });
}

int ccqref_load_model(const char* path, void** out) {
  return guard([&] { *out = new ccq::PackedModel(ccq::load_model(path)); });
}

int ccqref_write_container(void* h, const char* path) {
  return guard([&] { ccq::write_container(ccq::unpack_model(*M(h)), path); });
}

void ccqref_model_shape(void* h, std::int64_t* rows, std::int64_t* cols, int* family,
                        int* group_size, int* rounds, std::uint64_t* code_len,
                        std::uint64_t* scale_len, std::uint64_t* cluster_len) {
  const ccq::PackedModel& m = *M(h);
  *rows = m.rows;
  *cols = m.cols;
  *family = fam_index(m.family);
  *group_size = m.group_size;
  *rounds = m.rounds;
  *code_len = m.code_payload.size();
  *scale_len = m.scale_payload.size();
  *cluster_len = m.cluster_scales.size();
}

void ccqref_model_sections(void* h, std::uint8_t* code, std::uint8_t* scale, float* super,
                           float* cs, float* czp) {
  const ccq::PackedModel& m = *M(h);
  std::memcpy(code, m.code_payload.data(), m.code_payload.size());
  if (scale && !m.scale_payload.empty())
    std::memcpy(scale, m.scale_payload.data(), m.scale_payload.size());
  std::memcpy(super, m.super_scales.data(), m.super_scales.size() * 4);
  if (cs && !m.cluster_scales.empty())
    std::memcpy(cs, m.cluster_scales.data(), m.cluster_scales.size() * 4);
  if (czp && !m.cluster_zero_points.empty())
    std::memcpy(czp, m.cluster_zero_points.data(), m.cluster_zero_points.size() * 4);
}

std::uint64_t ccqref_payload_bytes(void* h) { return ccq::model_payload_bytes(*M(h)); }

int ccqref_dequantize(void* h, float* out) {
  return guard([&] {
    const ccq::Matrix d = ccq::dequantize(*M(h));
    std::memcpy(out, d.data.data(), d.data.size() * 4);
  });
}

// Centered levels via the quantizer-side decoder (quantizer.cpp:120-134).
int ccqref_levels(void* h, std::int8_t* out) {
  return guard([&] {
    const ccq::PackedModel& m = *M(h);
    const ccq::Scheme& s = ccq::family_scheme(m.family);
    const ccq::QuantizedTensor t = ccq::unpack_model(m);
    const std::int64_t wpg = t.words_per_group();
    const std::int64_t gpr = t.groups_per_row();
    for (std::int64_t gi = 0; gi < t.group_count(); ++gi) {
      const std::span<const std::uint16_t> words(t.code_words.data() + gi * wpg,
                                                 std::size_t(wpg));
      const std::vector<int> st = ccq::decode_group_states(words, s, t.group_size);
      const std::int64_t r = gi / gpr, gj = gi % gpr;
      for (int i = 0; i < t.group_size; ++i)
        out[r * t.cols + gj * t.group_size + i] = std::int8_t(st[std::size_t(i)] - s.zero_point);
    }
  });
}

int ccqref_gemv(void* h, const float* x, float* y) {
  return guard([&] {
    const ccq::PackedModel& m = *M(h);
    ccq::gemv(m, std::span<const float>(x, std::size_t(m.cols)),
              std::span<float>(y, std::size_t(m.rows)));
  });
}

int ccqref_gemv_batch(void* h, const float* x, std::int64_t batch, float* y) {
  return guard([&] {
    const ccq::PackedModel& m = *M(h);
    ccq::Matrix xm(batch, m.cols), ym(batch, m.rows);
    std::memcpy(xm.data.data(), x, sizeof(float) * xm.data.size());
    ccq::gemv_batch(m, xm, ym);
    std::memcpy(y, ym.data.data(), sizeof(float) * ym.data.size());
  });
}

// The reference gemv_batch run on contiguous row blocks, one std::thread per
// block (SURVEY §8d "all host cores").  Each output element is produced by
// the unmodified reference code.  Slicing happens before the timed call.
int ccqref_sliced_new(void* h, int parts, void** out_parts) {
  return guard([&] {
    const ccq::PackedModel& m = *M(h);
    for (int p = 0; p < parts; ++p) {
      const std::int64_t r0 = m.rows * p / parts, r1 = m.rows * (p + 1) / parts;
      out_parts[p] = new ccq::PackedModel(slice_rows(m, r0, r1));
    }
  });
}

int ccqref_gemv_batch_parts(void** parts, int nparts, const float* x, std::int64_t batch,
                            float* y, std::int64_t rows_total) {
  return guard([&] {
    std::vector<int> status(std::size_t(nparts), 0);
    std::vector<std::thread> th;
    std::int64_t r0 = 0;
    std::vector<ccq::Matrix> ys;
    ys.reserve(std::size_t(nparts));
    const ccq::PackedModel& first = *M(parts[0]);
    ccq::Matrix xm(batch, first.cols);
    std::memcpy(xm.data.data(), x, sizeof(float) * xm.data.size());
    for (int p = 0; p < nparts; ++p) ys.emplace_back(batch, M(parts[p])->rows);
    for (int p = 0; p < nparts; ++p) {
      th.emplace_back([&, p] {
        status[std::size_t(p)] = guard([&] { ccq::gemv_batch(*M(parts[p]), xm, ys[std::size_t(p)]); });
      });
    }
    for (auto& t : th) t.join();
    for (int p = 0; p < nparts; ++p) {
      if (status[std::size_t(p)] != 0) throw ccq::Error("shard failed: " + g_err);
      const std::int64_t rows = M(parts[p])->rows;
      for (std::int64_t b = 0; b < batch; ++b)
        std::memcpy(y + b * rows_total + r0, ys[std::size_t(p)].row(b).data(), sizeof(float) * rows);
      r0 += rows;
    }
  });
}

void ccqref_random_matrix(std::int64_t rows, std::int64_t cols, int dist, std::uint64_t seed,
                          float* out) {
  const ccq::Matrix m = ccq::random_matrix(
      rows, cols, dist == 0 ? ccq::Distribution::Gaussian : ccq::Distribution::Uniform, seed);
  std::memcpy(out, m.data.data(), m.data.size() * 4);
}

int ccqref_clustered_code_value(std::uint8_t q, float a, float b, int bits, std::uint16_t* out) {
  return guard([&] { *out = ccq::clustered_code_value(q, a, b, bits); });
}

int ccqref_group_geometry(int family, int group_size, int* out6) {
  return guard([&] {
    const ccq::GroupGeometry g = ccq::group_geometry(ccq::family_scheme(fam(family)), group_size);
    out6[0] = g.group_size;
    out6[1] = g.full_words;
    out6[2] = g.has_tail;
    out6[3] = g.words_per_group;
    out6[4] = g.embedded_scale;
    out6[5] = g.payload_bytes;
  });
}

}  // extern "C"
