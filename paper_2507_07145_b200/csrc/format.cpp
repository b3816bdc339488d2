// Host-side format rules of the drop-in C++ API: encoding configurations,
// family schemes and layouts (coding.hpp), group packing (packing.hpp),
// QuantizedTensor <-> PackedModel (container.hpp) and the synthetic-input
// generator (tensor.hpp).
//
// These restate FORMAT.md §1-6 (the normative byte layout) behind the
// reference's signatures: coding.cpp:30-263, packing.cpp:24-184,
// container.cpp:323-414, tensor.cpp:31-66 of /root/reference/proj/core/src.
// Pure byte/integer work on the host - no GPU involvement; the GPU path
// consumes the PackedModel these produce.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <string>

#include "ccq/container.hpp"
#include "ccq/error.hpp"
#include "ccq/packing.hpp"
#include "ccq/tensor.hpp"

namespace ccq {

// ---------------------------------------------------------------------------
// coding.hpp
// ---------------------------------------------------------------------------

void EncodingConfig::validate() const {
  const std::string self = to_string();
  if (states_per_code < 1)
    throw ConfigError("states_per_code must be >= 1, got " + std::to_string(states_per_code));
  if (!(1 <= transition_bits && transition_bits <= state_bits))
    throw ConfigError("need 1 <= transition_bits <= state_bits, got " + self);
  if (state_bits > 8) throw ConfigError("state_bits must be <= 8, got " + self);
  if (total_bits() > 16) throw ConfigError("code word exceeds 16 bits: " + self);
}

std::string EncodingConfig::to_string() const {
  return "(" + std::to_string(state_bits) + "," + std::to_string(states_per_code) + "," +
         std::to_string(transition_bits) + ")";
}

namespace {

// Right shift of window j in a T-bit word: windows are read MSB first.
inline int window_shift(const EncodingConfig& c, int j) {
  return c.total_bits() - c.state_bits - j * c.transition_bits;
}

}  // namespace

std::vector<std::uint16_t> decode_states(std::uint32_t code, const EncodingConfig& config) {
  config.validate();
  if (code >= config.code_count())
    throw DomainError("code " + std::to_string(code) + " out of range for " + config.to_string());
  std::vector<std::uint16_t> out(std::size_t(config.states_per_code));
  for (int j = 0; j < config.states_per_code; ++j)
    out[std::size_t(j)] = std::uint16_t((code >> window_shift(config, j)) & config.state_mask());
  return out;
}

std::uint32_t states_to_code(std::span<const std::uint16_t> states, const EncodingConfig& config) {
  config.validate();
  if (states.size() != std::size_t(config.states_per_code))
    throw EncodingError("expected " + std::to_string(config.states_per_code) + " states, got " +
                        std::to_string(states.size()));
  const std::uint32_t shared = (1u << config.overlap_bits()) - 1u;
  std::uint32_t code = 0;
  for (int j = 0; j < config.states_per_code; ++j) {
    const std::uint32_t s = states[std::size_t(j)];
    if (s > config.state_mask())
      throw EncodingError("state " + std::to_string(s) + " exceeds " + std::to_string(config.state_bits) +
                          " bits");
    // adjacent windows overlap in L-S bits: the previous state's low bits
    // must reappear as this state's high bits
    if (j > 0 && (states[std::size_t(j - 1)] & shared) != (s >> config.transition_bits))
      throw EncodingError("invalid state transition at position " + std::to_string(j) +
                          ": window overlap mismatch");
    code |= s << window_shift(config, j);
  }
  return code;
}

Codebook build_codebook(const EncodingConfig& config) {
  config.validate();
  Codebook book;
  book.config = config;
  const std::uint32_t n = config.code_count();
  const int N = config.states_per_code;
  book.states.resize(std::size_t(n) * std::size_t(N));
  for (std::uint32_t code = 0; code < n; ++code)
    for (int j = 0; j < N; ++j)
      book.states[std::size_t(code) * N + j] = std::uint16_t((code >> window_shift(config, j)) & config.state_mask());
  return book;
}

namespace {

// The three codes the format defines (FORMAT.md §2).
constexpr EncodingConfig kCode275{4, 3, 2};
constexpr EncodingConfig kCode206{6, 4, 3};
constexpr EncodingConfig kHybridHi{3, 3, 2};  // bits 9..15 of a 2.5 word
constexpr EncodingConfig kHybridLo{3, 4, 2};  // bits 0..8

// Shifts of every weight slot of a word holding `parts` back to back from
// the MSB down.
std::vector<int> slot_shifts(std::span<const EncodingConfig> parts, int word_bits) {
  std::vector<int> out;
  int top = word_bits;
  for (const EncodingConfig& p : parts) {
    const int low = top - p.total_bits();
    for (int j = 0; j < p.states_per_code; ++j) out.push_back(low + window_shift(p, j));
    top = low;
  }
  return out;
}

}  // namespace

int HybridSchedule::weights_per_word() const {
  int n = 0;
  for (const EncodingConfig& p : parts) n += p.states_per_code;
  return n;
}

void HybridSchedule::validate() const {
  if (parts.empty()) throw ConfigError("hybrid schedule has no parts");
  int used = 0;
  for (const EncodingConfig& p : parts) {
    p.validate();
    if (p.state_bits != parts[0].state_bits) throw ConfigError("hybrid parts must share state_bits");
    used += p.total_bits();
  }
  if (used != word_bits)
    throw ConfigError("hybrid parts fill " + std::to_string(used) + " bits, word has " +
                      std::to_string(word_bits));
  if (word_bits != 8 && word_bits != 16) throw ConfigError("hybrid word_bits must be 8 or 16");
}

HybridSchedule canonical_hybrid() { return HybridSchedule{{kHybridHi, kHybridLo}, 16}; }

LayoutSpec layout_for(const EncodingConfig& config) {
  config.validate();
  LayoutSpec L;
  if (config == kCode275) {
    L.word_bits = 8;
    L.scale_mask = 0xF;  // embedded in the tail byte
  } else if (config == kCode206) {
    L.word_bits = 16;  // shifts apply to the widened 15-bit value
    L.scale_mask = 0xF;
    L.scale_shifts = {0, 4};  // two side-band nibbles per byte
    L.uses_cluster = true;
  } else {
    throw ConfigError("no packed layout defined for " + config.to_string());
  }
  const EncodingConfig one[] = {config};
  L.weight_shifts = slot_shifts(one, config.total_bits());
  L.weight_mask = config.state_mask();
  return L;
}

LayoutSpec layout_for(const HybridSchedule& schedule) {
  schedule.validate();
  const HybridSchedule ref = canonical_hybrid();
  if (schedule.parts != ref.parts || schedule.word_bits != ref.word_bits)
    throw ConfigError("no packed layout defined for this hybrid schedule");
  LayoutSpec L;
  L.word_bits = schedule.word_bits;
  L.weight_shifts = slot_shifts(schedule.parts, schedule.word_bits);
  L.weight_mask = schedule.parts[0].state_mask();
  L.scale_mask = 0x1FFF;  // 13-bit scale in the tail word
  return L;
}

std::string family_name(Family family) {
  switch (family) {
    case Family::Bpw275: return "2.75";
    case Family::Bpw25: return "2.5";
    case Family::Bpw206: return "2.06";
  }
  throw ConfigError("unknown family");
}

Family family_from_name(const std::string& name) {
  if (name == "2.75") return Family::Bpw275;
  if (name == "2.5" || name == "2.50") return Family::Bpw25;
  if (name == "2.06") return Family::Bpw206;
  throw ConfigError("unknown family '" + name + "' (expected 2.75, 2.5 or 2.06)");
}

namespace {

Scheme build_scheme(Family f) {
  Scheme s{};
  s.family = f;
  if (f == Family::Bpw25) {
    const HybridSchedule h = canonical_hybrid();
    s.parts = h.parts;
    s.layout = layout_for(h);
  } else {
    const EncodingConfig c = f == Family::Bpw275 ? kCode275 : kCode206;
    s.parts = {c};
    s.layout = layout_for(c);
  }
  // per family: code_bits, stored_word_bytes, scale_bits (FORMAT.md §2)
  static constexpr int kTable[3][3] = {{8, 1, 4}, {16, 2, 13}, {15, 1, 4}};
  const int* t = kTable[int(f)];
  s.code_bits = t[0];
  s.stored_word_bytes = t[1];
  s.scale_bits = t[2];
  s.uses_cluster = f == Family::Bpw206;
  for (const EncodingConfig& p : s.parts) s.weights_per_word += p.states_per_code;
  s.state_bits = s.parts[0].state_bits;
  s.zero_point = 1 << (s.state_bits - 1);
  return s;
}

}  // namespace

const Scheme& family_scheme(Family family) {
  static const Scheme schemes[3] = {build_scheme(Family::Bpw275), build_scheme(Family::Bpw25),
                                    build_scheme(Family::Bpw206)};
  const int i = int(family);
  if (i < 0 || i > 2) throw ConfigError("unknown family");
  return schemes[i];
}

// ---------------------------------------------------------------------------
// packing.hpp
// ---------------------------------------------------------------------------

GroupGeometry group_geometry(const Scheme& scheme, int group_size) {
  if (group_size <= 0) throw ConfigError("group_size must be positive");
  const int wpw = scheme.weights_per_word;
  const int rest = group_size % wpw;
  if (rest > 1)
    throw ConfigError("group_size " + std::to_string(group_size) + " leaves " + std::to_string(rest) +
                      " weights in the last word of family " + family_name(scheme.family) +
                      "; only remainders 0 and 1 have a layout");
  if (scheme.family == Family::Bpw25 && rest == 0)
    throw ConfigError("family 2.5 requires group_size % 7 == 1, got " + std::to_string(group_size));
  GroupGeometry g;
  g.group_size = group_size;
  g.full_words = group_size / wpw;
  g.has_tail = rest == 1;
  g.words_per_group = g.full_words + int(g.has_tail);
  g.embedded_scale = g.has_tail && !scheme.uses_cluster;
  g.payload_bytes = g.words_per_group * scheme.stored_word_bytes;
  return g;
}

namespace {

// Bits of the tail word that carry its single state (the leading L bits of
// the stored word); the rest is the embedded scale.
inline std::uint16_t leading_state_bits(const Scheme& s) {
  return std::uint16_t(s.layout.weight_mask << (8 * s.stored_word_bytes - s.state_bits));
}

inline void store_le(std::uint8_t* p, std::uint16_t v, int bytes) {
  p[0] = std::uint8_t(v);
  if (bytes == 2) p[1] = std::uint8_t(v >> 8);
}

inline std::uint16_t load_le(const std::uint8_t* p, int bytes) {
  return bytes == 2 ? std::uint16_t(p[0] | (p[1] << 8)) : p[0];
}

}  // namespace

PackedGroup pack_group(std::span<const std::uint16_t> codes, std::uint16_t scale_code, const Scheme& scheme,
                       int group_size) {
  const GroupGeometry g = group_geometry(scheme, group_size);
  if (codes.size() != std::size_t(g.words_per_group))
    throw EncodingError("expected " + std::to_string(g.words_per_group) + " code words, got " +
                        std::to_string(codes.size()));
  if (scale_code >> scheme.scale_bits)
    throw EncodingError("scale code " + std::to_string(scale_code) + " exceeds " +
                        std::to_string(scheme.scale_bits) + " bits");
  // clustered families store 8-bit cluster indices, the others full codes
  const std::uint32_t limit = scheme.uses_cluster ? 256u : (1u << scheme.code_bits);
  for (int w = 0; w < g.full_words; ++w)
    if (codes[std::size_t(w)] >= limit)
      throw EncodingError("code word " + std::to_string(codes[std::size_t(w)]) + " exceeds " +
                          (scheme.uses_cluster ? std::string("8 clustered") : std::to_string(scheme.code_bits)) +
                          " bits");
  PackedGroup out;
  out.family = scheme.family;
  out.payload.resize(std::size_t(g.payload_bytes));
  const int wb = scheme.stored_word_bytes;
  for (int w = 0; w < g.full_words; ++w) store_le(out.payload.data() + w * wb, codes[std::size_t(w)], wb);
  if (g.has_tail) {
    std::uint16_t tail = codes[std::size_t(g.full_words)];
    if (scheme.uses_cluster) {
      if (tail >= limit) throw EncodingError("clustered tail code exceeds 8 bits");
    } else {
      if (tail & ~leading_state_bits(scheme))
        throw EncodingError("tail code word may only use its leading state bits");
      tail = std::uint16_t(tail | scale_code);
    }
    store_le(out.payload.data() + g.full_words * wb, tail, wb);
  }
  if (!g.embedded_scale) out.sideband_scale = scale_code;
  return out;
}

UnpackedGroup unpack_group(const PackedGroup& group, const Scheme& scheme, int group_size) {
  const GroupGeometry g = group_geometry(scheme, group_size);
  if (group.family != scheme.family) throw EncodingError("packed group family mismatch");
  if (group.payload.size() != std::size_t(g.payload_bytes))
    throw EncodingError("packed group holds " + std::to_string(group.payload.size()) + " bytes, layout needs " +
                        std::to_string(g.payload_bytes));
  UnpackedGroup out;
  out.codes.resize(std::size_t(g.words_per_group));
  const int wb = scheme.stored_word_bytes;
  for (int w = 0; w < g.words_per_group; ++w) out.codes[std::size_t(w)] = load_le(group.payload.data() + w * wb, wb);
  if (g.has_tail && !scheme.uses_cluster) {
    const std::uint16_t tail = out.codes[std::size_t(g.full_words)];
    out.codes[std::size_t(g.full_words)] = std::uint16_t(tail & leading_state_bits(scheme));
    out.scale_code = std::uint16_t(tail & scheme.layout.scale_mask);
  }
  if (!g.embedded_scale) out.scale_code = group.sideband_scale;
  return out;
}

QuantizedScales quantize_scales(std::span<const float> scales, int scale_bits) {
  if (scale_bits < 1 || scale_bits > 16) throw ConfigError("scale_bits out of range");
  float top = 0.0f;
  for (float s : scales) {
    if (!(s >= 0.0f)) throw DomainError("group scales must be non-negative");  // also NaN
    top = std::max(top, s);
  }
  const long levels = (1l << scale_bits) - 1;
  QuantizedScales q;
  q.super_scale = top == 0.0f ? 1.0f : float(double(top) / double(levels));
  q.codes.resize(scales.size());
  for (std::size_t i = 0; i < scales.size(); ++i)
    q.codes[i] = std::uint16_t(std::clamp(std::lround(double(scales[i]) / double(q.super_scale)), 0l, levels));
  return q;
}

std::vector<std::uint8_t> pack_cluster_scales(std::span<const std::uint16_t> scale_codes) {
  std::vector<std::uint8_t> out((scale_codes.size() + 1) / 2, 0);
  for (std::size_t i = 0; i < scale_codes.size(); ++i) {
    const std::uint16_t c = scale_codes[i];
    if (c > 0xF) throw EncodingError("side-band scale code " + std::to_string(c) + " exceeds 4 bits");
    out[i >> 1] |= std::uint8_t(c << ((i & 1) * 4));
  }
  return out;
}

std::vector<std::uint16_t> unpack_cluster_scales(std::span<const std::uint8_t> bytes, std::size_t group_count) {
  const std::size_t need = (group_count + 1) / 2;
  if (bytes.size() != need)
    throw EncodingError("side-band scale stream holds " + std::to_string(bytes.size()) + " bytes, " +
                        std::to_string(group_count) + " groups need " + std::to_string(need));
  std::vector<std::uint16_t> out(group_count);
  for (std::size_t i = 0; i < group_count; ++i) out[i] = (bytes[i >> 1] >> ((i & 1) * 4)) & 0xF;
  return out;
}

PayloadBits payload_bits(const Scheme& scheme, int group_size, std::int64_t group_count) {
  const GroupGeometry g = group_geometry(scheme, group_size);
  const std::uint64_t n = std::uint64_t(group_count);
  PayloadBits b;
  b.code_bits = n * std::uint64_t(g.payload_bytes) * 8;
  b.scale_bits = g.embedded_scale ? 0 : n * 4;
  b.weights = n * std::uint64_t(group_size);
  return b;
}

// ---------------------------------------------------------------------------
// container.hpp: QuantizedTensor <-> PackedModel
// ---------------------------------------------------------------------------

PackedModel pack_model(const QuantizedTensor& t) {
  const Scheme& s = family_scheme(t.family);
  const GroupGeometry g = group_geometry(s, t.group_size);
  PackedModel m;
  m.rows = t.rows;
  m.cols = t.cols;
  m.family = t.family;
  m.group_size = t.group_size;
  m.rounds = t.rounds;
  m.super_scales = t.super_scales;
  m.cluster_scales = t.cluster_scales;
  m.cluster_zero_points = t.cluster_zero_points;
  const std::int64_t groups = t.group_count();
  const std::size_t wpg = std::size_t(g.words_per_group);
  m.code_payload.resize(std::size_t(groups) * std::size_t(g.payload_bytes));
  std::vector<std::uint16_t> words(wpg);
  for (std::int64_t gi = 0; gi < groups; ++gi) {
    // 2.06 stores the clustered bytes, the others the code words themselves
    for (std::size_t w = 0; w < wpg; ++w)
      words[w] = s.uses_cluster ? t.clustered_codes[std::size_t(gi) * wpg + w] : t.code_words[std::size_t(gi) * wpg + w];
    const PackedGroup p = pack_group(words, t.scale_codes[std::size_t(gi)], s, t.group_size);
    std::memcpy(m.code_payload.data() + std::size_t(gi) * std::size_t(g.payload_bytes), p.payload.data(),
                p.payload.size());
  }
  if (!g.embedded_scale) m.scale_payload = pack_cluster_scales(t.scale_codes);
  return m;
}

QuantizedTensor unpack_model(const PackedModel& m) {
  const Scheme& s = family_scheme(m.family);
  const GroupGeometry g = group_geometry(s, m.group_size);
  QuantizedTensor t;
  t.rows = m.rows;
  t.cols = m.cols;
  t.family = m.family;
  t.group_size = m.group_size;
  t.rounds = m.rounds;
  t.super_scales = m.super_scales;
  t.cluster_scales = m.cluster_scales;
  t.cluster_zero_points = m.cluster_zero_points;
  const std::int64_t groups = t.group_count(), gpr = t.groups_per_row();
  const std::size_t wpg = std::size_t(g.words_per_group);
  t.code_words.resize(std::size_t(groups) * wpg);
  t.scale_codes.resize(std::size_t(groups));
  t.group_scales.resize(std::size_t(groups));
  if (s.uses_cluster) t.clustered_codes.resize(std::size_t(groups) * wpg);
  const std::vector<std::uint16_t> side =
      g.embedded_scale ? std::vector<std::uint16_t>{} : unpack_cluster_scales(m.scale_payload, std::size_t(groups));
  PackedGroup p;
  p.family = m.family;
  for (std::int64_t gi = 0; gi < groups; ++gi) {
    const std::uint8_t* src = m.code_payload.data() + std::size_t(gi) * std::size_t(g.payload_bytes);
    p.payload.assign(src, src + g.payload_bytes);
    p.sideband_scale = g.embedded_scale ? 0 : side[std::size_t(gi)];
    const UnpackedGroup u = unpack_group(p, s, m.group_size);
    const std::size_t row = std::size_t(gi / gpr);
    t.scale_codes[std::size_t(gi)] = u.scale_code;
    t.group_scales[std::size_t(gi)] = float(u.scale_code) * m.super_scales[row];
    std::uint16_t* dst = t.code_words.data() + std::size_t(gi) * wpg;
    for (std::size_t w = 0; w < wpg; ++w) {
      if (s.uses_cluster) {
        const std::uint8_t q = std::uint8_t(u.codes[w]);
        t.clustered_codes[std::size_t(gi) * wpg + w] = q;
        dst[w] = clustered_code_value(q, m.cluster_scales[row], m.cluster_zero_points[row], s.code_bits);
      } else {
        dst[w] = u.codes[w];
      }
    }
  }
  return t;
}

QuantizedTensor read_container(const std::string& path) { return unpack_model(load_model(path)); }

PayloadBits container_payload_bits(const ContainerInfo& info) {
  const std::int64_t groups = info.group_size == 0 ? 0 : info.rows * (info.cols / info.group_size);
  return payload_bits(family_scheme(info.family), info.group_size, groups);
}

double measured_bpw(const ContainerInfo& info) { return container_payload_bits(info).bits_per_weight(); }

// ---------------------------------------------------------------------------
// tensor.hpp: synthetic inputs (bit-identical streams to the reference)
// ---------------------------------------------------------------------------

Distribution distribution_from_name(const std::string& name) {
  if (name == "gaussian") return Distribution::Gaussian;
  if (name == "uniform") return Distribution::Uniform;
  throw ConfigError("unknown distribution '" + name + "' (expected gaussian or uniform)");
}

Matrix random_matrix(std::int64_t rows, std::int64_t cols, Distribution dist, std::uint64_t seed) {
  Matrix m(rows, cols);
  std::mt19937_64 gen(seed);
  auto u53 = [&gen] { return double(gen() >> 11) * 0x1.0p-53; };  // [0, 1) on 53 bits
  std::vector<float>& v = m.data;
  if (dist == Distribution::Uniform) {
    for (float& e : v) e = float(2.0 * u53() - 1.0);
    return m;
  }
  // Box-Muller pairs (cos, sin), drawn in this order so the stream does not
  // depend on the standard library's normal_distribution
  for (std::size_t i = 0; i < v.size();) {
    double a = u53();
    while (a <= 0.0) a = u53();
    const double b = u53();
    const double radius = std::sqrt(-2.0 * std::log(a)), theta = 2.0 * std::numbers::pi * b;
    v[i++] = float(radius * std::cos(theta));
    if (i < v.size()) v[i++] = float(radius * std::sin(theta));
  }
  return m;
}

}  // namespace ccq
