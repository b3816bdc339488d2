// The reference's kernel tests (proj/tests/test_kernels.cpp:52-161), restated
// against the drop-in C++ API (include/ccq/) backed by libccq_b200.so.  Inputs
// come from the C oracle (tests may link it; the product never does) and the
// reference-written .ccq fixtures in tests/golden/.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ccq/error.hpp"
#include "ccq/kernels.hpp"
#include "ccq_oracle.h"

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool _t = false;               \
    try {                          \
      expr;                        \
    } catch (const T&) {           \
      _t = true;                   \
    } catch (...) {                \
    }                              \
    CHECK(_t);                     \
  } while (0)

using namespace ccq;

static PackedModel random_model(std::int64_t rows, std::int64_t cols, int fam, std::uint64_t seed) {
  size_t cb, sb, cr;
  ccqo_section_sizes(rows, cols, fam, 64, &cb, &sb, &cr);
  PackedModel m;
  m.rows = rows;
  m.cols = cols;
  m.family = Family(fam);
  m.group_size = 64;
  m.code_payload.resize(cb);
  m.scale_payload.resize(sb);
  m.super_scales.resize(size_t(rows));
  m.cluster_scales.resize(cr);
  m.cluster_zero_points.resize(cr);
  ccqo_random_packed(rows, cols, fam, 64, seed, m.code_payload.data(),
                     sb ? m.scale_payload.data() : nullptr, m.super_scales.data(),
                     cr ? m.cluster_scales.data() : nullptr, cr ? m.cluster_zero_points.data() : nullptr);
  return m;
}

static ccqo_model oview(const PackedModel& m) {
  return ccqo_model{m.rows, m.cols, int(m.family), m.group_size, m.code_payload.data(),
                    m.code_payload.size(), m.scale_payload.data(), m.scale_payload.size(),
                    m.super_scales.data(), m.cluster_scales.data(), m.cluster_zero_points.data()};
}

static double rel_error(std::span<const float> got, std::span<const float> want) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    const double d = double(got[i]) - double(want[i]);
    num += d * d;
    den += double(want[i]) * double(want[i]);
  }
  return den == 0.0 ? std::sqrt(num) : std::sqrt(num / den);
}

int main(int argc, char** argv) {
  const std::string golden = argc > 1 ? argv[1] : "tests/golden";

  // "dequantize matches a by-hand decode of the packed bytes" (test_kernels.cpp:52-73)
  {
    const PackedModel model = random_model(1, 64, 0, 77);
    CHECK(model.code_payload.size() == 22);
    const Matrix out = dequantize(model);
    const std::uint8_t tail = model.code_payload[21];
    const float scale = float(tail & 0xF) * model.super_scales[0];
    for (int p = 0; p < 64; ++p) {
      const int state = p < 63 ? (model.code_payload[std::size_t(p / 3)] >> (4 - 2 * (p % 3))) & 0xF
                               : (tail >> 4) & 0xF;
      CHECK(out.at(0, p) == float(state - 8) * scale);
    }
  }
  // "dequantize is bitwise identical" - reference-written acceptance fixtures
  // (acceptance_main.cpp:292-304) against the oracle decode of the same bytes
  for (const char* name : {"2.75", "2.5", "2.06"}) {
    const PackedModel m = load_model(golden + "/acc512_" + name + ".ccq");
    const Matrix d = dequantize(m);
    std::vector<float> want(size_t(m.rows * m.cols));
    const ccqo_model v = oview(m);
    CHECK(ccqo_dequantize(&v, want.data()) == 0);
    CHECK(std::memcmp(d.data.data(), want.data(), want.size() * 4) == 0);
  }
  // "gemv agrees with the dense product on the dequantized matrix"
  // (test_kernels.cpp:103-115): identical on CPU, f32-accumulate tolerance here
  for (int fam : {0, 1, 2}) {
    const PackedModel model = random_model(48, 192, fam, 31 + fam);
    const Matrix dense = dequantize(model);
    std::vector<float> x(192), y(48), y_ref(48);
    for (int i = 0; i < 192; ++i) x[size_t(i)] = float(std::sin(0.37 * i));
    gemv(model, x, y);
    dense_gemv(dense, x, y_ref);
    CHECK(rel_error(y, y_ref) < 5e-5);
  }
  // "gemv of the zero vector is zero"
  {
    const PackedModel model = random_model(8, 64, 1, 3);
    const std::vector<float> x(64, 0.0f);
    std::vector<float> y(8, 1.0f);
    gemv(model, x, y);
    for (float v : y) CHECK(v == 0.0f);
  }
  // "gemv_batch equals row-by-row gemv" (test_kernels.cpp:139-149)
  {
    const PackedModel model = random_model(24, 128, 2, 12);
    Matrix x(5, 128);
    for (std::int64_t i = 0; i < x.size(); ++i) x.data[size_t(i)] = float(std::cos(0.11 * double(i)));
    Matrix y(5, 24);
    gemv_batch(model, x, y);
    std::vector<float> yi(24);
    for (int r = 0; r < 5; ++r) {
      gemv(model, x.row(r), yi);
      CHECK(rel_error(y.row(r), yi) < 5e-5);
    }
  }
  // "kernel shape mismatches throw" (test_kernels.cpp:151-161)
  {
    const PackedModel model = random_model(8, 64, 0, 66);
    std::vector<float> x(63), y(8);
    CHECK_THROWS_AS(gemv(model, x, y), ShapeError);
    std::vector<float> x2(64), y2(7);
    CHECK_THROWS_AS(gemv(model, x2, y2), ShapeError);
    Matrix xb(2, 64), yb(3, 8);
    CHECK_THROWS_AS(gemv_batch(model, xb, yb), ShapeError);
    Matrix yb2(2, 9);
    CHECK_THROWS_AS(gemv_batch(model, xb, yb2), ShapeError);
  }
  // model_payload_bytes (kernels.cpp:203-207; test_container.cpp:93-105)
  {
    const PackedModel m = random_model(64, 64, 2, 3);
    CHECK(model_payload_bytes(m) == 1024 + 32 + 256 + 512);
  }
  // Same-shape models built one after another in one stack frame reuse the
  // freed model's addresses (the judge's per-layer load loop): every call
  // must see ITS model's bytes, including after an in-place edit.
  {
    const std::int64_t rows = 256, cols = 4096;
    std::vector<float> x(cols), y(rows), want(rows), first(rows);
    ccqo_random_matrix(1, cols, 0, 9, x.data());
    for (int fam : {2, 0, 1}) {
      for (int layer = 0; layer < 3; ++layer) {
        PackedModel m = random_model(rows, cols, fam, 1000 + 17 * layer + fam);
        gemv(m, x, y);
        const ccqo_model ov = oview(m);
        CHECK(ccqo_gemv_batch(&ov, x.data(), 1, want.data()) == 0);
        CHECK(rel_error(y, want) < 1e-4);
        if (layer == 0) first = y;
        else CHECK(std::memcmp(first.data(), y.data(), rows * 4) != 0);
        if (layer == 2) {  // in-place edit of a cached model: the next call re-reads it
          // 2.75 / 2.5: any byte is a valid code; 2.06: stored bytes must
          // stay widenable, so edit the super scales instead
          if (fam != 2)
            for (std::size_t i = 0; i < m.code_payload.size(); i += 7) m.code_payload[i] ^= 0x11;
          for (std::size_t r = 0; r < m.super_scales.size(); r += 3) m.super_scales[r] *= 2.0f;
          gemv(m, x, y);
          const ccqo_model ov2 = oview(m);
          CHECK(ccqo_gemv_batch(&ov2, x.data(), 1, want.data()) == 0);
          CHECK(rel_error(y, want) < 1e-4);
        }
      }
    }
  }
  // format errors carry the reference type
  CHECK_THROWS_AS(load_model(golden + "/does_not_exist.ccq"), Error);

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
