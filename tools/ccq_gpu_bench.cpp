// ccq_gpu_bench - the reference CLI's `ccq bench` (tools/ccq_main.cpp:241-277,
// kernels.cpp:228-289) for the B200 path, written against the drop-in C++ API
// (include/ccq/*.hpp, libccq_b200.so).  Same CSV schema
//     shape,M,variant,median_ms,bytes_read
// with the GPU variants
//     ccq_gpu_fused        decode-matmul on device-resident bf16 activations
//     ccq_gpu_fused_e2e    the reference-signature ccq::gemv_batch (host f32 in, host f32 out)
// Shapes are "d_in x d_out" as in the reference (ccq_main.cpp:268-270);
// models are structurally valid random packed tensors (uniform code words and
// scale codes, super ~ U[0.001, 0.051), alpha/beta like synthetic.cpp:65-73).
//
//   ccq_gpu_bench [--shapes 4096x4096,4096x14336] [--m 1,4,16] [--bpw 2.06|2.5|2.75]
//                 [--iters 20] [--seed 1]
//
// `ccq_gpu_bench bench [...]` is the reference CLI's `ccq bench` itself
// (ccq_main.cpp:241-277, same options and defaults: --shapes
// 4096x4096,4096x1024,8192x8192,8192x1024 --m 1,4 --bpw 2.75 --group-size 64
// --iters 5 --seed 1 --out PATH): ccq::bench_model rows for every shape, the
// reference's three variants plus ccq_gpu_fused.  It is what acceptance
// criterion 10 drives through CCQ_BIN (tests/test_acceptance.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "ccq/cuda.hpp"
#include "ccq/kernels.hpp"

namespace {

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, c))
    if (!t.empty()) out.push_back(t);
  return out;
}

ccq::PackedModel random_model(std::int64_t rows, std::int64_t cols, ccq::Family fam, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> byte(0, 255);
  std::uniform_real_distribution<float> u01(0.f, 1.f);
  const std::int64_t groups = rows * (cols / 64);
  ccq::PackedModel m;
  m.rows = rows;
  m.cols = cols;
  m.family = fam;
  m.group_size = 64;
  m.super_scales.resize(std::size_t(rows));
  for (auto& v : m.super_scales) v = 0.001f + 0.05f * u01(rng);
  if (fam == ccq::Family::Bpw206) {
    m.code_payload.resize(std::size_t(groups) * 16);
    for (auto& b : m.code_payload) b = std::uint8_t(byte(rng));
    m.scale_payload.resize(std::size_t((groups + 1) / 2));
    for (auto& b : m.scale_payload) b = std::uint8_t(byte(rng));
    m.cluster_scales.resize(std::size_t(rows));
    m.cluster_zero_points.resize(std::size_t(rows));
    for (std::int64_t r = 0; r < rows; ++r) {
      const float a = 1.f + u01(rng) * (32767.f / 512.f);
      m.cluster_scales[r] = a;
      m.cluster_zero_points[r] = u01(rng) * (32767.f - 255.f * a);
    }
  } else {
    // tail word embeds the scale; random bytes everywhere is a valid stream
    const int pb = fam == ccq::Family::Bpw275 ? 22 : 20;
    m.code_payload.resize(std::size_t(groups) * pb);
    for (auto& b : m.code_payload) b = std::uint8_t(byte(rng));
  }
  return m;
}

template <class F>
double median_ms(int iters, F&& body) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> t;
  body();  // warm-up (upload, first launch)
  cudaDeviceSynchronize();
  for (int i = 0; i < iters; ++i) {
    cudaEventRecord(e0);
    body();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    t.push_back(ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

}  // namespace

// The reference CLI's bench subcommand on ccq::bench_model.
int cmd_bench(int argc, char** argv) {
  std::string shapes = "4096x4096,4096x1024,8192x8192,8192x1024", ms = "1,4", bpw = "2.75", out;
  int iters = 5, group_size = 64;
  std::uint64_t seed = 1;
  for (int i = 2; i < argc; i += 2) {
    const std::string k = argv[i];
    if (i + 1 >= argc) {
      std::fprintf(stderr, "option %s needs a value\n", k.c_str());
      return 2;
    }
    const std::string v = argv[i + 1];
    if (k == "--shapes") shapes = v;
    else if (k == "--m") ms = v;
    else if (k == "--bpw") bpw = v;
    else if (k == "--group-size") group_size = std::atoi(v.c_str());
    else if (k == "--iters") iters = std::atoi(v.c_str());
    else if (k == "--seed") seed = std::strtoull(v.c_str(), nullptr, 10);
    else if (k == "--out") out = v;
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  try {
    if (group_size != 64) throw ccq::ConfigError("ccq_gpu_bench models use group_size 64");
    const ccq::Family fam = ccq::family_from_name(bpw);
    std::vector<int> batches;
    for (const auto& b : split(ms, ',')) batches.push_back(std::atoi(b.c_str()));
    if (batches.empty()) throw ccq::ConfigError("no batch sizes given");
    std::vector<ccq::BenchRow> rows;
    for (const auto& sh : split(shapes, ',')) {
      const auto dims = split(sh, 'x');
      if (dims.size() != 2) throw ccq::ConfigError("shape must be AxB, got '" + sh + "'");
      const std::int64_t d_in = std::atoll(dims[0].c_str()), d_out = std::atoll(dims[1].c_str());
      if (d_in <= 0 || d_out <= 0) throw ccq::ConfigError("shape must be positive, got '" + sh + "'");
      const ccq::PackedModel model = random_model(d_out, d_in, fam, seed + std::uint64_t(d_in) * 31 + d_out);
      const auto r = ccq::bench_model(model, batches, iters, seed);
      rows.insert(rows.end(), r.begin(), r.end());
    }
    const std::string csv = ccq::bench_csv(rows);
    if (out.empty()) {
      std::fputs(csv.c_str(), stdout);
    } else {
      FILE* f = std::fopen(out.c_str(), "w");
      if (!f) throw ccq::Error("cannot open " + out + " for writing");
      std::fputs(csv.c_str(), f);
      std::fclose(f);
    }
  } catch (const ccq::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "bench") return cmd_bench(argc, argv);
  std::string shapes = "4096x4096", ms = "1,4,16", bpw = "2.06";
  int iters = 20;
  std::uint64_t seed = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--shapes") shapes = v;
    else if (k == "--m") ms = v;
    else if (k == "--bpw") bpw = v;
    else if (k == "--iters") iters = std::atoi(v.c_str());
    else if (k == "--seed") seed = std::strtoull(v.c_str(), nullptr, 10);
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  if (iters < 1) {
    std::fprintf(stderr, "iterations must be >= 1\n");  // ConfigError in the reference (kernels.cpp:230)
    return 2;
  }
  try {
    const ccq::Family fam = ccq::family_from_name(bpw);
    std::printf("shape,M,variant,median_ms,bytes_read\n");
    for (const auto& sh : split(shapes, ',')) {
      const auto dims = split(sh, 'x');
      if (dims.size() != 2) {
        std::fprintf(stderr, "bad shape %s\n", sh.c_str());
        return 2;
      }
      const std::int64_t d_in = std::atoll(dims[0].c_str()), d_out = std::atoll(dims[1].c_str());
      // the reference seeds each shape with seed + d_in*31 + d_out (ccq_main.cpp:269-271)
      const ccq::PackedModel model = random_model(d_out, d_in, fam, seed + std::uint64_t(d_in) * 31 + d_out);
      const std::uint64_t payload = ccq::model_payload_bytes(model);
      ccq::cuda::DeviceModel dm(model, 0);
      for (const auto& mstr : split(ms, ',')) {
        const std::int64_t M = std::atoll(mstr.c_str());
        if (M < 1) {
          std::fprintf(stderr, "batch must be >= 1\n");
          return 2;
        }
        std::vector<std::uint16_t> xb(std::size_t(M * d_in));
        std::mt19937_64 rng(seed + M);
        std::normal_distribution<float> g;
        ccq::Matrix x(M, d_in), y(M, d_out);
        for (std::size_t i = 0; i < xb.size(); ++i) {
          x.data[i] = g(rng);
          std::uint32_t u;
          std::memcpy(&u, &x.data[i], 4);
          xb[i] = std::uint16_t((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
        }
        void *dx = nullptr, *dy = nullptr;
        cudaMalloc(&dx, xb.size() * 2);
        cudaMalloc(&dy, std::size_t(M * d_out) * 4);
        cudaMemcpy(dx, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice);
        const double fused = median_ms(iters, [&] {
          dm.matmul(dx, ccq::cuda::DType::BF16, M, dy, ccq::cuda::DType::F32);
        });
        const double e2e = median_ms(iters, [&] { ccq::gemv_batch(model, x, y); });
        std::printf("%s,%lld,ccq_gpu_fused,%.6f,%llu\n", sh.c_str(), (long long)M, fused,
                    (unsigned long long)payload);
        std::printf("%s,%lld,ccq_gpu_fused_e2e,%.6f,%llu\n", sh.c_str(), (long long)M, e2e,
                    (unsigned long long)payload);
        cudaFree(dx);
        cudaFree(dy);
      }
    }
  } catch (const ccq::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
