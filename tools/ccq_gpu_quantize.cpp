// ccq_gpu_quantize - the reference CLI's `ccq quantize` step
// (tools/ccq_main.cpp, quantize_tensor + pack_model) on the GPU through the
// drop-in C++ API (ccq::cuda::quantize).  Reads a raw row-major f32 matrix,
// writes the packed sections as stored in a PackedModel, back to back:
//   code_payload | scale_payload | super_scales | cluster_scales | cluster_zero_points
//
//   ccq_gpu_quantize <in.f32> <rows> <cols> <2.75|2.5|2.06> <group_size> <rounds> <out.bin>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "ccq/cuda.hpp"

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: %s in.f32 rows cols family group_size rounds out.bin\n", argv[0]);
    return 2;
  }
  try {
    const std::int64_t rows = std::atoll(argv[2]), cols = std::atoll(argv[3]);
    ccq::Matrix w(rows, cols);
    std::ifstream in(argv[1], std::ios::binary);
    in.read(reinterpret_cast<char*>(w.data.data()), std::streamsize(w.data.size() * 4));
    if (!in) throw ccq::ShapeError("input file shorter than rows x cols floats");
    const ccq::PackedModel m =
        ccq::cuda::quantize(w, ccq::family_from_name(argv[4]), std::atoi(argv[5]), std::atoi(argv[6]));
    std::ofstream out(argv[7], std::ios::binary);
    auto put = [&](const void* p, std::size_t n) { out.write(static_cast<const char*>(p), std::streamsize(n)); };
    put(m.code_payload.data(), m.code_payload.size());
    put(m.scale_payload.data(), m.scale_payload.size());
    put(m.super_scales.data(), m.super_scales.size() * 4);
    put(m.cluster_scales.data(), m.cluster_scales.size() * 4);
    put(m.cluster_zero_points.data(), m.cluster_zero_points.size() * 4);
    std::printf("%zu %zu %zu %zu\n", m.code_payload.size(), m.scale_payload.size(), m.super_scales.size(),
                m.cluster_scales.size());
  } catch (const ccq::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
