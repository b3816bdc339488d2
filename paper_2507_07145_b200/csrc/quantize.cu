// Exhaustive trellis code search on the GPU - the inner step of the CCQ
// quantizer: ccq::search_codes (quantizer.cpp:36-103)
// for a batch of subvectors, bit-identical to the reference.
//
// For every subvector the reference walks all 2^(L + (valid-1)S) leaves of
// the code trellis (first window: L bits, every further window: S fresh
// bits), costs each leaf as  sum_j (x_j - (state_j - zp) * scale)^2  in
// double, added left to right, and keeps the first minimum in ascending code
// order.  Here one warp owns a subvector: its per-position cost tables
// (valid x 2^L doubles, the reference's `tables`) sit in shared memory, lanes
// take leaves lane, lane+32, ... (ascending, strict <), and a warp reduction
// picks the minimum cost, ties to the smaller code - the same answer as the
// sequential scan.  Products and sums are rounded separately
// (__dmul_rn/__dsub_rn/__dadd_rn): no FMA contraction, as in the reference's
// x86-64 build.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ccq_internal.hpp"

namespace ccqb {
namespace {

// Scan of this lane's leaves, ascending code order, strict <.  2.06 full
// words (L=6, S=3, 4 windows) take a nested walk with prefix sums, as the
// reference's depth-first descent: one add per leaf instead of three, and
// the inner two levels read the same table entry on every lane (their state
// depends only on fresh bits) - a broadcast.  The sums keep the reference's
// left-to-right order, so costs are bitwise the same.
__device__ __forceinline__ void leaf_scan(const double* t, int valid, int L, int S, int lane, double& best,
                                          uint32_t& bcode) {
  const int nst = 1 << L;
  if (L == 6 && S == 3 && valid == 4) {
    for (uint32_t s0 = lane; s0 < 64; s0 += 32) {
      const double a0 = t[s0];
      for (uint32_t f1 = 0; f1 < 8; ++f1) {
        const uint32_t s1 = ((s0 << 3) | f1) & 63u;
        const double a1 = __dadd_rn(a0, t[64 + s1]);
        for (uint32_t f2 = 0; f2 < 8; ++f2) {
          const uint32_t s2 = ((s1 << 3) | f2) & 63u;
          const double a2 = __dadd_rn(a1, t[128 + s2]);
#pragma unroll
          for (uint32_t f3 = 0; f3 < 8; ++f3) {
            const double c = __dadd_rn(a2, t[192 + (((s2 << 3) | f3) & 63u)]);
            if (c < best) {
              best = c;
              bcode = (s0 << 9) | (f1 << 6) | (f2 << 3) | f3;
            }
          }
        }
      }
    }
    return;
  }
  const uint32_t smask = uint32_t(nst - 1), fmask = (1u << S) - 1u;
  const uint32_t nleaf = 1u << (L + (valid - 1) * S);
  for (uint32_t leaf = lane; leaf < nleaf; leaf += 32) {
    uint32_t st = leaf >> ((valid - 1) * S);
    double acc = t[st];
    for (int j = 1; j < valid; ++j) {
      st = ((st << S) | ((leaf >> ((valid - 1 - j) * S)) & fmask)) & smask;
      acc = __dadd_rn(acc, t[j * nst + st]);
    }
    if (acc < best) {
      best = acc;
      bcode = leaf;
    }
  }
}

__global__ void __launch_bounds__(256) search_codes_kernel(const float* __restrict__ targets, int64_t n,
                                                           int valid, int stride, const double* __restrict__ scales,
                                                           int zp, int L, int N, int S,
                                                           uint32_t* __restrict__ codes) {
  extern __shared__ double tabs[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int nst = 1 << L;
  double* t = tabs + size_t(wib) * valid * nst;
  const uint32_t smask = uint32_t(nst - 1), fmask = (1u << S) - 1u;
  const int lbits = L + (valid - 1) * S;
  const uint32_t nleaf = 1u << lbits;
  for (int64_t i = int64_t(blockIdx.x) * wpb + wib; i < n; i += int64_t(gridDim.x) * wpb) {
    const double scale = scales[i];
    for (int e = lane; e < valid * nst; e += 32) {
      const int j = e / nst, s = e - j * nst;
      const double d = __dsub_rn(double(targets[i * stride + j]), __dmul_rn(double(s - zp), scale));
      t[e] = __dmul_rn(d, d);
    }
    __syncwarp();
    double best = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    uint32_t bcode = 0;
    leaf_scan(t, valid, L, S, lane, best, bcode);
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcode, off);
      if (ob < best || (ob == best && oc < bcode)) {
        best = ob;
        bcode = oc;
      }
    }
    if (lane == 0) codes[i] = bcode << ((N - valid) * S);
    __syncwarp();  // the table is rewritten for the next subvector
  }
}


// ---- the whole quantizer (quantize_tensor, quantizer.cpp:319-425) ----------

constexpr int kQWarps = 8;    // warps (groups in flight) per CTA
constexpr int kQMaxGS = 256;  // largest group size the GPU quantizer takes

// Family scheme (coding.cpp:24-27, 213-249): code parts, word layout.
struct QScheme {
  int nparts, L[2], N[2], S[2];
  int code_bits, wpw, zp, sb, gs, full_words, has_tail, words;
  uint32_t wmask;
  int shifts[8];
};

// search_codes for one subvector, the whole warp cooperating (see
// search_codes_kernel); tab holds valid x 2^L doubles.  All lanes return the code.
__device__ uint32_t warp_search(const float* tgt, int valid, double scale, int zp, int L, int N, int S,
                                double* tab) {
  const int lane = threadIdx.x & 31, nst = 1 << L;
  __syncwarp();
  for (int e = lane; e < valid * nst; e += 32) {
    const int j = e / nst, st = e - j * nst;
    const double d = __dsub_rn(double(tgt[j]), __dmul_rn(double(st - zp), scale));
    tab[e] = __dmul_rn(d, d);
  }
  __syncwarp();
  double best = __longlong_as_double(0x7FF0000000000000LL);
  uint32_t bcode = 0;
  leaf_scan(tab, valid, L, S, lane, best, bcode);
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcode, off);
    if (ob < best || (ob == best && oc < bcode)) {
      best = ob;
      bcode = oc;
    }
  }
  __syncwarp();
  return bcode << ((N - valid) * S);
}

// search_group (quantizer.cpp:157-170) -> words[], then the decoded states
// (decode_group_states, quantizer.cpp:120-133) and group_error (172-180;
// sequential sum on lane 0).  Returns the error on every lane.
__device__ double search_and_score(const QScheme& q, const float* g, double scale, uint16_t* words, int* st,
                                   double* tab) {
  const int lane = threadIdx.x & 31;
  for (int w = 0; w < q.words; ++w) {
    const bool tail = w == q.full_words;
    const float* tg = tail ? g + q.gs - 1 : g + w * q.wpw;
    const int len = tail ? 1 : q.wpw;
    uint32_t word = 0;
    int bits_left = q.code_bits, offset = 0;
    for (int p = 0; p < q.nparts; ++p) {
      bits_left -= q.L[p] + (q.N[p] - 1) * q.S[p];
      const int take = q.N[p] < len - offset ? q.N[p] : len - offset;
      const uint32_t code = warp_search(tg + offset, take, scale, q.zp, q.L[p], q.N[p], q.S[p], tab);
      word |= code << bits_left;
      offset += take;
      if (offset == len) break;
    }
    if (lane == 0) words[w] = uint16_t(word);
  }
  __syncwarp();
  for (int i = lane; i < q.gs; i += 32) st[i] = int((words[i / q.wpw] >> q.shifts[i % q.wpw]) & q.wmask);
  __syncwarp();
  double err = 0.0;
  if (lane == 0)
    for (int i = 0; i < q.gs; ++i) {
      const double d = __dsub_rn(double(g[i]), __dmul_rn(double(st[i] - q.zp), scale));
      err = __dadd_rn(err, __dmul_rn(d, d));
    }
  return __shfl_sync(0xffffffffu, err, 0);
}

__device__ double group_err(const QScheme& q, const float* g, const int* st, double scale) {
  double err = 0.0;
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < q.gs; ++i) {
      const double d = __dsub_rn(double(g[i]), __dmul_rn(double(st[i] - q.zp), scale));
      err = __dadd_rn(err, __dmul_rn(d, d));
    }
  return __shfl_sync(0xffffffffu, err, 0);
}

// quantize_group (quantizer.cpp:183-222) for every group: one warp per group.
// Outputs the best code words and the raw (pre-snapping) scale as float.
__global__ void __launch_bounds__(kQWarps * 32) quantize_groups(const float* __restrict__ W, int64_t rows,
                                                               int64_t cols, QScheme q, int rounds,
                                                               uint16_t* __restrict__ words_out,
                                                               float* __restrict__ scale_out) {
  __shared__ float gsh[kQWarps][kQMaxGS];
  __shared__ int stsh[kQWarps][kQMaxGS];
  __shared__ uint16_t cur[kQWarps][kQMaxGS / 3 + 2], best_w[kQWarps][kQMaxGS / 3 + 2];
  __shared__ double tab[kQWarps][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gpr = cols / q.gs, groups = rows * gpr;
  float* g = gsh[wib];
  int* st = stsh[wib];
  for (int64_t gi = int64_t(blockIdx.x) * kQWarps + wib; gi < groups; gi += int64_t(gridDim.x) * kQWarps) {
    const float* src = W + (gi / gpr) * cols + (gi % gpr) * q.gs;
    double mx = 0.0;
    for (int i = lane; i < q.gs; i += 32) {
      g[i] = src[i];
      mx = fmax(mx, fabs(double(g[i])));  // init_group_scale (quantizer.cpp:29-34); NaN ignored like std::max
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    __syncwarp();
    double scale = __ddiv_rn(mx, double((1 << (q.sb - 1)) - 1));
    double err = search_and_score(q, g, scale, cur[wib], st, tab[wib]);
    double bscale = scale, berr = err;
    for (int w = lane; w < q.words; w += 32) best_w[wib][w] = cur[wib][w];
    for (int round = 1; round <= rounds; ++round) {
      // optimize_scale (quantizer.cpp:105-118) on the current states, lane 0
      double ns = 0.0;
      if (lane == 0) {
        double num = 0.0, den = 0.0;
        for (int i = 0; i < q.gs; ++i) {
          const double c = double(st[i] - q.zp);
          num = __dadd_rn(num, __dmul_rn(double(g[i]), c));
          den = __dadd_rn(den, __dmul_rn(c, c));
        }
        ns = den == 0.0 ? scale : __ddiv_rn(num, den);
      }
      ns = __shfl_sync(0xffffffffu, ns, 0);
      scale = 0.0 < ns ? ns : 0.0;  // std::max(0.0, x)
      err = group_err(q, g, st, scale);
      if (err < berr) {
        __syncwarp();
        for (int w = lane; w < q.words; w += 32) best_w[wib][w] = cur[wib][w];
        bscale = scale;
        berr = err;
      }
      if (round < rounds) {
        err = search_and_score(q, g, scale, cur[wib], st, tab[wib]);
        if (err < berr) {
          __syncwarp();
          for (int w = lane; w < q.words; w += 32) best_w[wib][w] = cur[wib][w];
          bscale = scale;
          berr = err;
        }
      }
    }
    __syncwarp();
    for (int w = lane; w < q.words; w += 32) words_out[gi * q.words + w] = best_w[wib][w];
    if (lane == 0) scale_out[gi] = float(bscale);
    __syncwarp();
  }
}

// 2.06 cluster-aware re-search (quantizer.cpp:392-409, search_cluster_table
// 272-291): one thread per subvector, the row's 256-entry table.
__global__ void cluster_research(const float* __restrict__ W, int64_t rows, int64_t cols, QScheme q,
                                 const float* __restrict__ group_scales, const uint8_t* __restrict__ tstates,
                                 const uint16_t* __restrict__ tcodes, uint8_t* __restrict__ clustered,
                                 uint16_t* __restrict__ words) {
  const int64_t gpr = cols / q.gs, n = rows * gpr * q.words;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gi = i / q.words, r = gi / gpr;
    const int w = int(i - gi * q.words);
    const bool tail = q.has_tail && w == q.full_words;
    const float* g = W + r * cols + (gi % gpr) * q.gs;
    const float* t = tail ? g + q.gs - 1 : g + w * q.wpw;
    const int valid = tail ? 1 : q.wpw;
    const double scale = double(group_scales[gi]);
    const uint8_t* ts = tstates + r * 256 * 8;
    double best = __longlong_as_double(0x7FF0000000000000LL);
    int bq = 0;
    for (int c = 0; c < 256; ++c) {
      double cost = 0.0;
      for (int j = 0; j < valid; ++j) {
        const double d = __dsub_rn(double(t[j]), __dmul_rn(double(int(ts[c * 8 + j]) - q.zp), scale));
        cost = __dadd_rn(cost, __dmul_rn(d, d));
      }
      if (cost < best) {
        best = cost;
        bq = c;
      }
    }
    clustered[i] = uint8_t(bq);
    words[i] = tcodes[r * 256 + bq];
  }
}


// quantize_scales (packing.cpp:142-158), one warp per row: super scale, the
// snapped scale codes and group_scales = float(code) * super.  A negative or
// NaN raw scale flags the row (the reference's DomainError).
__global__ void snap_scales(const float* __restrict__ raw, int64_t rows, int64_t gpr, uint32_t levels,
                            float* __restrict__ super, uint16_t* __restrict__ scode, float* __restrict__ gscale,
                            unsigned long long* __restrict__ bad_row) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const float* rs = raw + r * gpr;
    float mx = 0.0f;
    bool bad = false;
    for (int64_t j = lane; j < gpr; j += 32) {
      const float v = rs[j];
      bad |= v < 0.0f || isnan(v);
      mx = fmaxf(mx, v);  // max of non-negative floats: order-free
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicMin(bad_row, (unsigned long long)r);
      continue;
    }
    const float sup = mx == 0.0f ? 1.0f : float(__ddiv_rn(double(mx), double(levels)));
    if (lane == 0) super[r] = sup;
    for (int64_t j = lane; j < gpr; j += 32) {
      long c = lround(__ddiv_rn(double(rs[j]), double(sup)));
      c = c < 0 ? 0 : (c > long(levels) ? long(levels) : c);
      scode[r * gpr + j] = uint16_t(c);
      gscale[r * gpr + j] = __fmul_rn(float(c), sup);
    }
  }
}

// cluster_channel + build_cluster_table (quantizer.cpp:224-270), one warp per
// row: code range -> (code_scale, code_zero_point), the 256 widened codes and
// their states; a code outside [0, 2^code_bits) flags (row, q).
__global__ void cluster_tables(const uint16_t* __restrict__ words, int64_t rows, int64_t wpr, QScheme q,
                               float* __restrict__ cscale, float* __restrict__ czp, uint8_t* __restrict__ tstates,
                               uint16_t* __restrict__ tcodes, unsigned long long* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t lo = 0xFFFFu, hi = 0u;
    for (int64_t i = lane; i < wpr; i += 32) {
      const uint32_t v = words[r * wpr + i];
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    const float zp = float(lo);
    const float cs = hi == lo ? 1.0f : float(__ddiv_rn(double(hi) - double(lo), 255.0));
    if (lane == 0) {
      cscale[r] = cs;
      czp[r] = zp;
    }
    for (int c = lane; c < 256; c += 32) {
      const long v = lround(__dadd_rn(__dmul_rn(double(c), double(cs)), double(zp)));
      if (v < 0 || v >= (1l << q.code_bits)) {
        atomicMin(bad, (unsigned long long)(r * 256 + c));
        continue;
      }
      tcodes[r * 256 + c] = uint16_t(v);
      for (int j = 0; j < q.wpw; ++j) tstates[(r * 256 + c) * 8 + j] = uint8_t((uint32_t(v) >> q.shifts[j]) & q.wmask);
    }
  }
}

// pack_model's payload (container.cpp:323-358, pack_group packing.cpp:71-114):
// one thread per group; words little-endian, the tail word of embedded-scale
// families carries the scale code.  Side-band nibbles: one thread per byte.
__global__ void pack_groups(const uint16_t* __restrict__ words, const uint8_t* __restrict__ clustered,
                            const uint16_t* __restrict__ scode, int64_t groups, QScheme q, int word_bytes,
                            int embedded, uint8_t* __restrict__ payload, uint8_t* __restrict__ nibbles) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t gi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; gi < groups; gi += stride) {
    uint8_t* out = payload + gi * q.words * word_bytes;
    for (int w = 0; w < q.words; ++w) {
      uint32_t v = clustered ? clustered[gi * q.words + w] : words[gi * q.words + w];
      if (q.has_tail && w == q.full_words && !clustered) v |= scode[gi];
      out[w * word_bytes] = uint8_t(v & 0xFF);
      if (word_bytes == 2) out[w * word_bytes + 1] = uint8_t(v >> 8);
    }
  }
  if (!embedded)
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < (groups + 1) / 2; b += stride) {
      uint32_t v = scode[2 * b] & 0xFu;
      if (2 * b + 1 < groups) v |= (scode[2 * b + 1] & 0xFu) << 4;
      nibbles[b] = uint8_t(v);
    }
}

}  // namespace
}  // namespace ccqb

using namespace ccqb;

extern "C" int ccq_cuda_search_codes(const float* targets, int64_t n, int32_t valid, int32_t stride,
                                     const double* scales, int32_t zero_point, int32_t state_bits,
                                     int32_t states_per_code, int32_t transition_bits, uint32_t* codes,
                                     void* stream) {
  // EncodingConfig::validate (coding.cpp:38-57) and search_codes' shape check
  const int L = state_bits, N = states_per_code, S = transition_bits;
  if (N < 1 || S < 1 || S > L || L > 8 || L + (N - 1) * S > 16)
    return fail(CCQ_ERR_CONFIG, "encoding config needs 1 <= S <= L <= 8, N >= 1 and L + (N-1)S <= 16");
  if (valid < 1 || valid > N)
    return fail(CCQ_ERR_SHAPE, "search target must hold 1.." + std::to_string(N) + " values, got " +
                                   std::to_string(valid));
  if (n < 0 || stride < valid) return fail(CCQ_ERR_SHAPE, "bad subvector count or stride");
  if (n == 0) return CCQ_OK;
  if (!targets || !scales || !codes) return fail(CCQ_ERR_INVALID, "null pointer");
  const size_t per_warp = size_t(valid) * size_t(1 << L) * sizeof(double);  // <= 16 x 256 x 8 B
  const int wpb = int(std::min<size_t>(8, (200 * 1024) / per_warp));
  const size_t smem = size_t(wpb) * per_warp;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t blocks = std::min<int64_t>((n + wpb - 1) / wpb, int64_t(num_sms(dev)) * 16);
  if (smem > 48 * 1024)
    if (int st = ensure_smem(reinterpret_cast<const void*>(search_codes_kernel), smem)) return st;
  search_codes_kernel<<<unsigned(blocks), wpb * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      targets, n, valid, stride, scales, zero_point, L, N, S, codes);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "search_codes launch");
}

// ---- quantize_tensor + pack_model on the GPU (host driver) -----------------
// Everything runs on the device, one stream-ordered chain and one sync: the
// per-group search and refinement (quantize_groups), scale snapping
// (snap_scales), the 2.06 code clusters and tables (cluster_tables) and
// cluster-aware re-search (cluster_research), and byte packing (pack_groups).
namespace ccqb {
namespace {

struct QuantRun {
  uint8_t* ws = nullptr;  // device workspace; the packed sections live in it
  size_t oPay = 0, oNib = 0, oSup = 0, oCs = 0, oCz = 0;
  size_t pay = 0, nib = 0;
  Geometry geo;
  FamilyConst fc;
};

// Validates like quantize_tensor, runs the device chain; on CCQ_OK the
// sections are in r.ws (caller frees).  w is host or device memory.
int run_quantizer(const float* w, int64_t rows, int64_t cols, int32_t family, int32_t group_size, int32_t rounds,
                  int32_t device, QuantRun& r) {
  int st = geometry_for(family, group_size, &r.geo);  // ConfigError as group_geometry
  if (st != CCQ_OK) return st;
  if (rounds < 0) return fail(CCQ_ERR_CONFIG, "refinement rounds must be >= 0");
  if (rows < 0 || cols < 0) return fail(CCQ_ERR_SHAPE, "negative shape");
  if (cols % group_size != 0)
    return fail(CCQ_ERR_SHAPE, "input dimension " + std::to_string(cols) + " is not a multiple of group size " +
                                   std::to_string(group_size));
  if (group_size > kQMaxGS) return fail(CCQ_ERR_CONFIG, "the GPU quantizer takes group sizes up to 256");
  const Geometry& geo = r.geo;
  const FamilyConst fc = family_const(family);
  r.fc = fc;
  QScheme q{};
  if (family == kF275) {
    q.nparts = 1; q.L[0] = 4; q.N[0] = 3; q.S[0] = 2;
  } else if (family == kF25) {
    q.nparts = 2; q.L[0] = 3; q.N[0] = 3; q.S[0] = 2; q.L[1] = 3; q.N[1] = 4; q.S[1] = 2;
  } else {
    q.nparts = 1; q.L[0] = 6; q.N[0] = 4; q.S[0] = 3;
  }
  q.code_bits = fc.code_bits; q.wpw = fc.wpw; q.zp = fc.zero_point; q.sb = fc.state_bits; q.gs = group_size;
  q.full_words = geo.full_words; q.has_tail = geo.has_tail; q.words = geo.words_per_group; q.wmask = fc.weight_mask;
  for (int i = 0; i < 8; ++i) q.shifts[i] = i < 7 ? fc.shifts[i] : 0;
  const int64_t gpr = cols / group_size, groups = rows * gpr, nw = groups * q.words;
  if (!w && groups) return fail(CCQ_ERR_INVALID, "null weights");

  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  // device workspace (one allocation): W | words | raw | scode | gscale |
  // super | cs | czp | tables | clustered | payload | nibbles | flags
  const uint32_t levels = (1u << fc.scale_bits) - 1u;
  r.pay = size_t(groups) * size_t(geo.payload_bytes);
  r.nib = geo.embedded_scale ? 0 : size_t((groups + 1) / 2);
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = (off + bytes + 255) & ~size_t(255); return o; };
  const size_t oW = take(size_t(rows * cols) * 4), oWd = take(size_t(nw) * 2), oRaw = take(size_t(groups) * 4);
  const size_t oSc = take(size_t(groups) * 2), oGs = take(size_t(groups) * 4);
  r.oSup = take(size_t(rows) * 4);
  r.oCs = take(fc.cluster ? size_t(rows) * 4 : 0);
  r.oCz = take(fc.cluster ? size_t(rows) * 4 : 0);
  const size_t oTs = take(fc.cluster ? size_t(rows) * 256 * 8 : 0), oTc = take(fc.cluster ? size_t(rows) * 256 * 2 : 0);
  const size_t oCl = take(fc.cluster ? size_t(nw) : 0);
  r.oPay = take(r.pay);
  r.oNib = take(r.nib);
  const size_t oFlag = take(16);
  uint8_t* ws = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&ws, off);
  r.ws = ws;
  auto P8 = [&](size_t o) { return ws + o; };
  unsigned long long flags[2] = {~0ull, ~0ull};  // [0] bad scale row, [1] bad cluster (row * 256 + q)
  if (e == cudaSuccess && groups) e = cudaMemcpy(P8(oW), w, size_t(rows * cols) * 4, cudaMemcpyDefault);
  if (e == cudaSuccess) e = cudaMemcpy(P8(oFlag), flags, sizeof(flags), cudaMemcpyHostToDevice);
  const float* dW = reinterpret_cast<const float*>(P8(oW));
  uint16_t* dwords = reinterpret_cast<uint16_t*>(P8(oWd));
  uint16_t* dscode = reinterpret_cast<uint16_t*>(P8(oSc));
  float* dgs = reinterpret_cast<float*>(P8(oGs));
  unsigned long long* dflag = reinterpret_cast<unsigned long long*>(P8(oFlag));
  const int sms = num_sms(device);
  if (e == cudaSuccess && groups == 0) {  // no groups: super scales are 1 (quantize_scales of nothing)
    std::vector<float> ones(size_t(rows), 1.0f);
    if (rows) e = cudaMemcpy(P8(r.oSup), ones.data(), size_t(rows) * 4, cudaMemcpyHostToDevice);
  } else if (e == cudaSuccess) {
    const int64_t blocks = std::min<int64_t>((groups + kQWarps - 1) / kQWarps, int64_t(sms) * 8);
    quantize_groups<<<unsigned(blocks), kQWarps * 32>>>(dW, rows, cols, q, rounds, dwords,
                                                       reinterpret_cast<float*>(P8(oRaw)));
    const unsigned rb = unsigned(std::min<int64_t>((rows + 7) / 8, int64_t(sms) * 16));
    snap_scales<<<rb, 256>>>(reinterpret_cast<const float*>(P8(oRaw)), rows, gpr, levels,
                             reinterpret_cast<float*>(P8(r.oSup)), dscode, dgs, dflag);
    count_launch(2);
    if (fc.cluster) {
      cluster_tables<<<rb, 256>>>(dwords, rows, gpr * q.words, q, reinterpret_cast<float*>(P8(r.oCs)),
                                  reinterpret_cast<float*>(P8(r.oCz)), P8(oTs), reinterpret_cast<uint16_t*>(P8(oTc)),
                                  dflag + 1);
      const int64_t cb = std::min<int64_t>((nw + 255) / 256, int64_t(sms) * 16);
      cluster_research<<<unsigned(cb), 256>>>(dW, rows, cols, q, dgs, P8(oTs), reinterpret_cast<uint16_t*>(P8(oTc)),
                                              P8(oCl), dwords);
      count_launch(2);
    }
    const int64_t pb = std::min<int64_t>((groups + 255) / 256, int64_t(sms) * 16);
    pack_groups<<<unsigned(pb), 256>>>(dwords, fc.cluster ? P8(oCl) : nullptr, dscode, groups, q, fc.word_bytes,
                                       geo.embedded_scale, P8(r.oPay), P8(r.oNib));
    count_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(flags, P8(oFlag), sizeof(flags), cudaMemcpyDeviceToHost);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaFree(ws);
    r.ws = nullptr;
    return cuda_fail(e, "gpu quantizer");
  }
  // errors in row order: a row's scales are snapped before it is clustered
  int bad = CCQ_OK;
  if (flags[0] != ~0ull && (flags[1] == ~0ull || flags[0] <= flags[1] / 256))
    bad = fail(CCQ_ERR_DOMAIN, "group scales must be non-negative");
  else if (flags[1] != ~0ull)
    bad = fail(CCQ_ERR_DOMAIN, "clustered code reconstructs outside [0, 2^" + std::to_string(fc.code_bits) +
                                   "): q=" + std::to_string(int(flags[1] % 256)));
  if (bad != CCQ_OK) {
    cudaFree(ws);
    r.ws = nullptr;
  }
  return bad;
}

}  // namespace
}  // namespace ccqb

extern "C" int ccq_quantize_host(const float* w, int64_t rows, int64_t cols, int32_t family, int32_t group_size,
                                 int32_t rounds, int32_t device, uint8_t* code_payload, uint8_t* scale_payload,
                                 float* super_scales, float* cluster_scales, float* cluster_zero_points) {
  Geometry g0;
  if (geometry_for(family, group_size, &g0) == CCQ_OK) {  // output pointer checks before any work
    const bool cl = family_const(family).cluster;
    if ((rows && !super_scales) || (!g0.embedded_scale && rows && cols && !scale_payload) ||
        (rows && cols && !code_payload) || (cl && rows && (!cluster_scales || !cluster_zero_points)))
      return fail(CCQ_ERR_INVALID, "null output section");
  }
  QuantRun r;
  const int st = run_quantizer(w, rows, cols, family, group_size, rounds, device, r);
  if (st != CCQ_OK) return st;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaSuccess;
  if (r.pay) e = cudaMemcpy(code_payload, r.ws + r.oPay, r.pay, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && r.nib) e = cudaMemcpy(scale_payload, r.ws + r.oNib, r.nib, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && rows) e = cudaMemcpy(super_scales, r.ws + r.oSup, size_t(rows) * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && r.fc.cluster && rows) {
    e = cudaMemcpy(cluster_scales, r.ws + r.oCs, size_t(rows) * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(cluster_zero_points, r.ws + r.oCz, size_t(rows) * 4, cudaMemcpyDeviceToHost);
  }
  cudaFree(r.ws);
  cudaSetDevice(prev);
  return e == cudaSuccess ? CCQ_OK : cuda_fail(e, "gpu quantizer copy-out");
}

// Quantize weights already in HBM and upload the result as a device model,
// with no host round trip: the packed sections go from the quantizer's
// workspace straight into the device re-layout (ccq_cuda_model_upload takes
// device-resident views).
extern "C" int ccq_cuda_quantize_model(const float* w, int64_t rows, int64_t cols, int32_t family,
                                       int32_t group_size, int32_t rounds, int32_t device, ccq_dev_model** out) {
  if (!out) return fail(CCQ_ERR_INVALID, "null output handle");
  *out = nullptr;
  QuantRun r;
  const int st = run_quantizer(w, rows, cols, family, group_size, rounds, device, r);
  if (st != CCQ_OK) return st;
  ccq_packed_view v{};
  v.rows = rows;
  v.cols = cols;
  v.family = family;
  v.group_size = group_size;
  v.rounds = rounds;
  v.code_payload = r.ws + r.oPay;
  v.code_bytes = r.pay;
  v.scale_payload = r.nib ? r.ws + r.oNib : nullptr;
  v.scale_bytes = r.nib;
  v.super_scales = reinterpret_cast<const float*>(r.ws + r.oSup);
  v.n_super_scales = uint64_t(rows);
  if (r.fc.cluster) {
    v.cluster_scales = reinterpret_cast<const float*>(r.ws + r.oCs);
    v.n_cluster_scales = uint64_t(rows);
    v.cluster_zero_points = reinterpret_cast<const float*>(r.ws + r.oCz);
    v.n_cluster_zero_points = uint64_t(rows);
  }
  const int up = ccq_cuda_model_upload(&v, device, out);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaFree(r.ws);
  cudaSetDevice(prev);
  return up;
}
