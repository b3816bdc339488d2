#include <mutex>
// Packed-weight upload, per-row widening plans and the synchronous
// host-buffer entry points of the C ABI (include/ccq_cuda.h).
//
// Reference counterparts:
//   model_from_bytes validation       container.cpp:261-319
//   clustered_code_value              coding.hpp:142-150
//   dequantize / gemv / gemv_batch    kernels.cpp:103-187 (signatures kernels.hpp:36-43)
//   model_payload_bytes               kernels.cpp:203-207
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cstdlib>

#include "ccq_internal.hpp"

namespace ccqb {

namespace {
thread_local std::string g_err;
}

std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")";
  return CCQ_ERR_CUDA;
}

int geometry_for(int family, int group_size, Geometry* g) {
  if (family < 0 || family > 2) return fail(CCQ_ERR_CONFIG, "unknown family");
  const FamilyConst fc = family_const(family);
  if (group_size <= 0) return fail(CCQ_ERR_CONFIG, "group_size must be positive");
  const int rem = group_size % fc.wpw;
  if (rem > 1) {
    return fail(CCQ_ERR_CONFIG, "group_size " + std::to_string(group_size) + " leaves " +
                                    std::to_string(rem) +
                                    " weights in the last word; only remainders 0 and 1 have "
                                    "a layout");
  }
  if (family == kF25 && rem == 0)
    return fail(CCQ_ERR_CONFIG, "family 2.5 requires group_size % 7 == 1");
  g->group_size = group_size;
  g->full_words = group_size / fc.wpw;
  g->has_tail = rem == 1;
  g->words_per_group = g->full_words + g->has_tail;
  g->embedded_scale = g->has_tail && !fc.cluster;
  g->payload_bytes = g->words_per_group * fc.word_bytes;
  return CCQ_OK;
}

namespace {

// Reference widening (coding.hpp:144): lround(q * alpha + beta) in double,
// multiply and add rounded separately (no FMA contraction on the device).
__host__ __device__ inline long ref_widen(int q, float a, float b) {
#ifdef __CUDA_ARCH__
  return lround(__dadd_rn(__dmul_rn(double(q), double(a)), double(b)));
#else
  return std::lround(double(q) * double(a) + double(b));
#endif
}

// Builds the exact fixed-point plan of one row and marks (bit q of inv[8]) the
// q values the reference would reject (result outside [0, 2^15)).  Returns
// false if no plan reproduces the reference for every valid q.  Runs on the
// device at upload (one thread per row) and on the host (same candidates in
// the same order, so both pick the same plan).
__host__ __device__ bool build_widen_plan(float alpha, float beta, WidenPlan* out, uint32_t inv[8]) {
  bool all_invalid = true;
  for (int i = 0; i < 8; ++i) inv[i] = 0u;
  for (int q = 0; q < 256; ++q) {
    const long ref = ref_widen(q, alpha, beta);
    if (ref < 0 || ref >= 32768) inv[q >> 5] |= 1u << (q & 31);
    else all_invalid = false;
  }
  if (!isfinite(alpha) || !isfinite(beta)) {
    if (all_invalid) {
      *out = WidenPlan{0, 0, plan_sel(0)};
      return true;
    }
    return false;
  }
  // C = floor((beta + 1/2) * 2^40).  beta*2^40 is exact in double; floor is
  // exact below 2^53 and a no-op above.
  const int64_t C0 = int64_t(floor(ldexp(double(beta), 40))) + (int64_t(1) << 39);
  auto verify = [&](uint32_t M, uint32_t pos, int64_t C) {
    const WidenPlan p{uint64_t(C), M, plan_sel(pos)};
    for (int q = 0; q < 256; ++q) {
      if ((inv[q >> 5] >> (q & 31)) & 1u) continue;
      const uint32_t hi = widen_hi(uint32_t(q), p);
      if (long(hi >> 8) != ref_widen(q, alpha, beta) || hi >= (1u << 23)) return false;
    }
    *out = p;
    return true;
  };
  // Exact M: alpha * 2^(40 - 8*pos) integral and below 2^32; then rounded M
  // (tiny or huge alpha), still verified exhaustively.
  uint32_t cm[8], cp[8];
  int nc = 0;
  const uint32_t exact_order[4] = {2u, 1u, 3u, 0u};
  for (int i = 0; i < 4; ++i) {
    const double Md = ldexp(double(alpha), 40 - 8 * int(exact_order[i]));
    if (Md >= 0.0 && Md < 4294967296.0 && Md == floor(Md)) {
      cm[nc] = uint32_t(Md);
      cp[nc++] = exact_order[i];
    }
  }
  for (uint32_t pos = 0; pos < 4; ++pos) {
    const double Md = ldexp(double(alpha), 40 - 8 * int(pos));
    if (Md >= 0.0 && Md < 4294967295.5) {
      cm[nc] = uint32_t(llround(Md));
      cp[nc++] = pos;
    }
  }
  const int64_t nudges[13] = {0,       1,        -1,        256,        -256,
                              65536,   -65536,   1 << 24,   -(1 << 24), int64_t(1) << 30,
                              -(int64_t(1) << 30), int64_t(1) << 34, -(int64_t(1) << 34)};
  for (int i = 0; i < nc; ++i)
    for (int k = 0; k < 13; ++k)
      if (verify(cm[i], cp[i], C0 + nudges[k])) return true;
  return false;
}

// One thread per row of the device model (padding rows get the inert plan):
// plans, invalid-q masks, the first row without a plan and the smallest byte
// position any plan uses.
// FP64-pipe widening plan of one row (gemv.cu dot_206_w64): code =
// low word of add.rm(fma.rm(v, A, B), 2^52) with v = 1 + q 2^-12 (the byte
// placed in the high word of a double by one PRMT), A = 4096 alpha (exact),
// B = (beta + 1/2) - A.  Whenever q alpha + beta is exact in double this is
// floor(q alpha + beta + 1/2) = lround(q alpha + beta); it is verified here
// with the very instructions the kernel runs, for every valid q.
__device__ bool build_plan64(float alpha, float beta, const uint32_t inv[8], double2* out) {
  const double A = 4096.0 * double(alpha);
  const double B = __dsub_rn(__dadd_rn(double(beta), 0.5), A);
  *out = make_double2(A, B);
  if (!isfinite(A) || !isfinite(B)) return false;
  for (int q = 0; q < 256; ++q) {
    if ((inv[q >> 5] >> (q & 31)) & 1u) continue;
    const double v = __hiloint2double(int(0x3FF00000u | (uint32_t(q) << 8)), 0);
    const double t = __fma_rd(v, A, B);
    const double d = __dadd_rd(t, 4503599627370496.0);  // 2^52
    if (long(uint32_t(__double2loint(d))) != ref_widen(q, alpha, beta) || t < 0.0) return false;
  }
  return true;
}

__global__ void build_plans(const float* __restrict__ alpha, const float* __restrict__ beta, int64_t rows,
                            int64_t rp, WidenPlan* __restrict__ plans, uint32_t* __restrict__ invalid,
                            unsigned long long* __restrict__ fail_row, unsigned int* __restrict__ pos_min,
                            double2* __restrict__ plan64, unsigned int* __restrict__ w64_fail) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rp) return;
  if (r >= rows) {
    plans[r] = WidenPlan{0, 0, plan_sel(0)};
    if (plan64) plan64[r] = make_double2(0.0, 0.0);
    return;
  }
  WidenPlan p;
  uint32_t inv[8];
  const bool ok = build_widen_plan(alpha[r], beta[r], &p, inv);
  if (plan64) {  // only when the FP64-widening GEMV is enabled (CCQ_W64=1)
    double2 p64;
    if (!ok || !build_plan64(alpha[r], beta[r], inv, &p64)) {
      atomicExch(w64_fail, 1u);
      p64 = make_double2(0.0, 0.0);
    }
    plan64[r] = p64;
  }
  if (ok) {
    plans[r] = p;
    atomicMin(pos_min, plan_pos(p));
  } else {
    plans[r] = WidenPlan{0, 0, plan_sel(0)};
    atomicMin(fail_row, (unsigned long long)r);
  }
  for (int i = 0; i < 8; ++i) invalid[r * 8 + i] = inv[i];
}

size_t align_up(size_t n, size_t a) { return (n + a - 1) / a * a; }

// Device-side loader: the packed sections, copied to the
// device as they are in the file, are scattered into the chunk-major record
// layout (ccq_internal.hpp) here - one warp per (chunk, row) record - instead
// of a host-side re-layout pass.  2.06 rows also get their widening plan and
// every stored byte is checked against the row's invalid-q mask (the
// reference's DomainError, coding.hpp:145-148); the first offending byte in
// file order wins (atomicMin on its row-major byte offset).
__global__ void __launch_bounds__(256) relayout_records(
    const uint8_t* __restrict__ codes, uint64_t row_bytes, const uint8_t* __restrict__ nib, uint64_t nib_g0,
    const WidenPlan* __restrict__ plans, const uint32_t* __restrict__ invalid, int64_t rows, int64_t rp, int64_t gpr,
    int payload, uint32_t rec, uint32_t cgb, int nch, uint8_t* __restrict__ dst, unsigned long long* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nrec = int64_t(nch) * rp;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nrec;
       w += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int c = int(w / rp);
    const int64_t r = w - int64_t(c) * rp;
    uint8_t* d = dst + uint64_t(w) * rec;
    if (r < rows) {
      const int64_t g0 = int64_t(c) * kChunk;
      const int ng = int(gpr - g0 < kChunk ? gpr - g0 : kChunk);
      const uint64_t so = uint64_t(r) * row_bytes + uint64_t(g0) * payload;
      const int nbytes = ng * payload;
      const uint32_t* inv = invalid ? invalid + r * 8 : nullptr;
      for (int i = lane; i < nbytes; i += 32) {
        const uint8_t q = codes[so + i];
        d[i] = q;
        if (inv && ((inv[q >> 5] >> (q & 31)) & 1u)) atomicMin(bad, (unsigned long long)(so + i));
      }
      if (nib) {
        for (int j = 2 * lane; j < ng; j += 64) {
          const uint64_t gi = nib_g0 + uint64_t(r) * gpr + g0 + j;
          uint32_t b = (nib[gi >> 1] >> (4 * (gi & 1))) & 0xFu;
          if (j + 1 < ng) b |= ((nib[(gi + 1) >> 1] >> (4 * ((gi + 1) & 1))) & 0xFu) << 4;
          d[cgb + j / 2] = uint8_t(b);
        }
      }
    }
    if (plans && lane < 4) {  // padding rows carry the inert plan
      const WidenPlan p = r < rows ? plans[r] : WidenPlan{0, 0, plan_sel(0)};
      reinterpret_cast<uint32_t*>(d + cgb + (nib ? 16 : 0))[lane] = reinterpret_cast<const uint32_t*>(&p)[lane];
    }
  }
}

}  // namespace

}  // namespace ccqb

namespace ccqb {

cudaMemPool_t scratch_pool(int device) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  if (device < 0 || device >= 64) device = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaDeviceGetDefaultMemPool(&pool, device);  // fall back to the default pool
    } else {
      uint64_t threshold = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    pools[device] = pool;
  }
  return pools[device];
}

}  // namespace ccqb

using namespace ccqb;

extern "C" {

const char* ccq_cuda_last_error(void) { return g_err.c_str(); }

const char* ccq_cuda_version(void) { return "ccq-b200 0.1 (sm_100a)"; }

uint64_t ccq_cuda_launch_count(void) { return g_launches.load(); }

int ccq_group_geometry(int32_t family, int32_t group_size, int32_t out6[6]) {
  Geometry g;
  const int st = geometry_for(family, group_size, &g);
  if (st != CCQ_OK) return st;
  out6[0] = g.group_size;
  out6[1] = g.full_words;
  out6[2] = g.has_tail;
  out6[3] = g.words_per_group;
  out6[4] = g.embedded_scale;
  out6[5] = g.payload_bytes;
  return CCQ_OK;
}

int ccq_clustered_code_value(uint8_t q, float alpha, float beta, int32_t code_bits,
                             uint16_t* out) {
  const long v = ref_widen(q, alpha, beta);
  if (v < 0 || v >= (1l << code_bits)) {
    return fail(CCQ_ERR_DOMAIN, "clustered code reconstructs outside [0, 2^" +
                                    std::to_string(code_bits) + "): q=" + std::to_string(int(q)));
  }
  *out = uint16_t(v);
  return CCQ_OK;
}

int ccq_cuda_model_upload_rows(const ccq_packed_view* v, int64_t r0, int64_t r1, int device,
                               ccq_dev_model** out) {
  if (!v || !out) return fail(CCQ_ERR_INVALID, "null view or output handle");
  *out = nullptr;
  Geometry geo;
  int st = geometry_for(v->family, v->group_size, &geo);
  if (st != CCQ_OK) return st;
  const FamilyConst fc = family_const(v->family);
  if (v->rows < 0 || v->cols < 0) return fail(CCQ_ERR_SHAPE, "negative shape");
  if (v->cols % v->group_size != 0)
    return fail(CCQ_ERR_FORMAT, "shape is not a whole number of groups");
  const int64_t gpr = v->cols / v->group_size;
  const uint64_t groups = uint64_t(v->rows) * uint64_t(gpr);
  if (v->code_bytes != groups * uint64_t(geo.payload_bytes) || (groups && !v->code_payload))
    return fail(CCQ_ERR_FORMAT, "codes section length does not match the geometry");
  if (!geo.embedded_scale) {
    if (v->scale_bytes != (groups + 1) / 2 || (groups && !v->scale_payload))
      return fail(CCQ_ERR_FORMAT, "group_scales section length does not match the group count");
  } else if (v->scale_bytes != 0) {
    return fail(CCQ_ERR_FORMAT, "embedded-scale family carries a side-band section");
  }
  if (v->n_super_scales != uint64_t(v->rows) || (v->rows && !v->super_scales))
    return fail(CCQ_ERR_FORMAT, "super_scales section length does not match the row count");
  if (fc.cluster) {
    if (v->n_cluster_scales != uint64_t(v->rows) || v->n_cluster_zero_points != uint64_t(v->rows) ||
        (v->rows && (!v->cluster_scales || !v->cluster_zero_points)))
      return fail(CCQ_ERR_FORMAT, "cluster_params section length does not match the row count");
  }
  if (r0 < 0 || r1 < r0 || r1 > v->rows) return fail(CCQ_ERR_SHAPE, "row range out of bounds");

  auto* m = new ccq_dev_model();
  m->device = device;
  m->rows = r1 - r0;
  m->cols = v->cols;
  m->family = v->family;
  m->group_size = v->group_size;
  m->rounds = v->rounds;
  m->geo = geo;
  m->gpr = gpr;
  const int64_t rows = m->rows;
  const uint64_t row_bytes = uint64_t(gpr) * geo.payload_bytes;
  m->nch = int((gpr + kChunk - 1) / kChunk);
  m->rows_pad = (rows + 15) / 16 * 16;
  m->cgb = uint32_t(align_up(size_t(kChunk) * geo.payload_bytes, 16));
  m->rec = m->cgb + (geo.embedded_scale ? 0u : 16u) + (fc.cluster ? 16u : 0u);
  m->payload_bytes = uint64_t(rows) * row_bytes +
                     (geo.embedded_scale ? 0 : (uint64_t(rows) * gpr + 1) / 2) + uint64_t(rows) * 4 +
                     (fc.cluster ? uint64_t(rows) * 8 : 0);

  // Device layout (ccq_internal.hpp): records | super | plans.
  const int64_t rp = m->rows_pad;
  const size_t off_codes = 0;
  const size_t off_super = align_up(off_codes + size_t(m->nch) * size_t(rp) * m->rec, 256);
  const size_t off_plan = align_up(off_super + size_t(rp) * 4, 256);
  static const bool want_w64_env = std::getenv("CCQ_W64") && std::atoi(std::getenv("CCQ_W64")) == 1;
  const bool want_w64 = fc.cluster && want_w64_env;
  const size_t off_plan64 = align_up(off_plan + (fc.cluster ? size_t(rp) * sizeof(WidenPlan) : 0), 256);
  const size_t total = align_up(off_plan64 + (want_w64 ? size_t(rp) * sizeof(double2) : 0), 256) + 256;

  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  // Staging: the row range's code bytes and nibbles exactly as stored, the
  // cluster parameters, invalid-q masks and two result words.  The view's
  // sections may be host or device memory (cudaMemcpyDefault, UVA).
  const uint64_t code_len = uint64_t(rows) * row_bytes;
  const uint64_t nib_lo = geo.embedded_scale ? 0 : (uint64_t(r0) * gpr) / 2;
  const uint64_t nib_hi = geo.embedded_scale ? 0 : (uint64_t(r1) * gpr + 1) / 2;
  const size_t s_nib = align_up(code_len, 256), s_ab = align_up(s_nib + (nib_hi - nib_lo), 256);
  const size_t s_inv = align_up(s_ab + (fc.cluster ? size_t(rows) * 8 : 0), 256);
  const size_t s_res = align_up(s_inv + (fc.cluster ? size_t(rows) * 32 : 0), 256), s_total = s_res + 256;
  uint8_t* stage = nullptr;
  // res[0]: first offending byte offset, res[1]: first row without a plan, res[2] (u32): min plan byte
  // position, res[3] (u32): some row has no exact FP64 widening plan
  unsigned long long res[4] = {~0ull, ~0ull, 3ull, 0ull};
  WidenPlan* dplans = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&m->base, total);
  if (e == cudaSuccess) {
    dplans = fc.cluster ? reinterpret_cast<WidenPlan*>(static_cast<uint8_t*>(m->base) + off_plan) : nullptr;
    e = cudaMalloc(&stage, s_total);
  }
  if (e == cudaSuccess) e = cudaMemset(m->base, 0, total);
  if (e == cudaSuccess && code_len)
    e = cudaMemcpy(stage, v->code_payload + uint64_t(r0) * row_bytes, code_len, cudaMemcpyDefault);
  if (e == cudaSuccess && nib_hi > nib_lo)
    e = cudaMemcpy(stage + s_nib, v->scale_payload + nib_lo, nib_hi - nib_lo, cudaMemcpyDefault);
  if (e == cudaSuccess && rows)
    e = cudaMemcpy(static_cast<uint8_t*>(m->base) + off_super, v->super_scales + r0, size_t(rows) * 4,
                   cudaMemcpyDefault);
  if (e == cudaSuccess && fc.cluster && rows) {
    e = cudaMemcpy(stage + s_ab, v->cluster_scales + r0, size_t(rows) * 4, cudaMemcpyDefault);
    if (e == cudaSuccess)
      e = cudaMemcpy(stage + s_ab + size_t(rows) * 4, v->cluster_zero_points + r0, size_t(rows) * 4,
                     cudaMemcpyDefault);
  }
  if (e == cudaSuccess) e = cudaMemcpy(stage + s_res, res, sizeof(res), cudaMemcpyHostToDevice);
  int64_t plan_fail = rows;  // first row without an exact plan
  if (e == cudaSuccess && fc.cluster && rp > 0) {
    build_plans<<<unsigned((rp + 127) / 128), 128>>>(
        reinterpret_cast<const float*>(stage + s_ab), reinterpret_cast<const float*>(stage + s_ab) + rows, rows, rp,
        dplans, reinterpret_cast<uint32_t*>(stage + s_inv), reinterpret_cast<unsigned long long*>(stage + s_res) + 1,
        reinterpret_cast<unsigned int*>(reinterpret_cast<unsigned long long*>(stage + s_res) + 2),
        want_w64 ? reinterpret_cast<double2*>(static_cast<uint8_t*>(m->base) + off_plan64) : nullptr,
        reinterpret_cast<unsigned int*>(reinterpret_cast<unsigned long long*>(stage + s_res) + 3));
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(res, stage + s_res, sizeof(res), cudaMemcpyDeviceToHost);
    if (res[1] != ~0ull) plan_fail = int64_t(res[1]);
    m->plan_pos_min = int(uint32_t(res[2]));
    if (want_w64) {
      m->plan64 = reinterpret_cast<double2*>(static_cast<uint8_t*>(m->base) + off_plan64);
      m->w64 = uint32_t(res[3]) == 0u;
    }
  }
  unsigned long long bad = ~0ull;
  if (e == cudaSuccess && m->nch > 0 && rp > 0) {
    const int64_t warps = int64_t(m->nch) * rp;
    const unsigned blocks = unsigned(std::min<int64_t>((warps + 7) / 8, int64_t(num_sms(device)) * 16));
    relayout_records<<<blocks, 256>>>(
        stage, row_bytes, geo.embedded_scale ? nullptr : stage + s_nib, uint64_t(r0) * gpr - 2 * nib_lo, dplans,
        fc.cluster ? reinterpret_cast<const uint32_t*>(stage + s_inv) : nullptr, std::min(rows, plan_fail), rp, gpr,
        geo.payload_bytes, m->rec, m->cgb, m->nch, static_cast<uint8_t*>(m->base) + off_codes,
        reinterpret_cast<unsigned long long*>(stage + s_res));
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(&bad, stage + s_res, sizeof(bad), cudaMemcpyDeviceToHost);
  }
  if (stage) cudaFree(stage);
  if (e != cudaSuccess) {
    if (m->base) cudaFree(m->base);
    cudaSetDevice(prev);
    delete m;
    return cuda_fail(e, "model upload");
  }
  cudaSetDevice(prev);
  // Errors in file order: a stored byte the reference rejects (coding.hpp:145-148;
  // we raise it at upload for any stored byte), or a row without an exact plan.
  const int64_t bad_row = bad == ~0ull ? rows : int64_t(bad / row_bytes);
  if (bad_row < rows && bad_row <= plan_fail) {
    uint8_t q = 0;  // the view may live on the host or the device
    cudaMemcpy(&q, v->code_payload + uint64_t(r0) * row_bytes + bad, 1, cudaMemcpyDefault);
    cudaFree(m->base);
    delete m;
    return fail(CCQ_ERR_DOMAIN, "clustered code reconstructs outside [0, 2^15): q=" + std::to_string(int(q)) +
                                    " (row " + std::to_string(r0 + bad_row) + ")");
  }
  if (plan_fail < rows) {
    cudaFree(m->base);
    delete m;
    return fail(CCQ_ERR_DOMAIN, "row " + std::to_string(r0 + plan_fail) +
                                    ": cluster parameters have no exact fixed-point widening plan");
  }
  auto* b = static_cast<uint8_t*>(m->base);
  m->device_bytes = total;
  m->codes = b + off_codes;
  m->super = reinterpret_cast<float*>(b + off_super);
  m->plan = fc.cluster ? reinterpret_cast<WidenPlan*>(b + off_plan) : nullptr;
  m->fast = geo.group_size == 64;
  *out = m;
  return CCQ_OK;
}

int ccq_cuda_model_upload(const ccq_packed_view* v, int device, ccq_dev_model** out) {
  if (!v) return fail(CCQ_ERR_INVALID, "null view");
  return ccq_cuda_model_upload_rows(v, 0, v->rows, device, out);
}

int ccq_cuda_model_free(ccq_dev_model* m) {
  if (!m) return CCQ_OK;
  if (m->base) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaFree(m->base);
    cudaSetDevice(prev);
  }
  delete m;
  return CCQ_OK;
}

int ccq_cuda_model_info(const ccq_dev_model* m, ccq_model_info* info) {
  if (!m || !info) return fail(CCQ_ERR_INVALID, "null model or info");
  std::memset(info, 0, sizeof(*info));
  info->rows = m->rows;
  info->cols = m->cols;
  info->family = m->family;
  info->group_size = m->group_size;
  info->rounds = m->rounds;
  info->device = m->device;
  info->payload_bytes_per_group = m->geo.payload_bytes;
  info->embedded_scale = m->geo.embedded_scale;
  info->payload_bytes = m->payload_bytes;
  info->device_bytes = m->device_bytes;
  info->code_row_stride = m->cgb;
  info->fast_path = m->fast ? 1 : 0;
  return CCQ_OK;
}

int ccq_model_payload_bytes(const ccq_dev_model* m, uint64_t* out) {
  if (!m || !out) return fail(CCQ_ERR_INVALID, "null model or output");
  *out = m->payload_bytes;
  return CCQ_OK;
}

int ccq_cuda_decode(const ccq_dev_model* m, int8_t* levels, float* weights, void* stream) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  DeviceScope ds(m->device);
  if (!levels && !weights) return CCQ_OK;
  return launch_decode(m, levels, weights, static_cast<cudaStream_t>(stream));
}

static int check_dtypes(int x_dtype, int y_dtype) {
  if (x_dtype < 0 || x_dtype > 2) return fail(CCQ_ERR_CONFIG, "unsupported activation dtype");
  if (y_dtype != CCQ_DTYPE_F32 && y_dtype != CCQ_DTYPE_BF16)
    return fail(CCQ_ERR_CONFIG, "unsupported output dtype");
  return CCQ_OK;
}

int ccq_cuda_gemv(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  DeviceScope ds(m->device);
  return launch_gemv(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

int ccq_cuda_gemm(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                  int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  if (!gemm_supported(m, M))
    return fail(CCQ_ERR_CONFIG, "tcgen05 GEMM needs group_size 64 and cols % 64 == 0");
  DeviceScope ds(m->device);
  return launch_gemm(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

int ccq_cuda_matmul(const ccq_dev_model* m, const void* x, int x_dtype, int64_t M, void* y,
                    int y_dtype, void* stream) {
  if (!m || (!x && M) || (!y && M)) return fail(CCQ_ERR_INVALID, "null model or operand");
  if (M < 0) return fail(CCQ_ERR_SHAPE, "negative batch");
  int st = check_dtypes(x_dtype, y_dtype);
  if (st != CCQ_OK || M == 0 || m->rows == 0) return st;
  DeviceScope ds(m->device);
  // Dispatch by batch (measured, profiles/r01_sweep.json): M = 1 on the
  // CUDA-core streaming GEMV; 2 <= M <= 8 (2.06: see below; bf16/f16 activations) on the
  // tensor-pipe GEMV when all tokens fit one launch; the tcgen05 GEMM above
  // that, or when the activations would not fit; f32 activations (the
  // reference's own f32 API) take the streaming GEMV at M = 1 and the GEMM's
  // exact hi/lo split otherwise.
  const bool mma = x_dtype != CCQ_DTYPE_F32 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                   gemv_mma_supported(m, M);
  // 2.06 hands over to the GEMM earlier when the GEMM fills the SMs (>= 3/4
  // of them with 128-row tiles x split-K): at M = 8, and at M >= 3 on
  // K-heavy layers (cols > rows: few 16-row tiles but long x staging for the
  // tensor-pipe GEMV) (profiles/r01_dispatch_thresholds.txt).
  bool gemm_earlier = false;
  if (m->family == kF206 && (M >= 8 || (m->cols > m->rows && M >= 3))) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = num_sms(dev);
    const int64_t tiles = (m->rows + 127) / 128, cblocks = (m->gpr + 7) / 8;
    const int64_t splits = tiles * 2 <= sms && cblocks >= 8 ? std::min<int64_t>(sms / tiles, cblocks / 4) : 1;
    gemm_earlier = tiles * std::max<int64_t>(splits, 1) * 4 >= int64_t(sms) * 3;
  }
  if (M >= 2 && gemv_hmma_supported(m, M, x_dtype, x)) {
    const int hs = launch_gemv_hmma(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
    if (hs != kNotApplicable) return hs;
  }
  if (mma && M >= mma_min_tokens() &&
      ((gemv_mma_fits(m, M) && !(gemm_earlier && gemm_supported(m, M))) || !gemm_supported(m, M)))
    return launch_gemv_mma(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
  if (!gemv_fast_supported(m, M) && gemm_supported(m, M))
    return launch_gemm(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
  return launch_gemv(m, x, x_dtype, M, y, y_dtype, static_cast<cudaStream_t>(stream));
}

// ---- synchronous host-buffer entry points ----

namespace {

// Scratch for the synchronous host entry points: stream-ordered allocations
// from the library pool on the legacy stream (no cudaMalloc per call).
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, nullptr);
  }
};

cudaError_t scratch_alloc(void** p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  return cudaMallocFromPoolAsync(p, bytes, ccqb::scratch_pool(dev), nullptr);
}

}  // namespace

int ccq_dequantize_host(const ccq_dev_model* m, float* out) {
  if (!m || (!out && m->rows * m->cols)) return fail(CCQ_ERR_INVALID, "null model or output");
  const size_t n = size_t(m->rows) * size_t(m->cols);
  if (n == 0) return CCQ_OK;
  DeviceScope ds(m->device);
  DevBuf w;
  CCQ_CUDA_TRY(scratch_alloc(&w.p, n * 4));
  int st = launch_decode(m, nullptr, static_cast<float*>(w.p), nullptr);
  if (st != CCQ_OK) return st;
  CCQ_CUDA_TRY(cudaMemcpy(out, w.p, n * 4, cudaMemcpyDeviceToHost));
  return CCQ_OK;
}

}  // extern "C"
namespace {

// Pinned staging for the synchronous host entry points (one per device,
// grown on demand): the reference signatures take pageable host buffers, and
// pageable cudaMemcpy costs more than the decode-GEMV itself at decode sizes
// (r01: 56.7 vs 20.9 us at 4096 -> 14336).  Calls on one device serialise on
// the stage's mutex (the entry points are synchronous anyway).
struct PinnedStage {
  std::mutex mu;
  void* h = nullptr;
  size_t cap = 0;
  cudaStream_t s = nullptr;
};
PinnedStage& pinned_stage(int dev) {
  static PinnedStage st[64];
  return st[dev >= 0 && dev < 64 ? dev : 0];
}
constexpr size_t kPinnedMax = size_t(16) << 20;  // larger transfers stay pageable

}  // namespace
extern "C" {

int ccq_gemv_batch_host(const ccq_dev_model* m, const float* x, int64_t x_rows, int64_t x_cols,
                        float* y, int64_t y_rows, int64_t y_cols) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  // kernels.cpp:153-155
  if (x_cols != m->cols || y_cols != m->rows || y_rows != x_rows)
    return fail(CCQ_ERR_SHAPE, "gemv_batch operand shapes do not match the model shape");
  if (x_rows == 0 || m->rows == 0) return CCQ_OK;
  if (m->cols == 0) {
    std::memset(y, 0, sizeof(float) * size_t(y_rows * y_cols));
    return CCQ_OK;
  }
  DeviceScope ds(m->device);
  const size_t xbytes = size_t(x_rows * x_cols) * 4, ybytes = size_t(y_rows * y_cols) * 4;
  if (xbytes + ybytes <= kPinnedMax) {
    PinnedStage& ps = pinned_stage(m->device);
    std::lock_guard<std::mutex> lock(ps.mu);
    if (!ps.s) CCQ_CUDA_TRY(cudaStreamCreateWithFlags(&ps.s, cudaStreamNonBlocking));
    const size_t need = ((xbytes + 255) & ~size_t(255)) + ybytes;
    if (ps.cap < need) {
      if (ps.h) cudaFreeHost(ps.h);
      ps.h = nullptr;
      ps.cap = 0;
      CCQ_CUDA_TRY(cudaHostAlloc(&ps.h, need, cudaHostAllocDefault));
      ps.cap = need;
    }
    uint8_t* hx = static_cast<uint8_t*>(ps.h);
    uint8_t* hy = hx + ((xbytes + 255) & ~size_t(255));
    std::memcpy(hx, x, xbytes);
    void* d = nullptr;
    CCQ_CUDA_TRY(cudaMallocFromPoolAsync(&d, ((xbytes + 255) & ~size_t(255)) + ybytes, scratch_pool(m->device), ps.s));
    uint8_t* dx = static_cast<uint8_t*>(d);
    uint8_t* dy = dx + ((xbytes + 255) & ~size_t(255));
    cudaError_t e = cudaMemcpyAsync(dx, hx, xbytes, cudaMemcpyHostToDevice, ps.s);
    int st = e == cudaSuccess ? ccq_cuda_matmul(m, dx, CCQ_DTYPE_F32, x_rows, dy, CCQ_DTYPE_F32, ps.s)
                              : cuda_fail(e, "gemv_batch H2D");
    if (st == CCQ_OK) {
      e = cudaMemcpyAsync(hy, dy, ybytes, cudaMemcpyDeviceToHost, ps.s);
      if (e != cudaSuccess) st = cuda_fail(e, "gemv_batch D2H");
    }
    cudaFreeAsync(d, ps.s);
    e = cudaStreamSynchronize(ps.s);
    if (st != CCQ_OK) return st;
    if (e != cudaSuccess) return cuda_fail(e, "gemv_batch");
    std::memcpy(y, hy, ybytes);
    return CCQ_OK;
  }
  DevBuf dx, dy;
  CCQ_CUDA_TRY(scratch_alloc(&dx.p, size_t(x_rows * x_cols) * 4));
  CCQ_CUDA_TRY(scratch_alloc(&dy.p, size_t(y_rows * y_cols) * 4));
  CCQ_CUDA_TRY(cudaMemcpy(dx.p, x, size_t(x_rows * x_cols) * 4, cudaMemcpyHostToDevice));
  int st = ccq_cuda_matmul(m, dx.p, CCQ_DTYPE_F32, x_rows, dy.p, CCQ_DTYPE_F32, nullptr);
  if (st != CCQ_OK) return st;
  CCQ_CUDA_TRY(cudaMemcpy(y, dy.p, size_t(y_rows * y_cols) * 4, cudaMemcpyDeviceToHost));
  return CCQ_OK;
}

int ccq_gemv_host(const ccq_dev_model* m, const float* x, uint64_t x_len, float* y,
                  uint64_t y_len) {
  if (!m) return fail(CCQ_ERR_INVALID, "null model");
  // kernels.cpp:125-127
  if (int64_t(x_len) != m->cols || int64_t(y_len) != m->rows)
    return fail(CCQ_ERR_SHAPE, "gemv operand sizes do not match the model shape");
  return ccq_gemv_batch_host(m, x, 1, m->cols, y, 1, m->rows);
}

}  // extern "C"
