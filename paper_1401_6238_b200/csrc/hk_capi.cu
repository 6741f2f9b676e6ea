// C ABI implementation (include/hankelfft_b200.h): plans, twiddle tables,
// validation, operand de-duplication and kernel dispatch.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>
#include <stdarg.h>
#include <stdio.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hankelfft_b200.h"
#include "hk_internal.h"
#include "hk_large.h"

using hk::Args1D;
using hk::Factor;

struct hk_plan {
  int kind;  // 1 = Hankel (1D), 2 = block / level-k
  int order;
  int levels;
  int device;
  std::vector<int64_t> sizes;   // 1D: n_p ; block: full mode sizes
  std::vector<int64_t> lshape;  // block: levels x order
  std::vector<int64_t> dof;     // per level: sum - m + 1
  std::vector<int64_t> L;       // per level FFT length
  const double2 *tw = nullptr;  // 1D twiddle table (length L[0])
  const double2 *tw0 = nullptr; // thread-major first-pass table for the fast kernels
  const double2 *tw1 = nullptr; // compact W_{L/R0} table for passes >= 1 (fast kernels)
  const float2 *twf = nullptr;  // single-precision W_L table (complex64 variant)
  // two-level plans (large 1D four-step or 2D block): L1 columns x L2 rows
  int two_level = 0;
  int twiddle = 0;               // 1D four-step (1) or 2D block (0)
  long long L1 = 0, L2 = 0;
  const double2 *thi = nullptr, *tlo = nullptr;    // four-step twiddles
  const double2 *ctw = nullptr, *ctw0 = nullptr;   // column plan tables (L1)
  const double2 *rtw = nullptr, *rtw0 = nullptr;   // row plan tables (L2)
  const double2 *rtw1 = nullptr;                     // row plan compact W_{L2/R0} table
  // block plans: inner (block) and outer sizes per mode
  std::vector<int64_t> inner, outer;
};

namespace {

thread_local std::string g_err;
bool g_force_generic = getenv("HK_FORCE_GENERIC") != nullptr;  // A/B switch for tests

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(HK_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// W_L^e = exp(-2 pi i e / L), e in [0, L), per (device, L); computed in long
// double on the host, uploaded once, never freed (bounded by the set of lengths).
std::mutex g_tw_mu;
std::map<std::pair<int, long long>, double2 *> g_tw;

int get_twiddles(int device, long long L, const double2 **out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(device, L);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) {
    *out = it->second;
    return HK_OK;
  }
  std::vector<double2> host(L);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (long long e = 0; e < L; ++e) {
    // exact symmetric reduction keeps W^{L/4}, W^{L/2} exact
    long double ang = two_pi * (long double)e / (long double)L;
    host[e].x = (double)cosl(ang);
    host[e].y = (double)-sinl(ang);
    if (4 * e == L) host[e] = make_double2(0.0, -1.0);
    if (2 * e == L) host[e] = make_double2(-1.0, 0.0);
    if (4 * e == 3 * L) host[e] = make_double2(0.0, 1.0);
  }
  double2 *d = nullptr;
  cudaError_t err = cudaMalloc(&d, L * sizeof(double2));
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(twiddles)");
  err = cudaMemcpy(d, host.data(), L * sizeof(double2), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(err, "cudaMemcpy(twiddles)");
  }
  g_tw[key] = d;
  *out = d;
  return HK_OK;
}

// Single-precision W_L^e (complex64 variant), rounded from long double.
std::map<std::pair<int, long long>, float2 *> g_twf;

int get_twiddles_f(int device, long long L, const float2 **out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(device, L);
  auto it = g_twf.find(key);
  if (it != g_twf.end()) {
    *out = it->second;
    return HK_OK;
  }
  std::vector<float2> host(L);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (long long e = 0; e < L; ++e) {
    long double ang = two_pi * (long double)e / (long double)L;
    host[e].x = (float)cosl(ang);
    host[e].y = (float)-sinl(ang);
    if (4 * e == L) host[e] = make_float2(0.f, -1.f);
    if (2 * e == L) host[e] = make_float2(-1.f, 0.f);
    if (4 * e == 3 * L) host[e] = make_float2(0.f, 1.f);
  }
  float2 *d = nullptr;
  cudaError_t err = cudaMalloc(&d, L * sizeof(float2));
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(twiddles f32)");
  err = cudaMemcpy(d, host.data(), L * sizeof(float2), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(err, "cudaMemcpy(twiddles f32)");
  }
  g_twf[key] = d;
  *out = d;
  return HK_OK;
}

// Thread-major first-pass twiddles: T0[(j-1) * (L/R0) + b] = W_L^{j b}.
std::map<std::pair<int, long long>, double2 *> g_tw0;

int get_twiddles0(int device, long long L, int R0, const double2 **out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(device, L * 1024 + R0);
  auto it = g_tw0.find(key);
  if (it != g_tw0.end()) {
    *out = it->second;
    return HK_OK;
  }
  const long long nb = L / R0;
  std::vector<double2> host((R0 - 1) * nb);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int j = 1; j < R0; ++j)
    for (long long b = 0; b < nb; ++b) {
      long long e = (j * b) % L;
      long double ang = two_pi * (long double)e / (long double)L;
      double2 w;
      w.x = (double)cosl(ang);
      w.y = (double)-sinl(ang);
      if (4 * e == L) w = make_double2(0.0, -1.0);
      if (2 * e == L) w = make_double2(-1.0, 0.0);
      if (4 * e == 3 * L) w = make_double2(0.0, 1.0);
      if (e == 0) w = make_double2(1.0, 0.0);
      host[(j - 1) * nb + b] = w;
    }
  double2 *d = nullptr;
  cudaError_t err = cudaMalloc(&d, host.size() * sizeof(double2));
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(twiddles0)");
  err = cudaMemcpy(d, host.data(), host.size() * sizeof(double2), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(err, "cudaMemcpy(twiddles0)");
  }
  g_tw0[key] = d;
  *out = d;
  return HK_OK;
}

// W_L^{q*step}, q < count (four-step twiddle tables), per (device, L, step).
std::map<std::tuple<int, long long, long long>, double2 *> g_tws;

int get_twiddles_step(int device, long long L, long long step, long long count,
                      const double2 **out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_tuple(device, L, step);
  auto it = g_tws.find(key);
  if (it != g_tws.end()) {
    *out = it->second;
    return HK_OK;
  }
  std::vector<double2> host(count);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (long long q = 0; q < count; ++q) {
    const long long e = (q * step) % L;
    long double ang = two_pi * (long double)e / (long double)L;
    host[q].x = (double)cosl(ang);
    host[q].y = (double)-sinl(ang);
    if (e == 0) host[q] = make_double2(1.0, 0.0);
    if (4 * e == L) host[q] = make_double2(0.0, -1.0);
    if (2 * e == L) host[q] = make_double2(-1.0, 0.0);
    if (4 * e == 3 * L) host[q] = make_double2(0.0, 1.0);
  }
  double2 *d = nullptr;
  cudaError_t err = cudaMalloc(&d, count * sizeof(double2));
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(twiddles)");
  err = cudaMemcpy(d, host.data(), count * sizeof(double2), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(err, "cudaMemcpy(twiddles)");
  }
  g_tws[key] = d;
  *out = d;
  return HK_OK;
}

// Tables of a length used as a row (fast / generic 1D kernel) or a column plan.
int line_tables(int dev, long long L, const double2 **tw, const double2 **tw0,
                const double2 **tw1 = nullptr) {
  int rc = get_twiddles(dev, L, tw);
  if (rc) return rc;
  const int r0 = hk::fast_first_radix(L);
  *tw0 = nullptr;
  if (tw1) *tw1 = nullptr;
  if (r0 > 0) rc = get_twiddles0(dev, L, r0, tw0);
  if (!rc && r0 > 0 && tw1 && L / r0 > 1) rc = get_twiddles(dev, L / r0, tw1);
  return rc;
}

int col_tables(int dev, long long L1, const double2 **tw, const double2 **tw0) {
  // column plans: first radix of Plan1D<L1, ...> used in hk_large.cu
  int r0 = 0;
  switch (L1) {
    case 8: r0 = 8; break;
    case 12: r0 = 12; break;
    case 16: r0 = 16; break;
    case 24: r0 = 24; break;
    case 32: r0 = 2; break;
    case 48: r0 = 3; break;
    case 64: r0 = 4; break;
    case 96: r0 = 6; break;
    case 128: r0 = 8; break;
    case 192: r0 = 12; break;
    case 256: r0 = 16; break;
    case 384: r0 = 24; break;
    case 512: r0 = 2; break;
    case 768: r0 = 3; break;
    case 1024: r0 = 4; break;
    case 1536: r0 = 6; break;
    case 2048: r0 = 8; break;
    case 3072: r0 = 12; break;
    case 4096: r0 = 16; break;
    default: return fail(HK_EUNSUPPORTED, "no column plan of length %lld", L1);
  }
  int rc = get_twiddles(dev, L1, tw);
  if (rc) return rc;
  *tw0 = nullptr;
  if (L1 <= 24) return HK_OK;  // single-pass column plans use no first-pass table
  return get_twiddles0(dev, L1, r0, tw0);
}

int check_plan(const hk_plan *p) {
  if (!p) return fail(HK_EINVAL, "plan is NULL");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != p->device)
    return fail(HK_EINVAL, "plan was created on device %d but current device is %d", p->device,
                dev);
  return HK_OK;
}

int operand_kind(int32_t dtype, int32_t *kind) {
  switch (dtype) {
    case HK_C128: *kind = hk::FK_C128; return HK_OK;
    case HK_F64: *kind = hk::FK_F64; return HK_OK;
    case HK_SPEC: *kind = hk::FK_SPEC; return HK_OK;
    case HK_C64: *kind = hk::FK_C64; return HK_OK;
    case HK_F32: *kind = hk::FK_F32; return HK_OK;
    default: return fail(HK_EINVAL, "unknown operand dtype %d", dtype);
  }
}

Factor make_factor(const hk_operand &o, int32_t kind, long long len, long long L) {
  Factor f{};
  f.ptr = o.data;
  f.bstride = o.batch_stride;
  f.sstride = 0;
  f.kind = kind;
  f.len = (int32_t)(kind == hk::FK_SPEC ? L : len);
  f.power = 1;
  f.estride = 1;
  return f;
}

Args1D base_args(const hk_plan *p, int64_t batch) {
  Args1D a{};
  a.batch = batch;
  a.nsub = 1;
  a.tw = p->tw;
  a.tw0 = p->tw0;
  a.tw1 = p->tw1;
  a.twf = p->twf;
  a.scale = 1.0 / (double)p->L[0];
  a.out_estride = 1;
  a.prefetch = getenv("HK_NO_PREFETCH") ? 0 : 1;
  return a;
}

int set_h(const hk_plan *p, const hk_operand &h, Args1D &a) {
  int32_t kind;
  int rc = operand_kind(h.dtype, &kind);
  if (rc) return rc;
  if (!h.data) return fail(HK_EINVAL, "generating vector pointer is NULL");
  a.h = make_factor(h, kind, p->dof[0], p->L[0]);
  return HK_OK;
}

// Distinct vector factors with multiplicities; mode_offset = 1 for partial
// products (xs[i] is mode i+2), 0 for full products.
int set_vectors(const hk_plan *p, const hk_operand *xs, int nx, int mode_offset, Args1D &a) {
  a.nfac = 0;
  for (int i = 0; i < nx; ++i) {
    int32_t kind;
    int rc = operand_kind(xs[i].dtype, &kind);
    if (rc) return rc;
    if (!xs[i].data) return fail(HK_EINVAL, "vector %d pointer is NULL", i);
    const long long len = p->sizes[i + mode_offset];
    bool merged = false;
    for (int f = 0; f < a.nfac; ++f) {
      Factor &fa = a.fac[f];
      if (fa.ptr == xs[i].data && fa.bstride == xs[i].batch_stride && fa.kind == kind &&
          (kind == hk::FK_SPEC || fa.len == len)) {
        fa.power += 1;
        merged = true;
        break;
      }
    }
    if (merged) continue;
    if (a.nfac >= hk::kMaxFactors)
      return fail(HK_EUNSUPPORTED, "more than %d distinct vectors in one product",
                  hk::kMaxFactors);
    a.fac[a.nfac++] = make_factor(xs[i], kind, len, p->L[0]);
  }
  return HK_OK;
}

bool single_kind(int32_t dtype) { return dtype == HK_C64 || dtype == HK_F32; }

// complex64 variant: every operand single precision, on-chip plan, no spectra.
int check_single(const hk_plan *p, const hk_operand &h, const hk_operand *xs, int nx) {
  if (!single_kind(h.dtype)) {
    for (int i = 0; i < nx; ++i)
      if (single_kind(xs[i].dtype))
        return fail(HK_EINVAL, "vector %d is single precision but h is not (mixed precision)", i);
    return 0;
  }
  for (int i = 0; i < nx; ++i)
    if (!single_kind(xs[i].dtype))
      return fail(HK_EINVAL, "vector %d must be HK_C64/HK_F32 when h is single precision", i);
  if (p->two_level || !p->twf)
    return fail(HK_EUNSUPPORTED, "the complex64 variant covers on-chip plans (L <= 8192)");
  return 1;
}

int launch_single(const hk_plan *p, const Args1D &a, void *stream) {
  cudaError_t e = hk::launch_c64_1d((int)p->L[0], a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "complex64 kernel launch");
  return HK_OK;
}

int launch(const hk_plan *p, const Args1D &a, void *stream) {
  cudaError_t e = cudaErrorNotSupported;
  if (!g_force_generic) e = hk::launch_small_1d((int)p->L[0], a, (cudaStream_t)stream);
  if (!g_force_generic && e == cudaErrorNotSupported)
    e = hk::launch_pp_1d((int)p->L[0], a, (cudaStream_t)stream);
  if (!g_force_generic && e == cudaErrorNotSupported)
    e = hk::launch_fast_1d((int)p->L[0], a, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) e = hk::launch_1d((int)p->L[0], a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "hankel 1d kernel launch");
  return HK_OK;
}

}  // namespace

extern "C" {

int hk_version(void) { return 100; }

const char *hk_last_error(void) { return g_err.c_str(); }

int hk_plan_create_hankel(hk_plan **plan, int order, const int64_t *mode_sizes, int64_t fft_len) {
  if (!plan) return fail(HK_EINVAL, "plan output pointer is NULL");
  *plan = nullptr;
  if (order < 2) return fail(HK_EINVAL, "order must be at least 2");
  if (!mode_sizes) return fail(HK_EINVAL, "mode_sizes is NULL");
  long long d = 0;
  for (int i = 0; i < order; ++i) {
    if (mode_sizes[i] < 1) return fail(HK_EINVAL, "shape entries must be positive");
    d += mode_sizes[i];
  }
  d = d - order + 1;
  if (fft_len > 0 && fft_len < d)
    return fail(HK_EINVAL, "fft_len %lld is shorter than d_H = %lld", (long long)fft_len, d);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  long long L = fft_len > 0 ? fft_len : hk::choose_len_1d(d);
  hk_plan *p = new hk_plan();
  p->kind = 1;
  p->order = order;
  p->levels = 1;
  p->device = dev;
  p->sizes.assign(mode_sizes, mode_sizes + order);
  p->dof = {d};
  int rc = HK_OK;
  if (L > 0 && hk::supported_1d(L)) {
    p->L = {L};
    rc = line_tables(dev, L, &p->tw, &p->tw0, &p->tw1);
    if (!rc) rc = get_twiddles_f(dev, L, &p->twf);
  } else {
    // two-level four-step: L = L1 * L2 (L1 column plan, L2 fast row plan)
    long long best1 = 0, best2 = 0;
    for (long long l2 : {256LL, 384LL, 512LL, 768LL, 1024LL, 1536LL, 2048LL, 3072LL, 4096LL,
                         6144LL, 8192LL})
      for (long long l1 : {8LL, 12LL, 16LL, 24LL, 32LL, 48LL, 64LL, 96LL, 128LL, 192LL, 256LL,
                           384LL, 512LL, 768LL, 1024LL, 1536LL, 2048LL, 3072LL, 4096LL}) {
        const long long l = l1 * l2;
        if (fft_len > 0 ? l != fft_len : l < d) continue;
        // smallest L; on ties prefer rows with a fast kernel, then fewer columns
        const bool fast2 = hk::fast_first_radix(l2) > 0;
        const bool bfast = best1 && hk::fast_first_radix(best2) > 0;
        // HK_ROW_LEN: A/B knob preferring a row length among equal-L splits
        // (B200 cfg3: 1536 x 8192 877 us, 2048 x 6144 1087 us)
        static const long long want2 = getenv("HK_ROW_LEN") ? atoll(getenv("HK_ROW_LEN")) : 0;
        // default: 4096-point rows (two resident row CTAs per SM: B200 cfg3 row
        // stage 137 vs 205 us for 8192) when the TMA column kernel covers L1
        auto prefer = [&](long long c1, long long c2) {
          return want2 > 0 ? c2 == want2 : (c2 == 4096 && hk::tma_col_len(c1));
        };
        const bool pref = prefer(l1, l2), bpref = best1 && prefer(best1, best2);
        if (!best1 || l < best1 * best2 ||
            (l == best1 * best2 &&
             (pref > bpref ||
              (pref == bpref && (fast2 > bfast || (fast2 == bfast && l1 < best1)))))) {
          best1 = l1;
          best2 = l2;
        }
      }
    if (!best1) {
      delete p;
      return fail(HK_EUNSUPPORTED, fft_len > 0 ? "FFT length %lld is not supported"
                                               : "d_H = %lld exceeds the supported lengths",
                  fft_len > 0 ? (long long)fft_len : d);
    }
    p->two_level = 1;
    p->twiddle = 1;
    p->L1 = best1;
    p->L2 = best2;
    p->L = {best1 * best2};
    const long long Lt = best1 * best2;
    rc = line_tables(dev, best2, &p->rtw, &p->rtw0, &p->rtw1);
    if (!rc) rc = col_tables(dev, best1, &p->ctw, &p->ctw0);
    if (!rc) rc = get_twiddles_step(dev, Lt, 4096, (Lt + 4095) / 4096, &p->thi);
    if (!rc) rc = get_twiddles_step(dev, Lt, 1, 4096, &p->tlo);
  }
  if (rc) {
    delete p;
    return rc;
  }
  *plan = p;
  return HK_OK;
}

int hk_plan_create_block(hk_plan **plan, int order, int levels, const int64_t *level_shapes,
                         const int64_t *fft_lens) {
  if (!plan) return fail(HK_EINVAL, "plan output pointer is NULL");
  *plan = nullptr;
  if (order < 2) return fail(HK_EINVAL, "order must be at least 2");
  if (!level_shapes) return fail(HK_EINVAL, "level_shapes is NULL");
  if (levels != 2)
    return fail(HK_EUNSUPPORTED, "block plans cover 2 levels (BHHB); use the Kronecker 1D form");
  long long din = 0, dout = 0;
  std::vector<int64_t> inner(order), outer(order), sizes(order);
  for (int i = 0; i < order; ++i) {
    inner[i] = level_shapes[i];
    outer[i] = level_shapes[order + i];
    if (inner[i] < 1 || outer[i] < 1) return fail(HK_EINVAL, "shape entries must be positive");
    din += inner[i];
    dout += outer[i];
    sizes[i] = inner[i] * outer[i];
  }
  din = din - order + 1;
  dout = dout - order + 1;
  long long L2 = fft_lens && fft_lens[0] > 0 ? fft_lens[0] : hk::choose_len_1d(din);
  if (!(fft_lens && fft_lens[0] > 0) && L2 > 0) {
    // rows run on the all-radix-16 plans (256, 4096: immediate-offset smem
    // addressing) when that costs at most 40% more length, e.g. 190 -> 256
    // rather than 192: measured faster on B200 despite the extra points
    // HK_PP192=1 (A/B): keep 192-point rows for the 16 x 12 ping-pong row kernel
    for (long long l2 : {256LL, 4096LL})
      if (l2 >= din && l2 != L2 && l2 * 10 <= L2 * 14 && !(L2 == 192 && getenv("HK_PP192"))) {
        L2 = l2;
        break;
      }
  }
  long long L1 = 0;
  if (fft_lens && fft_lens[1] > 0) {
    L1 = fft_lens[1];
  } else {
    for (long long l1 : {8LL, 12LL, 16LL, 24LL, 32LL, 48LL, 64LL, 96LL, 128LL, 192LL, 256LL,
                         384LL, 512LL, 768LL, 1024LL, 1536LL, 2048LL, 3072LL, 4096LL})
      if (l1 >= dout) {
        L1 = l1;
        break;
      }
  }
  const bool auto2 = !(fft_lens && fft_lens[0] > 0), auto1 = !(fft_lens && fft_lens[1] > 0);
  if ((auto2 && L2 <= 0) || (auto1 && L1 <= 0))  // no supported length covers the generator
    return fail(HK_EUNSUPPORTED, "block generator %lldx%lld exceeds the supported lengths", din,
                dout);
  if (L2 < din || L1 < dout) return fail(HK_EINVAL, "fft lengths shorter than the generator");
  if (L2 <= 0 || !hk::supported_1d(L2) || !hk::supported_col_len(L1))
    return fail(HK_EUNSUPPORTED, "block generator %lldx%lld exceeds the supported lengths", din,
                dout);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  hk_plan *p = new hk_plan();
  p->kind = 2;
  p->order = order;
  p->levels = 2;
  p->device = dev;
  p->sizes = sizes;
  p->inner = inner;
  p->outer = outer;
  p->dof = {din, dout};
  p->L = {L2, L1};
  p->two_level = 1;
  p->twiddle = 0;
  p->L1 = L1;
  p->L2 = L2;
  int rc = line_tables(dev, L2, &p->rtw, &p->rtw0);
  if (!rc) rc = col_tables(dev, L1, &p->ctw, &p->ctw0);
  if (rc) {
    delete p;
    return rc;
  }
  *plan = p;
  return HK_OK;
}

int hk_plan_destroy(hk_plan *plan) {
  delete plan;
  return HK_OK;
}

int64_t hk_plan_fft_len(const hk_plan *plan, int level) {
  if (!plan || level < 0 || level >= (int)plan->L.size()) return -1;
  return plan->L[level];
}

int64_t hk_plan_spectrum_len(const hk_plan *plan) {
  if (!plan) return -1;
  int64_t n = 1;
  for (auto l : plan->L) n *= l;
  return n;
}

namespace {
// Items processed per two-level chunk (bounds the workspace to ~1 GiB).
long long tl_per_item(const hk_plan *p) {
  return (long long)(p->order + 2) * p->L1 * p->L2 + p->L1;  // Wh, order x Wx, Wq, row sums
}
long long tl_chunk(const hk_plan *p, long long batch) {
  long long cap = std::max(1LL, (1LL << 28) / tl_per_item(p));  // 2^28 complex = 4 GiB
  static const long long env_cap = getenv("HK_TL_CHUNK") ? atoll(getenv("HK_TL_CHUNK")) : 0;
  if (env_cap > 0) cap = std::min(cap, env_cap);
  return std::max(1LL, std::min(batch, cap));
}
}  // namespace


namespace {

int launch_row(long long L2, const Args1D &a, cudaStream_t st) {
  cudaError_t e = cudaErrorNotSupported;
  // 4096-point rows: the TMA ping-pong kernel (two row products per SM)
  if (!g_force_generic) e = hk::launch_pp_1d((int)L2, a, st);
  if (!g_force_generic && e == cudaErrorNotSupported) e = hk::launch_fast_1d((int)L2, a, st);
  if (e == cudaErrorNotSupported) e = hk::launch_1d((int)L2, a, st);
  if (e != cudaSuccess) return cuda_fail(e, "row-stage kernel launch");
  return HK_OK;
}

int elem_bytes(int32_t dtype) { return dtype == HK_F64 ? 8 : 16; }

// Operand of mode `mode` (0-based) of a two-level plan as an L1 x L2 array.
// `es` is the element stride inside one vector (1 = contiguous; a column of a
// row-major matrix with R columns has es = R).
hk::large::Op2 tl_vector_op(const hk_plan *p, const hk_operand &o, int mode, long long b0,
                            int *ncols, long long es = 1) {
  hk::large::Op2 op{};
  op.ptr = static_cast<const char *>(o.data) + b0 * o.batch_stride * elem_bytes(o.dtype);
  op.item_stride = o.batch_stride;
  op.kind = o.dtype == HK_F64 ? hk::FK_F64 : hk::FK_C128;
  op.scale = 1.0;
  if (p->twiddle) {  // 1D four-step
    const long long n = p->sizes[mode];
    op.s1 = p->L2 * es;
    op.s2 = es;
    op.len = n;
    *ncols = (int)std::min<long long>(p->L2, n);
  } else {  // 2D block: F-order (inner n x outer N), element (i, j) at i + n j
    const long long n = p->inner[mode], N = p->outer[mode];
    op.s1 = n * es;
    op.s2 = es;
    op.len = -1;
    op.e1 = (int32_t)N;
    op.e2 = (int32_t)n;
    *ncols = (int)n;
  }
  return op;
}

// what: 0 partial (y), 1 full (alpha), 2 spectrum (stage-A output of h).
// xes: per-vector element strides (NULL = contiguous); oes: element stride of y.
int tl_run(const hk_plan *p, const hk_operand &h, const hk_operand *xs, int nx, int mode_offset,
           int64_t batch, void *out, int64_t out_stride, void *ws, void *stream, int what,
           const long long *xes = nullptr, long long oes = 1) {
  if (batch == 0) return HK_OK;
  if (!ws) return fail(HK_EINVAL, "two-level plans need a workspace of hk_workspace_bytes()");
  cudaStream_t st = (cudaStream_t)stream;
  const long long L1 = p->L1, L2 = p->L2, L = L1 * L2;
  // distinct vector factors
  struct Fac {
    hk_operand op;
    int mode;
    int power;
    long long es;
  };
  std::vector<Fac> fs;
  for (int i = 0; i < nx; ++i) {
    if (!xs[i].data) return fail(HK_EINVAL, "vector %d pointer is NULL", i);
    if (xs[i].dtype != HK_C128 && xs[i].dtype != HK_F64)
      return fail(HK_EINVAL, "vector %d: two-level plans take raw vectors", i);
    const int mode = i + mode_offset;
    const long long es = xes ? xes[i] : 1;
    bool merged = false;
    for (auto &f : fs)
      if (f.op.data == xs[i].data && f.op.batch_stride == xs[i].batch_stride &&
          f.op.dtype == xs[i].dtype && f.es == es && p->sizes[f.mode] == p->sizes[mode] &&
          (p->twiddle || (p->inner[f.mode] == p->inner[mode]))) {
        ++f.power;
        merged = true;
        break;
      }
    if (!merged) fs.push_back({xs[i], mode, 1, es});
  }
  if ((int)fs.size() > p->order || (int)fs.size() > hk::kMaxFactors)
    return fail(HK_EUNSUPPORTED, "too many distinct vectors for the two-level workspace");
  // 2-level block product with one distinct vector: the fused on-chip kernel
  // (192 x 192 spectrum in four residue passes, hk_bhhb_fused.cu)
  if (!p->twiddle && what == 0 && fs.size() == 1 && h.dtype == HK_C128 &&
      fs[0].op.dtype == HK_C128 && fs[0].es == 1 && oes == 1 &&
      p->inner[fs[0].mode] == p->inner[0] && p->outer[fs[0].mode] == p->outer[0]) {
    const double2 *t48 = nullptr, *t192 = nullptr;  // cached per device by get_twiddles
    int rc2 = get_twiddles(p->device, 48, &t48);
    if (!rc2) rc2 = get_twiddles(p->device, 192, &t192);
    if (!rc2) {
      hk::bhhb::Args ba{};
      ba.h = static_cast<const double2 *>(h.data);
      ba.h_bstride = h.batch_stride;
      ba.x = static_cast<const double2 *>(fs[0].op.data);
      ba.x_bstride = fs[0].op.batch_stride;
      ba.y = static_cast<double2 *>(out);
      ba.y_bstride = out_stride;
      ba.batch = batch;
      ba.din = (int)p->dof[0];
      ba.dout = (int)p->dof[1];
      ba.n = (int)p->inner[0];
      ba.N = (int)p->outer[0];
      ba.power = fs[0].power;
      ba.tw48 = t48;
      ba.tw192 = t192;
      ba.scale = 1.0 / (192.0 * 192.0);
      const cudaError_t e = hk::launch_bhhb_fused(ba, st);
      if (e == cudaSuccess) return HK_OK;
      if (e != cudaErrorNotSupported) return cuda_fail(e, "fused block kernel launch");
    }
  }
  const long long chunk = tl_chunk(p, batch);
  double2 *W = static_cast<double2 *>(ws);
  double2 *Wh = W;
  double2 *Wx = Wh + chunk * L;
  double2 *Wq = Wx + (long long)p->order * chunk * L;
  double2 *part = Wq + chunk * L;

  hk::large::ColArgs ca{};
  ca.L1 = (int32_t)L1;
  ca.L2 = (int32_t)L2;
  ca.L = L;
  ca.twiddle = p->twiddle;
  ca.thi = p->thi;
  ca.tlo = p->tlo;
  ca.ctw = p->ctw;
  ca.ctw0 = p->ctw0;
  const long long d = p->dof[0];
  const long long din = p->twiddle ? d : p->dof[0], dout = p->twiddle ? 0 : p->dof[1];
  const int hcols = (int)(p->twiddle ? std::min(L2, d) : din);
  int ocols = 0;
  hk::large::Out2 yout{};
  if (p->twiddle) {
    ocols = (int)std::min<long long>(L2, p->sizes[0]);
  } else {
    ocols = (int)p->inner[0];
  }
  // Real h and ONE real vector (the f64 configs, e.g. cfg3): one packed
  // column pass z = h + i x serves both (ST_A_PAIR).
  const bool pair = p->twiddle && what != 2 && h.dtype == HK_F64 && fs.size() == 1 &&
                    fs[0].op.dtype == HK_F64 && !getenv("HK_NO_PAIR");
  // Real h and real vectors make the spectral product Hermitian,
  // P(L - k) = conj P(k): rows k1 and L1 - k1 of every stage carry the same
  // information (Q(L1-k1, m2) = conj(W_L2^{m2} Q(k1, m2))), so the row stage
  // runs rows 0..L1/2 only and the final column pass synthesises the rest.
  const bool half = pair && what == 0 && L1 % 2 == 0 && !getenv("HK_NO_HALF");
  const long long rows_b = half ? L1 / 2 + 1 : L1;
  ca.half = 0;
  for (long long b0 = 0; b0 < batch; b0 += chunk) {
    const long long nb = std::min(chunk, batch - b0);
    cudaError_t e;
    // ---- stage A: h (inverse, 1/L applied here)
    const double2 *whp = Wh;
    long long wh_item = L;
    int pair_xcols = 0;
    if (pair) {
      ca.in = hk::large::Op2{};
      ca.in.ptr = static_cast<const char *>(h.data) + b0 * h.batch_stride * elem_bytes(h.dtype);
      ca.in.item_stride = h.batch_stride;
      ca.in.kind = hk::FK_F64;
      ca.in.scale = 1.0 / (double)L;
      ca.in.s1 = L2;
      ca.in.s2 = 1;
      ca.in.len = d;
      ca.in_n1_fast = 0;
      ca.in2 = tl_vector_op(p, fs[0].op, fs[0].mode, b0, &pair_xcols, fs[0].es);
      // Hermitian product: rows k1 > L1/2 are never read (see `half` below)
      const int32_t rows_out = half ? (int32_t)(L1 / 2 + 1) : (int32_t)L1;
      ca.out = hk::large::Out2{Wh, L, L2, 1, -1, rows_out, (int32_t)L2};
      ca.out2 = hk::large::Out2{Wx, L, L2, 1, -1, rows_out, (int32_t)L2};
      if ((e = hk::launch_cols(hk::large::ST_A_PAIR, ca, nb, hcols, st)) != cudaSuccess)
        return cuda_fail(e, "column stage (h + i x)");
    } else if (h.dtype == HK_SPEC) {
      whp = static_cast<const double2 *>(h.data) + b0 * h.batch_stride;
      wh_item = h.batch_stride;
    } else {
      ca.in = hk::large::Op2{};
      ca.in.ptr = static_cast<const char *>(h.data) + b0 * h.batch_stride * elem_bytes(h.dtype);
      ca.in.item_stride = h.batch_stride;
      ca.in.kind = h.dtype == HK_F64 ? hk::FK_F64 : hk::FK_C128;
      ca.in.scale = 1.0 / (double)L;
      if (p->twiddle) {
        ca.in.s1 = L2;
        ca.in.s2 = 1;
        ca.in.len = d;
        ca.in_n1_fast = 0;
      } else {  // H[s][t], s = inner sum (n2), t = outer sum (n1), t contiguous
        ca.in.s1 = 1;
        ca.in.s2 = dout;
        ca.in.len = -1;
        ca.in.e1 = (int32_t)dout;
        ca.in.e2 = (int32_t)din;
        ca.in_n1_fast = 1;
      }
      double2 *dst = what == 2 ? static_cast<double2 *>(out) + b0 * L : Wh;
      ca.out = hk::large::Out2{dst, L, L2, 1, -1, (int32_t)L1, (int32_t)L2};
      if ((e = hk::launch_cols(hk::large::ST_A_INV, ca, nb, hcols, st)) != cudaSuccess)
        return cuda_fail(e, "column stage (h)");
      if (what == 2) continue;
    }
    // ---- stage A: distinct vectors (forward)
    Args1D a{};
    a.batch = nb * rows_b;
    a.nsub = rows_b;
    a.tw = p->rtw;
    a.tw0 = p->rtw0;
    a.tw1 = p->rtw1;
    a.scale = 1.0;
    a.prefetch = 1;
    a.h.ptr = whp;
    a.h.bstride = wh_item;
    a.h.sstride = L2;
    a.h.len = hcols;
    a.h.power = 1;
    a.h.kind = hk::FK_C128;
    a.h.estride = 1;
    a.nfac = (int)fs.size();
    for (size_t f = 0; f < fs.size(); ++f) {
      int ncols = 0;
      double2 *wx = Wx + (long long)f * chunk * L;
      if (pair) {
        ncols = pair_xcols;  // written by the packed pass above
      } else {
        ca.in = tl_vector_op(p, fs[f].op, fs[f].mode, b0, &ncols, fs[f].es);
        ca.in_n1_fast = 0;
        ca.out = hk::large::Out2{wx, L, L2, 1, -1, (int32_t)L1, (int32_t)ncols};
        if ((e = hk::launch_cols(hk::large::ST_A_FWD, ca, nb, ncols, st)) != cudaSuccess)
          return cuda_fail(e, "column stage (x)");
      }
      hk::Factor &fa = a.fac[f];
      fa.ptr = wx;
      fa.bstride = L;
      fa.sstride = L2;
      fa.len = ncols;
      fa.power = fs[f].power;
      fa.kind = hk::FK_C128;
      fa.estride = 1;
    }
    // ---- stage B: row products
    if (what == 0) {
      a.mode = hk::M_PARTIAL;
      a.out = Wq;
      a.out_bstride = L;
      a.out_sstride = L2;
      a.out_estride = 1;
      a.out_len = ocols;
    } else {
      a.mode = hk::M_FULL;
      a.out = part;
      a.out_bstride = L1;
      a.out_sstride = 1;
      a.out_estride = 1;
    }
    int rc = launch_row(L2, a, st);
    if (rc) return rc;
    // ---- stage C: final column transform / reduction
    if (what == 0) {
      ca.in = hk::large::Op2{};
      ca.in.ptr = Wq;
      ca.in.item_stride = L;
      ca.in.s1 = L2;
      ca.in.s2 = 1;
      ca.in.len = -1;
      ca.in.e1 = (int32_t)L1;
      ca.in.e2 = ocols;
      ca.in.kind = hk::FK_C128;
      ca.in.scale = 1.0;
      ca.in_n1_fast = 0;
      yout.ptr = static_cast<double2 *>(out) + b0 * out_stride;
      yout.item_stride = out_stride;
      if (p->twiddle) {
        yout.s1 = L2 * oes;
        yout.s2 = oes;
        yout.len = p->sizes[0];
      } else {
        yout.s1 = p->inner[0] * oes;
        yout.s2 = oes;
        yout.len = -1;
        yout.e1 = (int32_t)p->outer[0];
        yout.e2 = (int32_t)p->inner[0];
      }
      ca.out = yout;
      ca.half = half ? 1 : 0;
      if ((e = hk::launch_cols(hk::large::ST_C, ca, nb, ocols, st)) != cudaSuccess)
        return cuda_fail(e, "column stage (y)");
    } else {
      if ((e = hk::launch_rowsum(part, L1, static_cast<double2 *>(out) + b0, nb, st)) !=
          cudaSuccess)
        return cuda_fail(e, "row-sum kernel");
    }
  }
  return HK_OK;
}

}  // namespace

namespace {

// times_matrices for two-level plans (L > 8192 1D four-step, 2D block): one
// four-step product per column combination, the columns read in place from
// the row-major matrices (element stride R) and T written in place (element
// stride = number of combinations).  The spectrum of h is computed once.  When
// m = 3 and both matrices are the same, only j2 <= j3 is computed and the
// result mirrored to T[:, j3, j2] by a strided device copy.
int tl_times_matrices(const hk_plan *p, const hk_operand &h, const void *const *mats,
                      const int64_t *mat_strides, const int64_t *ranks, int nmats, int64_t batch,
                      void *T, int64_t t_stride, void *workspace, void *stream,
                      long long ncombo) {
  const long long L = hk_plan_spectrum_len(p);
  double2 *wsb = static_cast<double2 *>(workspace);
  hk_operand hs = h;
  int rc;
  if (h.dtype != HK_SPEC) {
    if ((rc = tl_run(p, h, nullptr, 0, 0, batch, wsb, 0, wsb + batch * L, stream, 2))) return rc;
    hs = hk_operand{wsb, L, HK_SPEC, 0};
    wsb += batch * L;
  }
  for (int i = 0; i < nmats; ++i)
    if (!mats[i]) return fail(HK_EINVAL, "matrix %d pointer is NULL", i);
  const bool sym2 = nmats == 2 && mats[0] == mats[1] && mat_strides[0] == mat_strides[1] &&
                    ranks[0] == ranks[1] && p->sizes[1] == p->sizes[2];
  const long long n1 = p->sizes[0];
  std::vector<hk_operand> xs(nmats);
  std::vector<long long> es(nmats), j(nmats);
  for (long long c = 0; c < ncombo; ++c) {
    long long rem = c;
    for (int i = nmats - 1; i >= 0; --i) {
      j[i] = rem % ranks[i];
      rem /= ranks[i];
    }
    if (sym2 && j[1] < j[0]) continue;
    for (int i = 0; i < nmats; ++i) {
      xs[i] = hk_operand{static_cast<const double2 *>(mats[i]) + j[i], mat_strides[i], HK_C128, 0};
      es[i] = ranks[i];
    }
    if ((rc = tl_run(p, hs, xs.data(), nmats, 1, batch, static_cast<double2 *>(T) + c, t_stride,
                     wsb, stream, 0, es.data(), ncombo)))
      return rc;
    if (sym2 && j[1] != j[0]) {
      const long long c2 = j[1] * ranks[1] + j[0];
      const size_t pitch = (size_t)ncombo * sizeof(double2);
      cudaStream_t st = (cudaStream_t)stream;
      cudaError_t e = cudaSuccess;
      if (t_stride == n1 * ncombo) {
        e = cudaMemcpy2DAsync(static_cast<double2 *>(T) + c2, pitch, static_cast<double2 *>(T) + c,
                              pitch, sizeof(double2), (size_t)(batch * n1),
                              cudaMemcpyDeviceToDevice, st);
      } else {
        for (long long b = 0; b < batch && e == cudaSuccess; ++b)
          e = cudaMemcpy2DAsync(static_cast<double2 *>(T) + b * t_stride + c2, pitch,
                                static_cast<double2 *>(T) + b * t_stride + c, pitch,
                                sizeof(double2), (size_t)n1, cudaMemcpyDeviceToDevice, st);
      }
      if (e != cudaSuccess) return cuda_fail(e, "mirror copy of a symmetric combination");
    }
  }
  return HK_OK;
}

}  // namespace

size_t hk_workspace_bytes(const hk_plan *plan, int64_t batch) {
  if (!plan || !plan->two_level || batch <= 0) return 0;
  return (size_t)tl_chunk(plan, batch) * (size_t)tl_per_item(plan) * sizeof(double2);
}

int hk_spectrum(const hk_plan *plan, hk_operand h, int64_t batch, void *spec, void *workspace,
                void *stream) {
  (void)workspace;
  int rc = check_plan(plan);
  if (rc) return rc;
  if (batch < 0) return fail(HK_EINVAL, "negative batch");
  if (batch == 0) return HK_OK;
  if (h.dtype == HK_SPEC) return fail(HK_EINVAL, "h is already a spectrum");
  if (single_kind(h.dtype))
    return fail(HK_EUNSUPPORTED, "cached spectra exist for complex128 only");
  if (!spec) return fail(HK_EINVAL, "spec is NULL");
  if (plan->two_level) return tl_run(plan, h, nullptr, 0, 0, batch, spec, 0, workspace, stream, 2);
  Args1D a = base_args(plan, batch);
  if ((rc = set_h(plan, h, a))) return rc;
  a.nfac = 0;
  a.mode = hk::M_SPEC_H;
  a.out = spec;
  a.out_bstride = plan->L[0];
  return launch(plan, a, stream);
}

int hk_tvp_partial(const hk_plan *plan, hk_operand h, const hk_operand *xs, int nx,
                   int64_t batch, void *y, int64_t y_stride, void *workspace, void *stream) {
  (void)workspace;
  int rc = check_plan(plan);
  if (rc) return rc;
  if (nx != plan->order - 1)
    return fail(HK_EINVAL, "expected %d vectors, got %d", plan->order - 1, nx);
  if (batch < 0) return fail(HK_EINVAL, "negative batch");
  if (batch == 0) return HK_OK;
  if (!y) return fail(HK_EINVAL, "y is NULL");
  if (!xs) return fail(HK_EINVAL, "xs is NULL");
  const int single = check_single(plan, h, xs, nx);
  if (single < 0) return single;
  if (plan->two_level) return tl_run(plan, h, xs, nx, 1, batch, y, y_stride, workspace, stream, 0);
  Args1D a = base_args(plan, batch);
  if ((rc = set_h(plan, h, a))) return rc;
  if ((rc = set_vectors(plan, xs, nx, 1, a))) return rc;
  a.mode = hk::M_PARTIAL;
  a.out = y;
  a.out_bstride = y_stride;
  a.out_len = (int32_t)plan->sizes[0];
  return single ? launch_single(plan, a, stream) : launch(plan, a, stream);
}

int hk_tvp_partial_host(const hk_plan *plan, hk_operand h, const void *host_in, int64_t in_elems,
                        const int64_t *x_offsets, int nx, void *dev_in, void *dev_y,
                        void *host_y, void *stream) {
  int rc = check_plan(plan);
  if (rc) return rc;
  if (plan->two_level) return fail(HK_EUNSUPPORTED, "host latency path covers on-chip plans only");
  if (single_kind(h.dtype)) return fail(HK_EUNSUPPORTED, "host latency path is complex128 only");
  if (nx != plan->order - 1)
    return fail(HK_EINVAL, "expected %d vectors, got %d", plan->order - 1, nx);
  if (nx > hk::kMaxFactors) return fail(HK_EUNSUPPORTED, "too many vectors");
  if (!host_in || !dev_in || !dev_y || !host_y || !x_offsets || in_elems < 0)
    return fail(HK_EINVAL, "NULL buffer or negative size");
  for (int i = 0; i < nx; ++i)
    if (x_offsets[i] < 0 || x_offsets[i] + plan->sizes[i + 1] > in_elems)
      return fail(HK_EINVAL, "vector %d lies outside the input buffer", i);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n1 = plan->sizes[0];
  hk_operand xs[hk::kMaxFactors];
  // Zero-copy for the latency kernel's sizes: when both pinned buffers are
  // mapped into the device address space (always, under UVA) the kernel reads
  // the vectors and writes y over PCIe directly -- no copy launches.
  void *din = nullptr, *dy = nullptr;
  static const bool no_zc = getenv("HK_NO_ZEROCOPY") != nullptr;
  if (!no_zc && plan->L[0] <= 4096 &&
      cudaHostGetDevicePointer(&din, const_cast<void *>(host_in), 0) == cudaSuccess &&
      cudaHostGetDevicePointer(&dy, host_y, 0) == cudaSuccess) {
    for (int i = 0; i < nx; ++i)
      xs[i] = hk_operand{static_cast<double2 *>(din) + x_offsets[i], 0, HK_C128, 0};
    if ((rc = hk_tvp_partial(plan, h, xs, nx, 1, dy, n1, nullptr, stream))) return rc;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return HK_OK;
  }
  cudaGetLastError();  // clear a failed cudaHostGetDevicePointer
  cudaError_t e = cudaMemcpyAsync(dev_in, host_in, (size_t)in_elems * sizeof(double2),
                                  cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(H2D)");
  for (int i = 0; i < nx; ++i)
    xs[i] = hk_operand{static_cast<double2 *>(dev_in) + x_offsets[i], 0, HK_C128, 0};
  if ((rc = hk_tvp_partial(plan, h, xs, nx, 1, dev_y, n1, nullptr, stream))) return rc;
  e = cudaMemcpyAsync(host_y, dev_y, (size_t)n1 * sizeof(double2), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return HK_OK;
}

int hk_tvp_full(const hk_plan *plan, hk_operand h, const hk_operand *xs, int nx, int64_t batch,
                void *alpha, void *workspace, void *stream) {
  (void)workspace;
  int rc = check_plan(plan);
  if (rc) return rc;
  if (nx != plan->order) return fail(HK_EINVAL, "expected %d vectors, got %d", plan->order, nx);
  if (batch < 0) return fail(HK_EINVAL, "negative batch");
  if (batch == 0) return HK_OK;
  if (!alpha) return fail(HK_EINVAL, "alpha is NULL");
  if (!xs) return fail(HK_EINVAL, "xs is NULL");
  const int single = check_single(plan, h, xs, nx);
  if (single < 0) return single;
  if (plan->two_level) return tl_run(plan, h, xs, nx, 0, batch, alpha, 1, workspace, stream, 1);
  Args1D a = base_args(plan, batch);
  if ((rc = set_h(plan, h, a))) return rc;
  if ((rc = set_vectors(plan, xs, nx, 0, a))) return rc;
  a.mode = hk::M_FULL;
  a.out = alpha;
  a.out_bstride = 1;
  return single ? launch_single(plan, a, stream) : launch(plan, a, stream);
}

int hk_vector_spectra(const hk_plan *plan, int mode, const void *mats, int64_t mat_stride,
                      int64_t ncols, int64_t batch, void *spec, void *stream) {
  int rc = check_plan(plan);
  if (rc) return rc;
  if (mode < 1 || mode > plan->order) return fail(HK_EINVAL, "mode %d out of range", mode);
  if (ncols < 1 || batch < 0) return fail(HK_EINVAL, "bad ncols/batch");
  if (batch == 0) return HK_OK;
  if (!mats || !spec) return fail(HK_EINVAL, "NULL matrix or spectrum pointer");
  if (plan->two_level)
    return fail(HK_EUNSUPPORTED,
                "column spectra exist for on-chip plans only (two-level plans transform the "
                "columns inside hk_times_matrices)");
  const long long L = plan->L[0];
  Args1D a = base_args(plan, batch * ncols);
  a.nsub = ncols;
  a.nfac = 1;
  Factor &f = a.fac[0];
  f.ptr = mats;
  f.bstride = mat_stride;
  f.sstride = 1;
  f.estride = (int32_t)ncols;
  f.len = (int32_t)plan->sizes[mode - 1];
  f.power = 1;
  f.kind = hk::FK_C128;
  a.mode = hk::M_SPEC_F;
  a.out = spec;
  a.out_bstride = ncols * L;
  a.out_sstride = L;
  return launch(plan, a, stream);
}

size_t hk_times_matrices_workspace_bytes(const hk_plan *plan, const int64_t *ranks, int nmats,
                                         int64_t batch) {
  if (!plan || !ranks || batch <= 0) return 0;
  if (plan->two_level)  // cached spectrum of h + the four-step workspace
    return (size_t)batch * (size_t)hk_plan_spectrum_len(plan) * sizeof(double2) +
           hk_workspace_bytes(plan, batch);
  long long cols = 1;  // spectrum of h
  for (int i = 0; i < nmats; ++i) cols += ranks[i];
  return (size_t)cols * (size_t)plan->L[0] * (size_t)batch * sizeof(double2);
}

int hk_times_matrices(const hk_plan *plan, hk_operand h, const void *const *mats,
                      const int64_t *mat_strides, const int64_t *ranks, int nmats, int64_t batch,
                      void *T, int64_t t_stride, void *workspace, void *stream) {
  int rc = check_plan(plan);
  if (rc) return rc;
  const int m = plan->order;
  if (nmats != m - 1) return fail(HK_EINVAL, "expected %d matrices, got %d", m - 1, nmats);
  if (!mats || !mat_strides || !ranks) return fail(HK_EINVAL, "NULL matrix arguments");
  if (batch < 0) return fail(HK_EINVAL, "negative batch");
  long long ncombo = 1;
  for (int i = 0; i < nmats; ++i) {
    if (ranks[i] < 1) return fail(HK_EINVAL, "matrix %d has no columns", i);
    ncombo *= ranks[i];
  }
  if (batch == 0) return HK_OK;
  if (!T || !workspace) return fail(HK_EINVAL, "NULL output or workspace");
  if (single_kind(h.dtype)) return fail(HK_EUNSUPPORTED, "times_matrices is complex128 only");
  if (plan->two_level)
    return tl_times_matrices(plan, h, mats, mat_strides, ranks, nmats, batch, T, t_stride,
                             workspace, stream, ncombo);
  const long long L = plan->L[0];
  double2 *ws = static_cast<double2 *>(workspace);
  long long used = 0;
  // spectrum of h (once per item)
  hk_operand hs = h;
  if (h.dtype != HK_SPEC) {
    double2 *sp = ws + used;
    used += batch * L;
    if ((rc = hk_spectrum(plan, h, batch, sp, nullptr, stream))) return rc;
    hs.data = sp;
    hs.batch_stride = L;
    hs.dtype = HK_SPEC;
  }
  // column spectra per distinct matrix
  std::vector<const double2 *> cspec(nmats, nullptr);
  for (int i = 0; i < nmats; ++i) {
    for (int k = 0; k < i; ++k) {
      if (mats[k] == mats[i] && mat_strides[k] == mat_strides[i] && ranks[k] == ranks[i] &&
          plan->sizes[k + 1] == plan->sizes[i + 1]) {
        cspec[i] = cspec[k];
        break;
      }
    }
    if (cspec[i]) continue;
    double2 *sp = ws + used;
    used += batch * ranks[i] * L;
    if ((rc = hk_vector_spectra(plan, i + 2, mats[i], mat_strides[i], ranks[i], batch, sp,
                                stream)))
      return rc;
    cspec[i] = sp;
  }
  // Column combinations, at most kMaxCombos per launch.  When two matrices
  // share their spectra (same pointer/stride/rank/length) only the
  // non-decreasing combinations are computed and the result is stored to
  // every permuted slot (for m = 3: T[:, j2, j3] and T[:, j3, j2]).
  std::vector<int> share(nmats);
  for (int i = 0; i < nmats; ++i) {
    share[i] = i;
    for (int k = 0; k < i; ++k)
      if (cspec[k] == cspec[i]) {
        share[i] = k;
        break;
      }
  }
  const bool sym2 = nmats == 2 && share[1] == 0;
  std::vector<int64_t> j(nmats, 0);
  struct Combo {
    int16_t col[hk::kMaxComboFac];
    int32_t out, out2;
  };
  std::vector<Combo> combos;
  for (long long c = 0; c < ncombo; ++c) {
    long long rem = c;
    for (int i = nmats - 1; i >= 0; --i) {
      j[i] = rem % ranks[i];
      rem /= ranks[i];
    }
    if (sym2 && j[1] < j[0]) continue;
    Combo cb{};
    for (int i = 0; i < nmats && i < hk::kMaxComboFac; ++i) cb.col[i] = (int16_t)j[i];
    cb.out = (int32_t)c;
    cb.out2 = (sym2 && j[1] != j[0]) ? (int32_t)(j[1] * ranks[1] + j[0]) : -1;
    combos.push_back(cb);
  }
  if (nmats > hk::kMaxComboFac) {
    // rare: more than 4 matrices -- one launch per combination
    for (auto &cb : combos) {
      long long rem = cb.out;
      for (int i = nmats - 1; i >= 0; --i) {
        j[i] = rem % ranks[i];
        rem /= ranks[i];
      }
      Args1D a = base_args(plan, batch);
      if ((rc = set_h(plan, hs, a))) return rc;
      a.nfac = 0;
      for (int i = 0; i < nmats; ++i) {
        Factor &f = a.fac[a.nfac++];
        f.ptr = cspec[i] + j[i] * L;
        f.bstride = ranks[i] * L;
        f.kind = hk::FK_SPEC;
        f.len = (int32_t)L;
        f.power = 1;
        f.estride = 1;
      }
      a.mode = hk::M_PARTIAL;
      a.out = static_cast<double2 *>(T) + cb.out;
      a.out_bstride = t_stride;
      a.out_estride = (int32_t)ncombo;
      a.out_len = (int32_t)plan->sizes[0];
      if ((rc = launch(plan, a, stream))) return rc;
    }
    return HK_OK;
  }
  for (size_t c0 = 0; c0 < combos.size(); c0 += hk::kMaxCombos) {
    const int nc = (int)std::min<size_t>(hk::kMaxCombos, combos.size() - c0);
    Args1D a = base_args(plan, batch * nc);
    a.nsub = nc;
    a.ncombo = nc;
    if ((rc = set_h(plan, hs, a))) return rc;
    a.nfac = nmats;
    for (int i = 0; i < nmats; ++i) {
      Factor &f = a.fac[i];
      f.ptr = cspec[i];
      f.bstride = ranks[i] * L;
      f.sstride = L;
      f.kind = hk::FK_SPEC;
      f.len = (int32_t)L;
      f.power = 1;
      f.estride = 1;
    }
    for (int c = 0; c < nc; ++c) {
      const Combo &cb = combos[c0 + c];
      for (int i = 0; i < hk::kMaxComboFac; ++i) a.combo_col[c][i] = cb.col[i];
      a.combo_out[c] = cb.out;
      a.combo_out2[c] = cb.out2;
    }
    a.mode = hk::M_PARTIAL;
    a.out = T;
    a.out_bstride = t_stride;
    a.out_estride = (int32_t)ncombo;
    a.out_len = (int32_t)plan->sizes[0];
    if ((rc = launch(plan, a, stream))) return rc;
  }
  return HK_OK;
}

}  // extern "C"
