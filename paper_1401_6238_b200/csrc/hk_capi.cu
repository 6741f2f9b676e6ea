// C ABI implementation (include/hankelfft_b200.h): plans, twiddle tables,
// validation, operand de-duplication and kernel dispatch.
#include <math.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <stdarg.h>
#include <stdio.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hankelfft_b200.h"
#include "hk_internal.h"

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

// Thread-major first-pass twiddles: T0[(j-1) * (L/R0) + b] = W_L^{j b}.
std::map<std::pair<int, long long>, double2 *> g_tw0;

int get_twiddles0(int device, long long L, int R0, const double2 **out) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(device, L);
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

int launch(const hk_plan *p, const Args1D &a, void *stream) {
  cudaError_t e = cudaErrorNotSupported;
  if (!g_force_generic) e = hk::launch_pp_1d((int)p->L[0], a, (cudaStream_t)stream);
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
  long long L = fft_len > 0 ? fft_len : hk::choose_len_1d(d);
  if (L < 0)
    return fail(HK_EUNSUPPORTED, "d_H = %lld exceeds the largest on-chip FFT length", d);
  if (L < d) return fail(HK_EINVAL, "fft_len %lld is shorter than d_H = %lld", L, d);
  if (!hk::supported_1d(L)) return fail(HK_EUNSUPPORTED, "FFT length %lld is not supported", L);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  hk_plan *p = new hk_plan();
  p->kind = 1;
  p->order = order;
  p->levels = 1;
  p->device = dev;
  p->sizes.assign(mode_sizes, mode_sizes + order);
  p->dof = {d};
  p->L = {L};
  int rc = get_twiddles(dev, L, &p->tw);
  const int r0 = hk::fast_first_radix(L);
  if (!rc && r0 > 0) rc = get_twiddles0(dev, L, r0, &p->tw0);
  if (rc) {
    delete p;
    return rc;
  }
  *plan = p;
  return HK_OK;
}

int hk_plan_create_block(hk_plan **plan, int order, int levels, const int64_t *level_shapes,
                         const int64_t *fft_lens) {
  (void)order;
  (void)levels;
  (void)level_shapes;
  (void)fft_lens;
  if (plan) *plan = nullptr;
  return fail(HK_EUNSUPPORTED, "block plans are not built yet");
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

size_t hk_workspace_bytes(const hk_plan *plan, int64_t batch) {
  (void)plan;
  (void)batch;
  return 0;
}

int hk_spectrum(const hk_plan *plan, hk_operand h, int64_t batch, void *spec, void *workspace,
                void *stream) {
  (void)workspace;
  int rc = check_plan(plan);
  if (rc) return rc;
  if (batch < 0) return fail(HK_EINVAL, "negative batch");
  if (batch == 0) return HK_OK;
  if (h.dtype == HK_SPEC) return fail(HK_EINVAL, "h is already a spectrum");
  if (!spec) return fail(HK_EINVAL, "spec is NULL");
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
  Args1D a = base_args(plan, batch);
  if ((rc = set_h(plan, h, a))) return rc;
  if ((rc = set_vectors(plan, xs, nx, 1, a))) return rc;
  a.mode = hk::M_PARTIAL;
  a.out = y;
  a.out_bstride = y_stride;
  a.out_len = (int32_t)plan->sizes[0];
  return launch(plan, a, stream);
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
  Args1D a = base_args(plan, batch);
  if ((rc = set_h(plan, h, a))) return rc;
  if ((rc = set_vectors(plan, xs, nx, 0, a))) return rc;
  a.mode = hk::M_FULL;
  a.out = alpha;
  a.out_bstride = 1;
  return launch(plan, a, stream);
}

int hk_vector_spectra(const hk_plan *plan, int mode, const void *mats, int64_t mat_stride,
                      int64_t ncols, int64_t batch, void *spec, void *stream) {
  int rc = check_plan(plan);
  if (rc) return rc;
  if (mode < 1 || mode > plan->order) return fail(HK_EINVAL, "mode %d out of range", mode);
  if (ncols < 1 || batch < 0) return fail(HK_EINVAL, "bad ncols/batch");
  if (batch == 0) return HK_OK;
  if (!mats || !spec) return fail(HK_EINVAL, "NULL matrix or spectrum pointer");
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
  // one launch per column combination
  std::vector<int64_t> j(nmats, 0);
  for (long long c = 0; c < ncombo; ++c) {
    long long rem = c;
    for (int i = nmats - 1; i >= 0; --i) {
      j[i] = rem % ranks[i];
      rem /= ranks[i];
    }
    Args1D a = base_args(plan, batch);
    if ((rc = set_h(plan, hs, a))) return rc;
    a.nfac = 0;
    for (int i = 0; i < nmats; ++i) {
      const double2 *ptr = cspec[i] + j[i] * L;
      bool merged = false;
      for (int f = 0; f < a.nfac; ++f) {
        if (a.fac[f].ptr == ptr) {
          a.fac[f].power += 1;
          merged = true;
          break;
        }
      }
      if (merged) continue;
      Factor &f = a.fac[a.nfac++];
      f.ptr = ptr;
      f.bstride = ranks[i] * L;
      f.sstride = 0;
      f.kind = hk::FK_SPEC;
      f.len = (int32_t)L;
      f.power = 1;
      f.estride = 1;
    }
    a.mode = hk::M_PARTIAL;
    a.out = static_cast<double2 *>(T) + c;
    a.out_bstride = t_stride;
    a.out_estride = (int32_t)ncombo;
    a.out_len = (int32_t)plan->sizes[0];
    if ((rc = launch(plan, a, stream))) return rc;
  }
  return HK_OK;
}

}  // extern "C"
