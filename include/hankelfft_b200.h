/*
 * hankelfft_b200 -- C ABI of the B200-native fast Hankel tensor-vector product.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `hankelfft` 0.1.0 (arXiv 1401.6238; /root/reference/pkg/src/hankelfft).  The
 * reference has no FFI of its own (it is pure Python over numpy's pocketfft);
 * each entry point below names the Python interface it replaces, and
 * INTEGRATION.md shows the ctypes binding a maintainer would add.
 *
 * Conventions
 *  - Plain C: opaque plan handles, raw DEVICE pointers, element counts, and a
 *    cudaStream_t passed as `void *` (NULL = legacy default stream).
 *  - Complex data is interleaved complex128 (numpy / torch layout).
 *  - All launches are asynchronous on the given stream; nothing synchronises.
 *  - Return 0 on success or a negative HK_E* code; hk_last_error() gives a
 *    thread-local message.  No C++ exception crosses this boundary.
 *  - Plans are immutable after creation and may be used concurrently from
 *    several host threads / streams (reference SPEC.md "Concurrency Model").
 *  - Results are deterministic: no atomics, fixed-order reductions.
 */
#ifndef HANKELFFT_B200_H
#define HANKELFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HK_OK 0
#define HK_EINVAL (-1)      /* invalid argument (shape, length, count)        */
#define HK_ECUDA (-2)       /* CUDA runtime / launch failure                  */
#define HK_ENOMEM (-3)      /* device allocation failure                      */
#define HK_EUNSUPPORTED (-4) /* valid request outside what this build covers  */

/* operand element types */
#define HK_C128 0 /* complex128 vector / matrix                                  */
#define HK_F64 1  /* float64 (real) vector; promoted to complex like core.as_complex */
#define HK_SPEC 2 /* spectrum previously produced by hk_spectrum / hk_vector_spectra */
/* Single-precision variant (north_star: rel. error <= 1e-4).  A product whose
 * h is HK_C64 / HK_F32 takes only HK_C64 / HK_F32 vectors, computes in FP32 and
 * writes complex64 y / alpha; on-chip plans (L <= 8192), hk_tvp_partial and
 * hk_tvp_full only.  The reference itself is complex128-only (core.py:21-22). */
#define HK_C64 3  /* complex64 vector                                             */
#define HK_F32 4  /* float32 (real) vector, promoted to complex64                 */

/* One operand of a product: a batch of vectors (or spectra) in device memory.
 * Item b of the batch starts at data + b * batch_stride elements. */
typedef struct hk_operand {
  const void *data;
  int64_t batch_stride;
  int32_t dtype; /* HK_C128 | HK_F64 | HK_SPEC | HK_C64 | HK_F32 */
  int32_t reserved;
} hk_operand;

typedef struct hk_plan hk_plan;

/* Library version (major*10000 + minor*100 + patch). */
int hk_version(void);

/* Thread-local description of the last error returned on this thread. */
const char *hk_last_error(void);

/* Plan for the order-m Hankel tensor with mode sizes n_1..n_m (the
 * `HankelTensor(shape, h)` of hankel.py:89-119; d_H = sum(n_p) - m + 1,
 * hankel.py:108-111).  fft_len = 0 picks the smallest supported length
 * L >= d_H; any L >= d_H gives the identical product (no index sum wraps).
 * Creates the twiddle tables on the CURRENT CUDA device; use the plan only on
 * that device.  Replaces the `_embedding` / `embed()` plan objects
 * (hankel.py:121-128) and pocketfft's per-length plan cache. */
int hk_plan_create_hankel(hk_plan **plan, int order, const int64_t *mode_sizes, int64_t fft_len);

/* Plan for a level-k block Hankel tensor (BhhbTensor for k = 2, block.py:92-175;
 * LevelKHankelTensor, block.py:178-250).  level_shapes is k x m row-major:
 * level_shapes[l*m + p] = size of mode p at level l (level 0 innermost).
 * fft_lens (k entries, or NULL for auto) are the per-level transform lengths. */
int hk_plan_create_block(hk_plan **plan, int order, int levels, const int64_t *level_shapes,
                         const int64_t *fft_lens);

int hk_plan_destroy(hk_plan *plan);

/* Per-level FFT length of the plan (level 0 for 1D plans). */
int64_t hk_plan_fft_len(const hk_plan *plan, int level);

/* Number of complex128 elements of one cached spectrum (= prod of fft lens). */
int64_t hk_plan_spectrum_len(const hk_plan *plan);

/* Device workspace (bytes) needed by hk_tvp_partial / hk_tvp_full /
 * hk_times_matrices for `batch` items; 0 for on-chip (single-kernel) plans. */
size_t hk_workspace_bytes(const hk_plan *plan, int64_t batch);

/* S = ifft(h~) for a batch of generating vectors, written in the library's
 * internal spectrum layout (hk_plan_spectrum_len elements per item,
 * consecutive items).  Replaces the cached `spectrum` of the embedding
 * (hankel.py:37-40, block.py:125-127).  h.dtype: HK_C128 or HK_F64. */
int hk_spectrum(const hk_plan *plan, hk_operand h, int64_t batch, void *spec, void *workspace,
                void *stream);

/* y = H x_2 ... x_m for a batch: HankelTensor.tvp_partial (hankel.py:140-147),
 * i.e. fft(ifft(h~) .* fft(x~_2) .* ... .* fft(x~_m))[:n_1].
 * h may be a raw generating vector (HK_C128 / HK_F64) or a cached spectrum
 * (HK_SPEC).  xs has order-1 operands, xs[p] for mode p+2 (length n_{p+2}).
 * Operands with identical (data, batch_stride, dtype) are transformed once and
 * raised to their multiplicity (H x^{m-1} costs one vector transform).
 * y: complex128 (complex64 for HK_C64/HK_F32 operands), item b at
 * y + b * y_stride elements, n_1 values. */
int hk_tvp_partial(const hk_plan *plan, hk_operand h, const hk_operand *xs, int nx,
                   int64_t batch, void *y, int64_t y_stride, void *workspace, void *stream);

/* Latency form of hk_tvp_partial for ONE product with numpy-side operands
 * (the call behind HankelTensor.tvp_partial, hankel.py:140-147, when the
 * caller holds host arrays): copies `in_elems` complex128 values from pinned
 * host memory `host_in` to device scratch `dev_in`, runs the product with
 * vector p read from dev_in + x_offsets[p] (identical offsets = same vector),
 * copies the n_1 outputs to pinned host memory `host_y` and synchronises
 * `stream`.  h is a device operand (HK_C128 / HK_F64 / HK_SPEC).  One call
 * replaces two copies, a launch and a sync issued separately from Python. */
int hk_tvp_partial_host(const hk_plan *plan, hk_operand h, const void *host_in, int64_t in_elems,
                        const int64_t *x_offsets, int nx, void *dev_in, void *dev_y,
                        void *host_y, void *stream);

/* alpha = H x_1 ... x_m (unconjugated): HankelTensor.tvp_full
 * (hankel.py:149-154) / AntiCirculantTensor.tvp_full (hankel.py:47-59).
 * xs has `order` operands.  alpha: complex128[batch] (stride 1); complex64
 * for HK_C64/HK_F32 operands. */
int hk_tvp_full(const hk_plan *plan, hk_operand h, const hk_operand *xs, int nx, int64_t batch,
                void *alpha, void *workspace, void *stream);

/* Column spectra fft(m~_j) of the columns of a row-major (rows x ncols)
 * complex128 matrix per batch item (item stride `mat_stride` elements), for
 * mode `mode` (1-based, 2..m) of the plan.  Output: ncols spectra per item in
 * internal layout.  Building block of hk_times_matrices. */
int hk_vector_spectra(const hk_plan *plan, int mode, const void *mats, int64_t mat_stride,
                      int64_t ncols, int64_t batch, void *spec, void *stream);

/* T[:, j_2, ..., j_m] = H x_2 M_2[:, j_2] ... x_m M_m[:, j_m]: times_matrices
 * (hankel.py:174-194).  mats[p] is a row-major (n_{p+2} x ranks[p]) complex128
 * matrix per item (item stride mat_strides[p]); h as in hk_tvp_partial.
 * T: complex128 C-order (n_1, R_2, ..., R_m) per item, item stride t_stride.
 * Matrices passed with identical pointers/strides share their column spectra;
 * for m = 3 with mats[0] == mats[1] only the j_2 <= j_3 combinations are
 * transformed and mirrored.  workspace: hk_times_matrices_workspace_bytes(). */
size_t hk_times_matrices_workspace_bytes(const hk_plan *plan, const int64_t *ranks, int nmats,
                                         int64_t batch);

int hk_times_matrices(const hk_plan *plan, hk_operand h, const void *const *mats,
                      const int64_t *mat_strides, const int64_t *ranks, int nmats, int64_t batch,
                      void *T, int64_t t_stride, void *workspace, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HANKELFFT_B200_H */
