// Internal (non-exported) declarations shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {

// How one factor of the spectral product is supplied.
enum FactorKind : int32_t {
  FK_C128 = 0,  // complex128 vector, zero-padded to L and transformed in-kernel
  FK_F64 = 1,   // float64 vector (imaginary part zero), zero-padded and transformed
  FK_SPEC = 2,  // precomputed spectrum in the kernel's internal layout (length L)
  FK_C64 = 3,   // complex64 vector (complex64 variant, hk_c64.cu)
  FK_F32 = 4,   // float32 vector (complex64 variant)
};

enum Mode1D : int32_t {
  M_PARTIAL = 0,  // y = fft(S .* prod X)[:out_len]           (hankel.py:42-45,140-147)
  M_FULL = 1,     // alpha = sum(S .* prod X)                 (hankel.py:47-59,149-154)
  M_SPEC_H = 2,   // write S = ifft(h) in internal layout     (hankel.py:37-40)
  M_SPEC_F = 3,   // write X = fft(fac[0]) in internal layout (column spectra, K5)
};

// Batch index q of a launch splits as q = b * nsub + s; item (b, s) of a
// factor starts at ptr + b * bstride + s * sstride elements, and vector entry
// k sits at + k * estride.
struct Factor {
  const void *ptr;
  long long bstride;
  long long sstride;
  int32_t len;       // nonzero prefix length; positions >= len are zero
  int32_t power;     // multiplicity in the product
  int32_t kind;      // FactorKind
  int32_t estride;   // element stride inside one vector (1 = contiguous)
};

constexpr int kMaxFactors = 32;
constexpr int kMaxCombos = 64;     // column combinations per times_matrices launch
constexpr int kMaxComboFac = 4;    // distinct matrix factors addressed by the table

struct Args1D {
  Factor h;                 // generating vector (inverse transform) or cached spectrum
  Factor fac[kMaxFactors];  // distinct vector factors
  int32_t nfac;
  int32_t mode;
  void *out;                // complex128 output, same (b, s) addressing as factors
  long long out_bstride;
  long long out_sstride;
  int32_t out_len;          // number of outputs kept (n_1) for M_PARTIAL
  int32_t out_estride;      // element stride of y
  long long batch;          // total launch items (= outer * nsub)
  long long nsub;           // >= 1
  const double2 *tw;        // W_L^e, e in [0, L)
  const double2 *tw0;       // thread-major first-pass table (fast path), may be NULL
  const double2 *tw1;       // W_{L/R0}^e, e in [0, L/R0): passes >= 1 of the fast path, may be NULL
  const float2 *twf;        // complex64 variant: W_L^e in single precision
  double scale;             // 1/L for the inverse transform
  int32_t prefetch;         // fast path: L2-prefetch the next block's operands
  // times_matrices combo table (ncombo > 0): launch item q = b * ncombo + c;
  // factor f of combo c starts at ptr + b*bstride + combo_col[c][f]*sstride,
  // the output at out + b*out_bstride + combo_out[c] (and combo_out2[c] >= 0,
  // the mirrored slot of a symmetric product).
  int32_t diag;     // diagnostics switch (0 in production)
  int32_t ncombo;
  int16_t combo_col[kMaxCombos][kMaxComboFac];
  int32_t combo_out[kMaxCombos];
  int32_t combo_out2[kMaxCombos];
};

#ifdef __CUDACC__
// Launch item b = ob * nsub + os.  Plain batches have nsub == 1; otherwise a
// 32-bit division when both fit (always, in practice) instead of the emulated
// 64-bit one (~100 dependent instructions per product and thread).
__device__ __forceinline__ void split_item(long long b, long long nsub, long long &ob,
                                           long long &os) {
  if (nsub == 1) {
    ob = b;
    os = 0;
  } else if ((((unsigned long long)b | (unsigned long long)nsub) >> 32) == 0) {
    const unsigned q = (unsigned)b / (unsigned)nsub;
    ob = q;
    os = (unsigned)b - q * (unsigned)nsub;
  } else {
    ob = b / nsub;
    os = b - ob * nsub;
  }
}
#endif

// Launch the fused 1D kernel for FFT length L (must be supported).
cudaError_t launch_1d(int L, const Args1D &a, cudaStream_t stream);
bool supported_1d(long long L);
// Fast path (hk_fast1d.cu): cudaErrorNotSupported if not applicable.
cudaError_t launch_fast_1d(int L, const Args1D &a, cudaStream_t stream);
int fast_first_radix(long long L);  // R_0 of the fast plan, 0 if none
// Producer/consumer TMA variant (hk_pp1d.cu) for batched H x^{m-1}.
cudaError_t launch_pp_1d(int L, const Args1D &a, cudaStream_t stream);
// complex64 / float32 variant (hk_c64.cu): M_PARTIAL and M_FULL, on-chip L.
cudaError_t launch_c64_1d(int L, const Args1D &a, cudaStream_t stream);
// Latency kernel (hk_small.cu) for a few small direct products.
cudaError_t launch_small_1d(int L, const Args1D &a, cudaStream_t stream);

long long choose_len_1d(long long d);  // smallest supported on-chip L >= d, or -1

}  // namespace hk
