// Two-level (large-L 1D four-step / 2D block) kernels: argument structs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {
namespace large {

// ST_A_PAIR: real h (in) and real x (in2) packed as z = h + i x, ONE forward
// column DFT, split by conjugate symmetry into the stage-A outputs of h
// (inverse, scaled, -> out) and of x (forward, -> out2).
enum ColStage : int { ST_A_FWD = 0, ST_A_INV = 1, ST_C = 2, ST_A_PAIR = 3 };

// An operand viewed as an L1 x L2 array; element (n1, n2) of item b sits at
// ptr + b*item_stride + n1*s1 + n2*s2 (elements).  Valid iff
//   1D (len >= 0): n2 + L2*n1 < len      2D (len < 0): n1 < e1 && n2 < e2
struct Op2 {
  const void *ptr;
  long long item_stride;
  long long s1, s2;
  long long len;
  int32_t e1, e2;
  int32_t kind;  // FK_C128 | FK_F64
  int32_t pad;
  double scale;
};

struct Out2 {
  void *ptr;
  long long item_stride;
  long long s1, s2;
  long long len;
  int32_t e1, e2;
};

struct ColArgs {
  Op2 in;
  Out2 out;
  Op2 in2;    // ST_A_PAIR only: the real vector x
  Out2 out2;  // ST_A_PAIR only: stage-A output of x
  int32_t L1, L2;
  int32_t twiddle;       // 1: four-step twiddle W_L^{n2 k1} (1D mode); 0: 2D mode
  int32_t in_n1_fast;    // tile-load order: 1 when the operand is contiguous along n1
  long long L;           // L1 * L2
  const double2 *thi;    // W_L^{q*4096}
  const double2 *tlo;    // W_L^{r}, r < 4096
  const double2 *ctw;    // column plan table W_L1^e
  const double2 *ctw0;   // column plan first-pass table
  // ST_C of a Hermitian spectral product (real h and x, 1D four-step): only
  // rows k1 <= L1/2 of the row-stage output exist; row L1-k1 is synthesised
  // as conj(W_L2^{m2} Q(k1, m2)) on load.
  int32_t half;
};

}  // namespace large

namespace bhhb {
// Fused BHHB product (hk_bhhb_fused.cu): one item per CTA, everything on chip.
struct Args {
  const double2 *h;  // (batch, din, dout) row-major: H[a][c] at a*dout + c
  long long h_bstride;
  const double2 *x;  // (batch, n*N) F-order: X[i][j] at i + n*j
  long long x_bstride;
  double2 *y;        // (batch, n*N) F-order
  long long y_bstride;
  long long batch;
  int din, dout, n, N, power;
  const double2 *tw48, *tw192;  // W_48^e, W_192^e
  double scale;                 // 1 / 192^2
};
}  // namespace bhhb
cudaError_t launch_bhhb_fused(const bhhb::Args &a, cudaStream_t stream);

bool supported_col_len(long long L1);
bool tma_col_len(long long L1);  // column lengths of the TMA column kernel
cudaError_t launch_cols(int stage, const large::ColArgs &a, long long items, int ncols,
                        cudaStream_t stream);
// TMA-fed column passes (hk_cols_tma.cu); cudaErrorNotSupported outside their shapes
cudaError_t launch_cols_tma(int stage, const large::ColArgs &a, long long items, int ncols,
                            cudaStream_t stream);
cudaError_t launch_rowsum(const double2 *part, long long rows, double2 *out, long long n,
                          cudaStream_t stream);

}  // namespace hk
