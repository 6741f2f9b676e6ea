// Fast-kernel instantiations for L = 256 (BHHB rows padded to 256, cfg4:
// 64 nonzero x entries, 64 outputs), plain and with cp.async operand staging.
#include <stdlib.h>

#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_256(const Args1D &a, cudaStream_t stream, int maxlen, int outl,
                            bool staged) {
  using PL = Plan1D<256, 16, 16, 16>;
  const int s0 = PL::stride(0);
  const int nz = (maxlen + s0 - 1) / s0, no = (outl + s0 - 1) / s0;
  if (staged) {
    // 6 products (3 warps) per CTA, 4 CTAs per SM: the per-item CTA barrier
    // that bounds warp drift spans 3 warps instead of 4 (B200, cfg4: G=6
    // 985 us, G=8 1050 us, G=4 1093 us, G=12 1168 us).  HK_G256=8: previous.
    static const bool g8 = getenv("HK_G256") && atoi(getenv("HK_G256")) == 8;
    if (g8) return fast::Pruned<fast::Regroup<PL, 8>, 4, 8, 16>::launch<true>(a, stream, nz, no);
    return fast::Pruned<fast::Regroup<PL, 6>, 4, 8, 16>::launch<true>(a, stream, nz, no);
  }
  return fast::Pruned<PL, 4, 8, 16>::launch(a, stream, nz, no);
}

}  // namespace hk
