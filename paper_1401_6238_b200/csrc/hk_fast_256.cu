// Fast-kernel instantiations for L = 256 (BHHB rows padded to 256, cfg4:
// 64 nonzero x entries, 64 outputs), plain and with cp.async operand staging.
#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_256(const Args1D &a, cudaStream_t stream, int maxlen, int outl,
                            bool staged) {
  using PL = Plan1D<256, 16, 16, 16>;
  const int s0 = PL::stride(0);
  const int nz = (maxlen + s0 - 1) / s0, no = (outl + s0 - 1) / s0;
  if (staged)
    return fast::Pruned<fast::Regroup<PL, 8>, 4, 8, 16>::launch<true>(a, stream, nz, no);
  return fast::Pruned<PL, 4, 8, 16>::launch(a, stream, nz, no);
}

}  // namespace hk
