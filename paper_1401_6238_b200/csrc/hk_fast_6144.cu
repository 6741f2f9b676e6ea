// Fast-kernel instantiations for L = 6144 (radix 24 x 16 x 16; cfg5).
#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_6144(const Args1D &a, cudaStream_t stream, int maxlen, int outl) {
  using PL = Plan1D<6144, 384, 24, 16, 16>;
  const int s0 = PL::stride(0);
  return fast::Pruned<PL, 8, 12, 24>::launch(a, stream, (maxlen + s0 - 1) / s0,
                                             (outl + s0 - 1) / s0);
}

}  // namespace hk
