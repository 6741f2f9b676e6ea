// Fast-kernel instantiations for L = 4096 (radix 16^3; see hk_fast1d.cuh).
#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_4096(const Args1D &a, cudaStream_t stream, int maxlen, int outl) {
  using PL = Plan1D<4096, 256, 16, 16, 16>;
  const int s0 = PL::stride(0);
  return fast::Pruned<PL, 4, 8, 16>::launch(a, stream, (maxlen + s0 - 1) / s0,
                                            (outl + s0 - 1) / s0);
}

}  // namespace hk
