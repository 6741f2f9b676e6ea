// Fast-kernel instantiations for L = 192, 384, 512, 1024, 2048.
#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_small(int L, const Args1D &a, cudaStream_t stream, int maxlen, int outl) {
  switch (L) {
    case 192: {  // BHHB rows (cfg4): x rows carry n << 192 entries, outputs n_1 << 192
      using PL = Plan1D<192, 12, 12, 16>;
      const int s0 = PL::stride(0);
      return fast::Pruned<PL, 4, 6, 12>::launch(a, stream, (maxlen + s0 - 1) / s0,
                                                (outl + s0 - 1) / s0);
    }
    case 384: {
      using PL = Plan1D<384, 24, 24, 16>;
      const int s0 = PL::stride(0);
      return fast::Pruned<PL, 8, 12, 24>::launch(a, stream, (maxlen + s0 - 1) / s0,
                                                 (outl + s0 - 1) / s0);
    }
    case 2048:
      return fast::launch_variant<Plan1D<2048, 128, 8, 16, 16>, 8, 8>(a, stream);
    case 1024:
      return fast::launch_variant<Plan1D<1024, 64, 4, 16, 16>, 4, 4>(a, stream);
    case 512:
      return fast::launch_variant<Plan1D<512, 32, 2, 16, 16>, 2, 2>(a, stream);
    default:
      return cudaErrorNotSupported;
  }
}

}  // namespace hk
