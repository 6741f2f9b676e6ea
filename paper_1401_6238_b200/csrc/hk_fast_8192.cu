// Fast-kernel instantiation for L = 8192 (radix 2 x 16^3; cfg3 rows).
#include "hk_fast1d.cuh"

namespace hk {

cudaError_t launch_fast_8192(const Args1D &a, cudaStream_t stream) {
  return fast::launch_variant<Plan1D<8192, 512, 2, 16, 16, 16>, 2, 2>(a, stream);
}

}  // namespace hk
