// Fast-path dispatch (the kernels are instantiated per length in
// hk_fast_*.cu, see hk_fast1d.cuh); returns cudaErrorNotSupported when L has
// no fast variant or the request needs a mode the fast kernel does not
// implement.
#include <stdlib.h>

#include "hk_fast1d.cuh"

namespace hk {

int fast_first_radix(long long L) {
  switch (L) {
    case 192: return 12;
    case 384: return 24;
    case 4096: return 16;
    case 6144: return 24;
    case 2048: return 8;
    case 1024: return 4;
    case 512: return 2;
    case 256: return 16;
    case 8192: return 2;
    default: return 0;
  }
}

// Staged operand path: raw h and first vector factor, product modes only.
static bool stageable(const Args1D &a) {
  static const bool off = getenv("HK_NO_STAGE") != nullptr;
  if (off || (a.mode != M_PARTIAL && a.mode != M_FULL) || a.nfac < 1) return false;
  const auto raw = [](const Factor &f) { return f.kind == FK_C128 || f.kind == FK_F64; };
  return raw(a.h) && raw(a.fac[0]);
}

cudaError_t launch_fast_1d(int L, const Args1D &a, cudaStream_t stream) {
  if (!a.tw0) return cudaErrorNotSupported;
  int maxlen = 1;
  for (int f = 0; f < a.nfac; ++f)
    if (a.fac[f].kind != FK_SPEC && a.fac[f].len > maxlen) maxlen = a.fac[f].len;
  const int outl = a.mode == M_PARTIAL ? a.out_len : L;
  switch (L) {
    case 4096: return launch_fast_4096(a, stream, maxlen, outl);
    case 6144: return launch_fast_6144(a, stream, maxlen, outl);
    case 256: return launch_fast_256(a, stream, maxlen, outl, stageable(a));
    case 192:
    case 384:
    case 512:
    case 1024:
    case 2048: return launch_fast_small(L, a, stream, maxlen, outl);
    case 8192: return launch_fast_8192(a, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace hk
