// K0: latency kernel for a few small products (cfg1: one order-3 product,
// n = 100, L = 384; reference hankel.py:140-154 called once per request).
//
// With one product in flight the fused kernels of hk_fast1d.cu are bound by
// instruction fetch, not by math: their fully unrolled codelets execute
// ~60 KB of straight-line SASS once per launch, and a cold single-CTA launch
// waits on the instruction cache for most of its ~35 us (ncu: "no
// instruction" is the top stall).  This kernel keeps the code small and hot
// instead: one CTA per product, 256 threads, every array in shared memory,
// and a rolled mixed-radix Stockham loop (runtime radix 2/3/4/8, autosorting,
// natural order in and out), so each codelet's SASS is fetched once and
// re-executed by every stage and every thread.
//
//   1. stage conj(h~)/L and every distinct x~_f (zero-padded to L) in smem;
//   2. forward FFT of all 1 + nfac arrays together (one barrier per stage);
//   3. S = conj(FFT(conj(h~)/L)) = ifft(h~);  P = S .* prod_f X_f^{p_f}
//      (reference multiplication order, hankel.py:61-71);
//   4. M_FULL:    alpha = sum_k P_k (fixed-order tree: deterministic);
//      M_PARTIAL: y = FFT(P)[:n_1]  (hankel.py:42-45).
#include <stdio.h>

#include <atomic>

#include "hk_fastcore.cuh"

namespace hk {
namespace small {

constexpr int kThreads = 256;
constexpr int kMaxStages = 16;

struct Stages {
  int32_t L;
  int32_t n;
  int32_t r[kMaxStages];
};

// One Stockham butterfly: inputs j + r*L/R, twiddles W_{Ns R}^{r (j mod Ns)},
// outputs (j / Ns) * Ns * R + (j mod Ns) + r * Ns.
template <int R>
__device__ __forceinline__ void stockham(const cplx *__restrict__ in, cplx *__restrict__ out, int L,
                                         int Ns, int j, const cplx *__restrict__ tw) {
  cplx v[R];
  const int NR = L / R;
  const int k = j % Ns;
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = in[j + r * NR];
  if (Ns > 1) {
    const int step = (L / (Ns * R)) * k;  // W_L^{r * step} = W_{Ns R}^{r k}
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[r * step]));
  }
  Dft<R, false>::run(v);
  const int o = (j / Ns) * Ns * R + k;
#pragma unroll
  for (int r = 0; r < R; ++r) out[o + r * Ns] = v[r];
}

// Forward FFT of `na` contiguous length-L arrays, ping-ponging between the
// two buffer sets; returns the set holding the result.
__device__ __noinline__ cplx *fft_arrays(cplx *src, cplx *dst, int na, const Stages &st,
                                         const cplx *__restrict__ tw) {
  const int L = st.L;
  int Ns = 1;
  for (int s = 0; s < st.n; ++s) {
    const int R = st.r[s];
    const int per = L / R;
    for (int w = threadIdx.x; w < na * per; w += blockDim.x) {
      const int arr = w / per, j = w - arr * per;
      const cplx *in = src + arr * L;
      cplx *out = dst + arr * L;
      switch (R) {
        case 2: stockham<2>(in, out, L, Ns, j, tw); break;
        case 3: stockham<3>(in, out, L, Ns, j, tw); break;
        case 4: stockham<4>(in, out, L, Ns, j, tw); break;
        default: stockham<8>(in, out, L, Ns, j, tw); break;
      }
    }
    Ns *= R;
    cplx *t = src;
    src = dst;
    dst = t;
    __syncthreads();
  }
  return src;
}

__global__ void __launch_bounds__(kThreads) k_small(const __grid_constant__ Args1D a,
                                                    const __grid_constant__ Stages st) {
  extern __shared__ __align__(16) cplx sm[];
  __shared__ cplx red[kThreads];
  const int L = st.L;
  const int na = 1 + a.nfac;
  cplx *set0 = sm, *set1 = sm + na * L;
  for (long long q = blockIdx.x; q < a.batch; q += gridDim.x) {
    const long long ob = q / a.nsub, os = q - ob * a.nsub;
    // ---- 1. stage conj(h~)/L and the vectors
    const long long hoff = ob * a.h.bstride + os * a.h.sstride;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const cplx hv = fast::load_elem(a.h, hoff, i, a.scale);
      set0[i] = make_double2(hv.x, -hv.y);
    }
    for (int f = 0; f < a.nfac; ++f) {
      const Factor &fa = a.fac[f];
      const long long off = ob * fa.bstride + os * fa.sstride;
      for (int i = threadIdx.x; i < L; i += blockDim.x)
        set0[(1 + f) * L + i] = fast::load_elem(fa, off, i, 1.0);
    }
    __syncthreads();
    // ---- 2. all spectra at once
    cplx *spec = fft_arrays(set0, set1, na, st, a.tw);
    cplx *other = spec == set0 ? set1 : set0;
    // ---- 3. P = ifft(h~) .* prod X_f^{p_f}
    cplx part = make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      cplx acc = make_double2(spec[k].x, -spec[k].y);
      for (int f = 0; f < a.nfac; ++f) {
        const cplx xv = spec[(1 + f) * L + k];
        for (int p = 0; p < a.fac[f].power; ++p) acc = cmul(acc, xv);
      }
      if (a.mode == M_FULL)
        part = cadd(part, acc);
      else
        other[k] = acc;
    }
    if (a.mode == M_FULL) {
      // ---- 4a. alpha = sum_k P_k, fixed-order tree
      red[threadIdx.x] = part;
      __syncthreads();
      for (int w = kThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
      }
      if (threadIdx.x == 0) static_cast<cplx *>(a.out)[ob * a.out_bstride + os * a.out_sstride] = red[0];
      __syncthreads();
      continue;
    }
    __syncthreads();
    // ---- 4b. y = fft(P)[:n_1]
    const cplx *y = fft_arrays(other, spec, 1, st, a.tw);
    cplx *out = static_cast<cplx *>(a.out) + ob * a.out_bstride + os * a.out_sstride;
    for (int k = threadIdx.x; k < a.out_len; k += blockDim.x) out[(long long)k * a.out_estride] = y[k];
    __syncthreads();
  }
}

}  // namespace small

// Batches up to this size take the latency kernel (one CTA per product).
constexpr long long kSmallMaxBatch = 32;

// Latency path; cudaErrorNotSupported unless the request is a small batch of
// small direct products (no cached spectra, no combo tables).
cudaError_t launch_small_1d(int L, const Args1D &a, cudaStream_t stream) {
  if (getenv("HK_NO_SMALL")) return cudaErrorNotSupported;
  if (a.batch <= 0 || a.batch > kSmallMaxBatch || L < 2 || L > 4096 || !a.tw)
    return cudaErrorNotSupported;
  if (a.mode != M_PARTIAL && a.mode != M_FULL) return cudaErrorNotSupported;
  if (a.ncombo != 0 || a.nfac < 1 || a.nfac > 3 || a.h.kind == FK_SPEC) return cudaErrorNotSupported;
  for (int f = 0; f < a.nfac; ++f)
    if (a.fac[f].kind == FK_SPEC) return cudaErrorNotSupported;
  small::Stages st{};
  st.L = L;
  int rem = L;
  if (rem % 3 == 0) {
    st.r[st.n++] = 3;
    rem /= 3;
  }
  while (rem > 1) {
    const int r = rem % 8 == 0 ? 8 : (rem % 4 == 0 ? 4 : 2);
    if (rem % r != 0 || st.n >= small::kMaxStages) return cudaErrorNotSupported;
    st.r[st.n++] = r;
    rem /= r;
  }
  const int smem = 2 * (1 + a.nfac) * L * (int)sizeof(cplx);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(small::k_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  small::k_small<<<(unsigned)a.batch, small::kThreads, smem, stream>>>(a, st);
  return cudaGetLastError();
}

}  // namespace hk
