// K1 / K2: fused batched 1D Hankel tensor products, one FFT length per
// template instance, a group of T threads per product (G products per CTA).
//
// Per product b (reference hankel.py:140-154 via the anti-circulant
// embedding, hankel.py:42-71):
//   acc = ifft(h~)                       -- or the cached spectrum
//   acc *= fft(x~_f)^{power_f}           -- one transform per DISTINCT vector
//   partial: y = fft(acc)[:n_1]          -- transposed network, natural order out
//   full:    alpha = sum(acc)            -- fixed-order deterministic reduction
// The zero padding to L and the truncation to n_1 never touch memory: loads
// beyond len return 0, stores beyond out_len are skipped.
#include <atomic>

#include "hk_fft1d.cuh"
#include "hk_internal.h"
#include "hk_tmem.cuh"

namespace hk {

__device__ __forceinline__ long long item_off(long long bstride, long long sstride, long long ob,
                                              long long os) {
  return ob * bstride + os * sstride;
}

__device__ __forceinline__ cplx load_factor(const Factor &f, long long off, int pos,
                                            double scale) {
  if (pos >= f.len) return make_double2(0.0, 0.0);
  const long long k = (long long)pos * f.estride;
  if (f.kind == FK_F64) {
    const double *p = static_cast<const double *>(f.ptr) + off;
    return make_double2(__ldg(p + k) * scale, 0.0);
  }
  const cplx *p = static_cast<const cplx *>(f.ptr) + off;
  cplx v = __ldg(p + k);
  return make_double2(v.x * scale, v.y * scale);
}

// The accumulator acc = ifft(h) .* prod X lives in TMEM (4 x 32-bit columns per
// complex value, warp w on lanes 32*(w%4).. and slab w/4) whenever every
// thread holds a multiple of 4 values, so only one length-L working set is in
// registers while the next vector transform runs (with acc and w both in
// registers the kernel needed 255 registers and still spilled 80-530 bytes).
template <class PL>
struct GenTr {
  static constexpr bool tmem = PL::V % 4 == 0;
  static constexpr int warps = PL::CTA / 32;
  static constexpr int slabs = (warps + 3) / 4;
  static constexpr int need = slabs * 4 * PL::V;
  static constexpr int cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128
                              : need <= 256 ? 256 : 512;
  static_assert(!tmem || need <= 512, "accumulator does not fit in TMEM");
};

template <class PL>
__global__ void __launch_bounds__(PL::CTA, 1) k_hankel_1d(const __grid_constant__ Args1D a) {
  using Tr = GenTr<PL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplx *smem = reinterpret_cast<cplx *>(smem_raw);
  constexpr int T = PL::T;
  constexpr int V = PL::V;
  const int g = threadIdx.x / T;
  const int t = threadIdx.x - g * T;
  const int warp = threadIdx.x >> 5;
  long long b = (long long)blockIdx.x * PL::G + g;
  const bool active = b < a.batch;
  if (!active) b = a.batch - 1;  // idle groups shadow a valid item; their stores are masked
  long long ob, os;
  split_item(b, a.nsub, ob, os);
  cplx *sbuf = smem + (PL::P > 1 ? g * PL::L : 0);
  const cplx *__restrict__ tw = a.tw;
  uint32_t tmy = 0;
  if constexpr (Tr::tmem) {
    if (warp == 0) tmem_alloc<Tr::cols>(&tmem_slot);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tmy = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 4 * V);
  }

  cplx acc[Tr::tmem ? 1 : V];
  cplx w[V];
  auto acc_put = [&](cplx(&v)[V]) {
    if constexpr (Tr::tmem) {
#pragma unroll
      for (int c = 0; c < V / 4; ++c) tmem_st4(tmy + 16 * c, &v[4 * c]);
      tmem_wait_st();
    } else {
#pragma unroll
      for (int r = 0; r < V; ++r) acc[r] = v[r];
    }
  };
  if (a.mode != M_SPEC_F) {
    if (a.h.kind == FK_SPEC) {
      const cplx *sp = static_cast<const cplx *>(a.h.ptr) + item_off(a.h.bstride, a.h.sstride, ob, os);
#pragma unroll
      for (int r = 0; r < V; ++r) w[r] = __ldg(sp + r * T + t);
    } else {
      const Factor &hf = a.h;
      const double sc = a.scale;
      const long long off = item_off(hf.bstride, hf.sstride, ob, os);
      fft_dif<PL, true>(sbuf, t, tw, [&](int pos) { return load_factor(hf, off, pos, sc); }, w);
    }
    acc_put(w);
  }

  for (int f = 0; f < a.nfac; ++f) {
    const Factor &fa = a.fac[f];
    const long long off =
        ob * fa.bstride + (a.ncombo ? (long long)a.combo_col[os][f] : os) * fa.sstride;
    if (fa.kind == FK_SPEC) {
      const cplx *sp = static_cast<const cplx *>(fa.ptr) + off;
#pragma unroll
      for (int r = 0; r < V; ++r) w[r] = __ldg(sp + r * T + t);
    } else {
      fft_dif<PL, false>(sbuf, t, tw, [&](int pos) { return load_factor(fa, off, pos, 1.0); }, w);
    }
    if (a.mode == M_SPEC_F) {
      acc_put(w);
    } else if constexpr (Tr::tmem) {
#pragma unroll
      for (int c = 0; c < V / 4; ++c) {
        cplx q[4];
        tmem_ld4(tmy + 16 * c, q);
        for (int k = 0; k < fa.power; ++k) {
#pragma unroll
          for (int e = 0; e < 4; ++e) q[e] = cmul(q[e], w[4 * c + e]);
        }
        tmem_st4(tmy + 16 * c, q);
      }
      tmem_wait_st();
    } else {
      for (int k = 0; k < fa.power; ++k) {
#pragma unroll
        for (int r = 0; r < V; ++r) acc[r] = cmul(acc[r], w[r]);
      }
    }
  }
  // final: acc -> registers (w)
  if constexpr (Tr::tmem) {
#pragma unroll
    for (int c = 0; c < V / 4; ++c) tmem_ld4(tmy + 16 * c, &w[4 * c]);
  } else {
#pragma unroll
    for (int r = 0; r < V; ++r) w[r] = acc[r];
  }

  cplx *out = static_cast<cplx *>(a.out) + ob * a.out_bstride +
              (a.ncombo ? (long long)a.combo_out[os] : os * a.out_sstride);
  cplx *out2 = (a.ncombo && a.combo_out2[os] >= 0)
                   ? static_cast<cplx *>(a.out) + ob * a.out_bstride + a.combo_out2[os]
                   : nullptr;
  if (a.mode == M_PARTIAL) {
    const int n1 = a.out_len;
    const long long es = a.out_estride;
    fft_dit_final<PL>(sbuf, t, tw, w, [&](int pos, cplx v) {
      if (active && pos < n1) {
        out[pos * es] = v;
        if (out2) out2[pos * es] = v;
      }
    });
  } else if (a.mode == M_FULL) {
    cplx s = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < V; ++r) s = cadd(s, w[r]);
    // deterministic: per-thread partials in smem, summed in thread order
    __syncthreads();
    cplx *red = smem + g * T;  // G*T <= G*L slots
    red[t] = s;
    __syncthreads();
    if (t == 0 && active) {
      cplx tot = make_double2(0.0, 0.0);
      for (int k = 0; k < T; ++k) tot = cadd(tot, red[k]);
      out[0] = tot;
    }
  } else {
    if (active) {
#pragma unroll
      for (int r = 0; r < V; ++r) out[r * T + t] = w[r];
    }
  }
  if constexpr (Tr::tmem) {
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc<Tr::cols>(tmem_slot);
    }
  }
}

template <class PL>
static cudaError_t launch_plan(const Args1D &a, cudaStream_t stream) {
  // M_FULL reuses smem for T partial sums; make sure it exists when P == 1.
  int smem = PL::SMEM_BYTES;
  const int red_bytes = PL::G * PL::T * (int)sizeof(cplx);
  if (smem < red_bytes) smem = red_bytes;
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_1d<PL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  const long long grid = (a.batch + PL::G - 1) / PL::G;
  if (grid <= 0) return cudaSuccess;
  k_hankel_1d<PL><<<(unsigned)grid, PL::CTA, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_1d(int L, const Args1D &a, cudaStream_t stream) {
  switch (L) {
#define HK_CASE(len, ...) \
  case len:              \
    return launch_plan<__VA_ARGS__>(a, stream);
    HK_PLAN_LIST(HK_CASE)
#undef HK_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

bool supported_1d(long long L) {
  switch (L) {
#define HK_CASE(len, ...) \
  case len:              \
    return true;
    HK_PLAN_LIST(HK_CASE)
#undef HK_CASE
    default:
      return false;
  }
}

long long choose_len_1d(long long d) {
  long long best = -1;
#define HK_CASE(len, ...) \
  if (len >= d && (best < 0 || len < best)) best = len;
  HK_PLAN_LIST(HK_CASE)
#undef HK_CASE
  return best;
}

}  // namespace hk
