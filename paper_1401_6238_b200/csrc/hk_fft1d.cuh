// CTA-level mixed-radix FFT engine used by the fused Hankel product kernels.
//
// Length L = R_0 * R_1 * ... * R_{P-1}.  Positions use the in-place
// decimation-in-frequency layout: pass p combines the elements
// base + j * s_p (j < R_p, s_p = L / (R_0...R_p)) and multiplies output j by
// W_L^{j * lo * L / (s_p R_p)} with lo = base mod s_p.  After the last pass a
// thread owns V = L / T frequency samples in digit-reversed order, in
// registers.
//
// The product kernels exploit two facts:
//  * every spectrum in a product (ifft(h), fft(x_p)) is produced with the same
//    decomposition and thread mapping, so the pointwise product
//    ifft(h) .* prod fft(x_p) (reference hankel.py:61-71) is a register-only
//    operation on matching positions;
//  * the final forward FFT (hankel.py:45) is the transpose of the DIF network
//    (the DFT matrix is symmetric), so it consumes the digit-reversed
//    registers directly by running the passes in reverse order with the
//    twiddle applied before each butterfly, and emits natural-order output --
//    no reordering step at all.
// Passes exchange through shared memory with an XOR swizzle on 16-byte
// elements (bits 0-2 ^= bits 4-6) that keeps every 8-lane phase of a 128-bit
// access on distinct bank groups for the strides used here.
#pragma once

#include "hk_dft.cuh"

namespace hk {

template <int L_, int T_, int... Rs>
struct Plan1D {
  static constexpr int L = L_;
  static constexpr int T = T_;
  static constexpr int P = sizeof...(Rs);
  static constexpr int radix[P] = {Rs...};
  static constexpr int Rlast = radix[P - 1];
  static_assert((L / Rlast) % T == 0, "last pass must split evenly over the threads");
  static constexpr int V = L / T;  // values per thread after the last pass
  static constexpr int prod() {
    int r = 1;
    for (int q = 0; q < P; ++q) r *= radix[q];
    return r;
  }
  static_assert(prod() == L, "radices must multiply to L");
  static constexpr int stride(int p) {
    int s = L;
    for (int q = 0; q <= p; ++q) s /= radix[q];
    return s;
  }
  // independent products per CTA: as many as fit 256 threads, rounded so the
  // CTA is a whole number of warps (tcgen05 TMEM ops are warp-collective)
  static constexpr int pick_g() {
    if (T >= 256) return 1;
    for (int g = 256 / T; g > 1; --g)
      if ((g * T) % 32 == 0) return g;
    return 256 / T;
  }
  static constexpr int G = pick_g();
  static constexpr int CTA = G * T;
  static constexpr int SMEM_BYTES = (P > 1) ? G * L * (int)sizeof(cplx) : 16;
};

// Supported on-chip lengths.  Power-of-two lengths use radix-16 passes with one
// small leading radix; 3*2^k lengths put a radix-12/24/3/6 pass first.
#define HK_PLAN_LIST(X)                     \
  X(2, Plan1D<2, 1, 2>)                     \
  X(4, Plan1D<4, 1, 4>)                     \
  X(8, Plan1D<8, 1, 8>)                     \
  X(16, Plan1D<16, 1, 16>)                  \
  X(32, Plan1D<32, 2, 2, 16>)               \
  X(64, Plan1D<64, 4, 4, 16>)               \
  X(128, Plan1D<128, 8, 8, 16>)             \
  X(256, Plan1D<256, 16, 16, 16>)           \
  X(512, Plan1D<512, 32, 2, 16, 16>)        \
  X(1024, Plan1D<1024, 64, 4, 16, 16>)      \
  X(2048, Plan1D<2048, 128, 8, 16, 16>)     \
  X(4096, Plan1D<4096, 256, 16, 16, 16>)    \
  X(8192, Plan1D<8192, 512, 2, 16, 16, 16>) \
  X(12, Plan1D<12, 1, 12>)                  \
  X(24, Plan1D<24, 1, 24>)                  \
  X(48, Plan1D<48, 3, 3, 16>)               \
  X(96, Plan1D<96, 6, 6, 16>)               \
  X(192, Plan1D<192, 12, 12, 16>)           \
  X(384, Plan1D<384, 24, 24, 16>)           \
  X(768, Plan1D<768, 48, 3, 16, 16>)        \
  X(1536, Plan1D<1536, 96, 6, 16, 16>)      \
  X(3072, Plan1D<3072, 192, 12, 16, 16>)    \
  X(6144, Plan1D<6144, 384, 24, 16, 16>)

__device__ __forceinline__ int swz(int pos) { return pos ^ ((pos >> 4) & 7); }
// Swizzle by element size: 16-byte (complex128) elements as above; 8-byte
// (complex64) elements are served 16 lanes per phase, so the low 4 position
// bits are XORed with bits 4-7 (the last radix-16 pass reads 16 consecutive
// positions per thread at a 16-element lane stride).
template <class C>
__device__ __forceinline__ int swz_t(int pos) {
  if constexpr (sizeof(C) == 8)
    return pos ^ ((pos >> 4) & 15);
  else
    return swz(pos);
}

// One DIF pass.  load(pos) -> cplx ; store(i, j, pos, value).
template <class PL, int p, bool INV, class C, class Load, class Store>
__device__ __forceinline__ void dif_pass(int t, const C *__restrict__ tw, Load &&load,
                                         Store &&store) {
  constexpr int R = PL::radix[p];
  constexpr int s = PL::stride(p);
  constexpr int Lp = s * R;
  constexpr int NBUT = PL::L / R;
  constexpr int NB = (NBUT + PL::T - 1) / PL::T;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int beta = t + i * PL::T;
    if (NBUT % PL::T == 0 || beta < NBUT) {
      const int lo = beta % s;
      const int base = (beta / s) * Lp + lo;
      C a[R];
      sfor<R>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        a[j] = load(base + j * s);
      });
      Dft<R, INV>::run(a);
      if constexpr (p < PL::P - 1) {
        const int e1 = lo * (PL::L / Lp);
        sfor<R>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          if constexpr (j > 0) a[j] = cmul_dir<INV>(a[j], __ldg(&tw[j * e1]));
        });
      }
      sfor<R>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        store(i, j, base + j * s, a[j]);
      });
    }
  }
}

// One transposed (DIT) pass of the forward transform: twiddle, then butterfly.
// load(i, j, pos) -> cplx ; store(i, j, pos, value).
template <class PL, int p, class C, class Load, class Store>
__device__ __forceinline__ void dit_pass(int t, const C *__restrict__ tw, Load &&load,
                                         Store &&store) {
  constexpr int R = PL::radix[p];
  constexpr int s = PL::stride(p);
  constexpr int Lp = s * R;
  constexpr int NBUT = PL::L / R;
  constexpr int NB = (NBUT + PL::T - 1) / PL::T;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int beta = t + i * PL::T;
    if (NBUT % PL::T == 0 || beta < NBUT) {
      const int lo = beta % s;
      const int base = (beta / s) * Lp + lo;
      C a[R];
      sfor<R>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        a[j] = load(i, j, base + j * s);
      });
      if constexpr (p < PL::P - 1) {
        const int e1 = lo * (PL::L / Lp);
        sfor<R>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          if constexpr (j > 0) a[j] = cmul(a[j], __ldg(&tw[j * e1]));
        });
      }
      Dft<R, false>::run(a);
      sfor<R>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        store(i, j, base + j * s, a[j]);
      });
    }
  }
}

// Full DIF transform: global loader -> registers (digit-reversed).
template <class PL, bool INV, class C, class GLoad>
__device__ __forceinline__ void fft_dif(C *sbuf, int t, const C *__restrict__ tw,
                                        GLoad &&gload, C (&out)[PL::V]) {
  constexpr int RL = PL::Rlast;
  auto reg_store = [&](int i, int j, int, C v) { out[i * RL + j] = v; };
  if constexpr (PL::P == 1) {
    dif_pass<PL, 0, INV>(t, tw, gload, reg_store);
  } else {
    auto s_load = [&](int pos) { return sbuf[swz_t<C>(pos)]; };
    auto s_store = [&](int, int, int pos, C v) { sbuf[swz_t<C>(pos)] = v; };
    __syncthreads();  // previous readers of sbuf are done
    dif_pass<PL, 0, INV>(t, tw, gload, s_store);
    sfor<PL::P - 2>([&](auto qc) {
      constexpr int q = decltype(qc)::value + 1;
      __syncthreads();
      dif_pass<PL, q, INV>(t, tw, s_load, s_store);
    });
    __syncthreads();
    dif_pass<PL, PL::P - 1, INV>(t, tw, s_load, reg_store);
  }
}

// Final forward transform: digit-reversed registers -> natural order via gstore(pos, v).
template <class PL, class C, class GStore>
__device__ __forceinline__ void fft_dit_final(C *sbuf, int t, const C *__restrict__ tw,
                                              C (&in)[PL::V], GStore &&gstore) {
  constexpr int RL = PL::Rlast;
  auto reg_load = [&](int i, int j, int) { return in[i * RL + j]; };
  auto g_store = [&](int, int, int pos, C v) { gstore(pos, v); };
  if constexpr (PL::P == 1) {
    dit_pass<PL, 0>(t, tw, reg_load, g_store);
  } else {
    auto s_load = [&](int, int, int pos) { return sbuf[swz_t<C>(pos)]; };
    auto s_store = [&](int, int, int pos, C v) { sbuf[swz_t<C>(pos)] = v; };
    __syncthreads();
    dit_pass<PL, PL::P - 1>(t, tw, reg_load, s_store);
    sfor<PL::P - 2>([&](auto qc) {
      constexpr int q = PL::P - 2 - decltype(qc)::value;
      __syncthreads();
      dit_pass<PL, q>(t, tw, s_load, s_store);
    });
    __syncthreads();
    dit_pass<PL, 0>(t, tw, s_load, g_store);
  }
}

}  // namespace hk
