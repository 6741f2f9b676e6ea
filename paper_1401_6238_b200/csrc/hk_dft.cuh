// Register-resident DFT codelets for the fused Hankel product kernels.
//
// All radices are compile-time: loops are expanded with `sfor<N>` so every
// array index and every twiddle constant is a constant expression, which keeps
// the butterflies entirely in registers and turns twiddles into immediates.
//
// Sign convention (numpy / reference fourier.py:1-7): forward uses
// exp(-2*pi*i*j*k/n), inverse the conjugate kernel (the 1/n factor is applied
// by the caller).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace hk {

using cplx = double2;

// ---------------------------------------------------------------- compile-time loop
template <int I, int N, class F>
__device__ __forceinline__ void sfor_impl(F &&f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    sfor_impl<I + 1, N>(f);
  }
}
template <int N, class F>
__device__ __forceinline__ void sfor(F &&f) { sfor_impl<0, N>(f); }

// ---------------------------------------------------------------- complex helpers
// Every codelet is generic over the complex type C: double2 (complex128, the
// reference's precision) or float2 (the complex64 variant).
template <class C>
struct CT;
template <>
struct CT<double2> {
  using S = double;
  __device__ __forceinline__ static double2 make(double x, double y) { return make_double2(x, y); }
};
template <>
struct CT<float2> {
  using S = float;
  __device__ __forceinline__ static float2 make(float x, float y) { return make_float2(x, y); }
};

__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ cplx cmulc(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ cplx cswapfma(cplx a, double kx, double ky) {
  return make_double2(fma(kx, a.y, a.x), fma(ky, a.x, a.y));
}
__device__ __forceinline__ cplx caxpy(cplx a, double s, cplx b) {
  return make_double2(fma(s, b.x, a.x), fma(s, b.y, a.y));
}
// a * (-i) and a * (+i)
__device__ __forceinline__ cplx mul_mi(cplx a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ cplx mul_pi(cplx a) { return make_double2(-a.y, a.x); }

// complex64: the two components of a float2 sit in an aligned register pair,
// so sums, differences and real-scalar FMAs are ONE packed sm_100 instruction
// (FADD2 / FFMA2 on .f32x2) instead of two: the complex64 kernels are bound by
// instruction issue (FP32 runs at one warp instruction per clock per
// scheduler), so halving the additive instructions is what speeds them up.
__device__ __forceinline__ unsigned long long pk2(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
  float2 c;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c.x), "=f"(c.y) : "l"(r));
  return c;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
// a + s * b, s a real scalar (both components): one FFMA2
__device__ __forceinline__ float2 caxpy(float2 a, float s, float2 b) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(make_float2(s, s))), "l"(pk2(b)), "l"(pk2(a)));
  return upk2(r);
}
__device__ __forceinline__ unsigned long long pk2s(float x, float y) { return pk2(make_float2(x, y)); }
// Complex products stay scalar (two FMUL + two FFMA): the packed form needs a
// (-1, 1) sign pair per product and measured more instructions, not fewer.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
// a + (kx, ky) .* (a.y, a.x): the (1 + i k) rotations of the radix-16 codelet, one FFMA2
__device__ __forceinline__ float2 cswapfma(float2 a, float kx, float ky) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2s(kx, ky)), "l"(pk2s(a.y, a.x)), "l"(pk2(a)));
  return upk2(r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
__device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }

template <bool INV, class C>
__device__ __forceinline__ C cmul_dir(C a, C w) { return INV ? cmulc(a, w) : cmul(a, w); }
// z^3 = a (a^2 - 3 b^2) + i b (3 a^2 - b^2): six FP64 instructions (two cmuls: eight)
__device__ __forceinline__ cplx ccube(cplx z) {
  const double a2 = z.x * z.x, b2 = z.y * z.y;
  return make_double2(z.x * fma(-3.0, b2, a2), z.y * fma(3.0, a2, -b2));
}

// ---------------------------------------------------------------- constexpr twiddles
// cos / sin of 2*pi*e/R computed at compile time: exact integer reduction to a
// quadrant, Taylor series on |phi| <= pi/4 (error ~1 ulp).
constexpr double kHalfPi = 1.57079632679489661923132169163975144;

constexpr double taylor_sin(double x) {
  double term = x, sum = x;
  for (int k = 1; k < 14; ++k) {
    term *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 14; ++k) {
    term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
    sum += term;
  }
  return sum;
}
// angle 2*pi*e/R = (quarter turns) 4e/R; q = nearest integer, phi = (4e - qR)/R * pi/2
constexpr double tw_cos(long long e, long long R) {
  e %= R;
  if (e < 0) e += R;
  long long num = 4 * e;
  long long q = (2 * num + R) / (2 * R);
  double phi = (double)(num - q * R) / (double)R * kHalfPi;
  double c = taylor_cos(phi), s = taylor_sin(phi);
  switch (q & 3) {
    case 0: return c;
    case 1: return -s;
    case 2: return -c;
    default: return s;
  }
}
constexpr double tw_sin(long long e, long long R) {
  e %= R;
  if (e < 0) e += R;
  long long num = 4 * e;
  long long q = (2 * num + R) / (2 * R);
  double phi = (double)(num - q * R) / (double)R * kHalfPi;
  double c = taylor_cos(phi), s = taylor_sin(phi);
  switch (q & 3) {
    case 0: return s;
    case 1: return c;
    case 2: return -s;
    default: return -c;
  }
}

// a * exp(sign * 2*pi*i*E/R), sign = -1 forward, +1 inverse; E, R compile time.
template <int E, int R, bool INV, class C>
__device__ __forceinline__ C twc(C a) {
  using S = typename CT<C>::S;
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return a;
  } else if constexpr (4 * e == 2 * R) {
    return CT<C>::make(-a.x, -a.y);
  } else if constexpr (4 * e == R) {
    return INV ? mul_pi(a) : mul_mi(a);
  } else if constexpr (4 * e == 3 * R) {
    return INV ? mul_mi(a) : mul_pi(a);
  } else {
    constexpr S c = (S)tw_cos(e, R);
    constexpr S s = (S)(INV ? tw_sin(e, R) : -tw_sin(e, R));
    return CT<C>::make(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// ---------------------------------------------------------------- codelets
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *) {}
};

template <bool INV>
struct Dft<2, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <bool INV>
struct Dft<3, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    using S = typename CT<C>::S;
    constexpr S s3 = (S)0.866025403784438646763723170752936183;  // sin(2pi/3)
    C a = v[0], s = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    C m = CT<C>::make(fma((S)-0.5, s.x, a.x), fma((S)-0.5, s.y, a.y));
    // forward: X1 = m - i*s3*d, X2 = m + i*s3*d
    C r = CT<C>::make(-s3 * d.y, s3 * d.x);  // i*s3*d
    v[0] = cadd(a, s);
    if (INV) {
      v[1] = cadd(m, r);
      v[2] = csub(m, r);
    } else {
      v[1] = csub(m, r);
      v[2] = cadd(m, r);
    }
  }
};

template <bool INV>
struct Dft<4, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    C t2 = cadd(v[1], v[3]), t3 = csub(v[1], v[3]);
    t3 = INV ? mul_pi(t3) : mul_mi(t3);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

constexpr int first_factor(int R) { return (R % 4 == 0 && R != 8) ? 4 : (R % 2 == 0 ? 2 : 3); }

// Composite R = R1 * R2 (natural-order in and out):
//   X[k1 + R1 k2] = sum_{n2} W_R2^{n2 k2} W_R^{n2 k1} sum_{n1} v[n1 R2 + n2] W_R1^{n1 k1}
template <int R, bool INV>
struct Dft {
  static_assert(R > 4, "composite codelet");
  static constexpr int R1 = first_factor(R);
  static constexpr int R2 = R / R1;
  static_assert(R1 * R2 == R, "radix must factor into 2,3,4");
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C t[R];
    sfor<R2>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      C a[R1];
      sfor<R1>([&](auto n1c) {
        constexpr int n1 = decltype(n1c)::value;
        a[n1] = v[n1 * R2 + n2];
      });
      Dft<R1, INV>::run(a);
      sfor<R1>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        t[k1 * R2 + n2] = twc<n2 * k1, R, INV>(a[k1]);
      });
    });
    sfor<R1>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      C b[R2];
      sfor<R2>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        b[n2] = t[k1 * R2 + n2];
      });
      Dft<R2, INV>::run(b);
      sfor<R2>([&](auto k2c) {
        constexpr int k2 = decltype(k2c)::value;
        v[k1 + R1 * k2] = b[k2];
      });
    });
  }
};

// radix-8 as 2 x 4 keeps the W8 twiddles to the two odd slots
template <bool INV>
struct Dft<8, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C e[4] = {v[0], v[2], v[4], v[6]};
    C o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, INV>::run(e);
    Dft<4, INV>::run(o);
    o[1] = twc<1, 8, INV>(o[1]);
    o[2] = twc<2, 8, INV>(o[2]);
    o[3] = twc<3, 8, INV>(o[3]);
    sfor<4>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    });
  }
};

// radix-16 as 4 x 4 with the inner twiddles in scaled form.  b * W16^E is
// written as sigma * u: u needs at most two FMAs (tangent form, tau =
// tan(pi/8)) or two adds (W8 = cos(pi/4) (1 -+ i)), and the real scale sigma
// (1, cos(pi/8) or cos(pi/4)) is folded into the FMAs of the second radix-4
// stage.  In column k1 the inputs b1, b3 (exponents k1, 3k1) share one sigma,
// so their sum and difference carry it too.  144 FP instructions per
// butterfly instead of 160 (8 twiddles x 4 + 128 adds).
namespace r16 {
constexpr double kC1 = 0.923879532511286756128183189396788933;   // cos(pi/8)
constexpr double kTau = 0.414213562373095048801688724209698079;  // tan(pi/8)
constexpr double kC2 = 0.707106781186547524400844362104849039;   // cos(pi/4)
// reduced exponent: W16^E = i^(sign*m) * exp(i*sign*r*pi/8), r in {-1,0,1,2}
constexpr int red_m(int E) {
  const int e = ((E % 16) + 16) % 16;
  return (e % 4 == 3) ? e / 4 + 1 : e / 4;
}
constexpr int red_r(int E) {
  const int e = ((E % 16) + 16) % 16;
  return (e % 4 == 3) ? -1 : e % 4;
}
// scale code: 0 -> 1, 1 -> cos(pi/8), 2 -> cos(pi/4)
constexpr int sigma_code(int E) { return red_r(E) == 0 ? 0 : (red_r(E) == 2 ? 2 : 1); }
constexpr double sigma_val(int code) { return code == 0 ? 1.0 : (code == 1 ? kC1 : kC2); }

template <int Q, class C>
__device__ __forceinline__ C rot_i(C a) {  // a * i^Q
  constexpr int q = ((Q % 4) + 4) % 4;
  if constexpr (q == 0) return a;
  else if constexpr (q == 1) return CT<C>::make(-a.y, a.x);
  else if constexpr (q == 2) return CT<C>::make(-a.x, -a.y);
  else return CT<C>::make(a.y, -a.x);
}

// u with b * W16^E = sigma_val(sigma_code(E)) * u; forward W = exp(-2 pi i E / 16)
template <int E, bool INV, class C>
__device__ __forceinline__ C tw_u(C b) {
  using S = typename CT<C>::S;
  constexpr int sg = INV ? 1 : -1;
  constexpr int r = red_r(E), m = red_m(E);
  C u;
  if constexpr (r == 0) {
    u = b;
  } else if constexpr (r == 2) {  // (1 + i sg)
    if constexpr (sizeof(S) == 4)
      u = cswapfma(b, (S)-sg, (S)sg);
    else
      u = sg > 0 ? CT<C>::make(b.x - b.y, b.y + b.x) : CT<C>::make(b.x + b.y, b.y - b.x);
  } else {  // (1 + i k tau), k = sg * r
    constexpr S kt = (S)(sg * r * kTau);
    u = cswapfma(b, -kt, kt);
  }
  return rot_i<sg * m>(u);
}

// a + s * b with s a compile-time scale code and sign
template <int CODE, int SIGN, class C>
__device__ __forceinline__ C axpy(C a, C b) {
  using S = typename CT<C>::S;
  if constexpr (CODE == 0) {
    return SIGN > 0 ? cadd(a, b) : csub(a, b);
  } else {
    constexpr S s = (S)(SIGN * sigma_val(CODE));
    return caxpy(a, s, b);
  }
}
}  // namespace r16

namespace r16 {
// second radix-4 stage of the 4 x 4 radix-16: t[k1 * 4 + n2] -> v[k1 + 4 k2]
template <bool INV, class C>
__device__ __forceinline__ void stage2(const C (&t)[16], C *v) {
  sfor<4>([&](auto k1c) {
    constexpr int k1 = decltype(k1c)::value;
    constexpr int s2 = sigma_code(2 * k1), s1 = sigma_code(k1);
    static_assert(sigma_code(3 * k1) == s1, "b1 and b3 share their scale");
    const C b0 = t[k1 * 4];
    const C u1 = tw_u<k1, INV>(t[k1 * 4 + 1]);
    const C u2 = tw_u<2 * k1, INV>(t[k1 * 4 + 2]);
    const C u3 = tw_u<3 * k1, INV>(t[k1 * 4 + 3]);
    const C t0 = axpy<s2, 1>(b0, u2), t1 = axpy<s2, -1>(b0, u2);
    const C sm = cadd(u1, u3);
    const C df = INV ? mul_pi(csub(u1, u3)) : mul_mi(csub(u1, u3));
    v[k1] = axpy<s1, 1>(t0, sm);
    v[k1 + 8] = axpy<s1, -1>(t0, sm);
    v[k1 + 4] = axpy<s1, 1>(t1, df);
    v[k1 + 12] = axpy<s1, -1>(t1, df);
  });
}

// Column-major twiddle chunks of a radix-16 butterfly: chunk c holds the
// input twiddles of stage-1 column n2 = c, i.e. j = c + 4q (q = 0..3; chunk 0
// holds j = 4, 8, 12 and one pad).  0 marks the pad slot.
constexpr int colj(int c, int q) { return c == 0 ? (q < 3 ? 4 * (q + 1) : 0) : c + 4 * q; }

// q + x * w (INV: q + x * conj w) in four FMAs
template <bool INV, class C>
__device__ __forceinline__ C cfma_dir(C q, C x, C w) {
  if constexpr (INV)
    return CT<C>::make(fma(x.x, w.x, fma(x.y, w.y, q.x)), fma(x.y, w.x, fma(-x.x, w.y, q.y)));
  else
    return CT<C>::make(fma(x.x, w.x, fma(-x.y, w.y, q.x)), fma(x.x, w.y, fma(x.y, w.x, q.y)));
}
// 2 q - s (the difference partner of s = q + d, one FMA per component)
template <class C>
__device__ __forceinline__ C twice_minus(C q, C s) {
  using S = typename CT<C>::S;
  return CT<C>::make(fma((S)2, q.x, -s.x), fma((S)2, q.y, -s.y));  // (negated addend: scalar form)
}

// Radix-16 with input twiddles v[j] *= w_j (j = 1..15) folded into the first
// radix-4 stage (the transposed-DIT passes of the final transform):
//   x0 + w2 x2 = four FMAs, x0 - w2 x2 = 2 x0 - (x0 + w2 x2) = two more,
// so a twiddled column costs 24-28 FP64 instructions instead of 28-32.
// getw(c, w) loads chunk c in the colj layout.
template <bool INV, class C, class GetW>
__device__ __forceinline__ void dft16_tw_in(C (&v)[16], GetW &&getw) {
  C t[16];
  sfor<4>([&](auto n2c) {
    constexpr int n2 = decltype(n2c)::value;
    C w[4];
    getw(n2, w);
    // x_n1 = v[4 n1 + n2] carries twiddle j = 4 n1 + n2 = w[n2 ? n1 : n1 - 1]
    const C q0 = n2 == 0 ? v[n2] : cmul_dir<INV>(v[n2], w[0]);
    const C w1 = w[n2 ? 1 : 0], w2 = w[n2 ? 2 : 1], w3 = w[n2 ? 3 : 2];
    const C s0 = cfma_dir<INV>(q0, v[8 + n2], w2);
    const C s1 = twice_minus(q0, s0);
    const C p = cmul_dir<INV>(v[4 + n2], w1);
    const C s2 = cfma_dir<INV>(p, v[12 + n2], w3);
    C s3 = twice_minus(p, s2);
    s3 = INV ? mul_pi(s3) : mul_mi(s3);
    t[0 * 4 + n2] = cadd(s0, s2);
    t[2 * 4 + n2] = csub(s0, s2);
    t[1 * 4 + n2] = cadd(s1, s3);
    t[3 * 4 + n2] = csub(s1, s3);
  });
  stage2<INV>(t, v);
}
}  // namespace r16

template <bool INV>
struct Dft<16, INV> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C t[16];
    sfor<4>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      C a[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      Dft<4, INV>::run(a);
      sfor<4>([&](auto k1c) { t[decltype(k1c)::value * 4 + n2] = a[decltype(k1c)::value]; });
    });
    r16::stage2<INV>(t, v);
  }
};

}  // namespace hk

namespace hk {

// ---------------------------------------------------------------- pruned codelets
// DftP<R, INV, NZ, NO>: inputs v[n] are zero for n >= NZ (not read), and only
// outputs v[k], k < NO, are produced (the rest are left undefined).  Used for
// the zero-padded first pass of a vector transform (x has n << L nonzeros) and
// the truncated last pass of the final transform (only y[:n_1] is kept).
template <int R, bool INV, int NZ, int NO, bool Composite = (R > 4)>
struct DftP;

// small radices: full codelet when nothing is pruned, direct sums otherwise
template <int R, bool INV, int NZ, int NO>
struct DftP<R, INV, NZ, NO, false> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    if constexpr (NZ >= R && NO >= R) {
      Dft<R, INV>::run(v);
    } else if constexpr (NZ == 1) {
      sfor<NO>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr (k > 0) v[k] = v[0];
      });
    } else {
      C x[NZ];
      sfor<NZ>([&](auto nc) { x[decltype(nc)::value] = v[decltype(nc)::value]; });
      sfor<NO>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        C s = x[0];
        sfor<NZ - 1>([&](auto nc) {
          constexpr int n = decltype(nc)::value + 1;
          s = cadd(s, twc<n * k, R, INV>(x[n]));
        });
        v[k] = s;
      });
    }
  }
};

template <int R, bool INV, int NZ, int NO>
struct DftP<R, INV, NZ, NO, true> {
  static constexpr int R1 = first_factor(R);
  static constexpr int R2 = R / R1;
  static constexpr int NZ2 = NZ < R2 ? NZ : R2;  // nonzero n2 columns
  static constexpr int NO1 = NO < R1 ? NO : R1;  // needed k1 rows
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    if constexpr (NZ >= R && NO >= R) {
      Dft<R, INV>::run(v);
    } else {
      C t[R];
      sfor<NZ2>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        constexpr int nz1c = (NZ - n2 + R2 - 1) / R2;
        constexpr int nz1 = nz1c > R1 ? R1 : nz1c;
        C a[R1];
        sfor<nz1>([&](auto n1c) {
          constexpr int n1 = decltype(n1c)::value;
          a[n1] = v[n1 * R2 + n2];
        });
        DftP<R1, INV, nz1, NO1>::run(a);
        sfor<NO1>([&](auto k1c) {
          constexpr int k1 = decltype(k1c)::value;
          t[k1 * R2 + n2] = twc<n2 * k1, R, INV>(a[k1]);
        });
      });
      sfor<NO1>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        constexpr int no2c = (NO - k1 + R1 - 1) / R1;
        constexpr int no2 = no2c > R2 ? R2 : no2c;
        C b[R2];
        sfor<NZ2>([&](auto n2c) {
          constexpr int n2 = decltype(n2c)::value;
          b[n2] = t[k1 * R2 + n2];
        });
        DftP<R2, INV, NZ2, no2>::run(b);
        sfor<no2>([&](auto k2c) {
          constexpr int k2 = decltype(k2c)::value;
          v[k1 + R1 * k2] = b[k2];
        });
      });
    }
  }
};

// radix-16 with only inputs 0..3 nonzero (zero-padded first pass, L = 4 n):
// the first radix-4 stage is the identity, t[k1 * 4 + n2] = v[n2].
template <bool INV, int NO>
struct DftP<16, INV, 4, NO, true> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    C t[16];
    sfor<4>([&](auto k1c) {
      sfor<4>([&](auto n2c) { t[decltype(k1c)::value * 4 + decltype(n2c)::value] = v[decltype(n2c)::value]; });
    });
    r16::stage2<INV>(t, v);  // outputs k >= NO are dead code
  }
};
// radix-16 keeping NO < 16 outputs: the full codelet, the unused outputs'
// arithmetic is dead code once inlined (their stores are pruned by the pass).
template <bool INV, int NO>
struct DftP<16, INV, 16, NO, true> {
  template <class C>
  __device__ __forceinline__ static void run(C *v) {
    Dft<16, INV>::run(v);
  }
};

}  // namespace hk
