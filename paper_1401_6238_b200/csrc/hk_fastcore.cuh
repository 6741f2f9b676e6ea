// Shared device code of the fast fused 1D kernels (hk_fast1d.cu, hk_pp1d.cu):
// pass engine with pluggable synchronisation and first-pass twiddle source,
// pruned first/last passes, conflict-free swizzle.
#pragma once

#include <type_traits>

#include "hk_fft1d.cuh"
#include "hk_internal.h"
#include "hk_tmem.cuh"

namespace hk {
namespace fast {

__device__ __forceinline__ int swz2(int pos) { return pos ^ (((pos >> 4) ^ (pos >> 8)) & 7); }
// 8-byte (complex64) elements are served 16 lanes per wavefront: XOR the low
// FOUR position bits with bits 4-7 ^ 8-11 (conflict-free in every pass of the
// radix-16 plans for both thread mappings used by `pass`).
__device__ __forceinline__ int swz8(int pos) { return pos ^ (((pos >> 4) ^ (pos >> 8)) & 15); }
template <class C>
__device__ __forceinline__ int swzc(int pos) {
  if constexpr (sizeof(C) == 8)
    return swz8(pos);
  else
    return swz2(pos);
}

// Cheap addressing of swz2-swizzled shared memory for radix-16 plans with
// L <= 4096 (positions = 3 hex digits d2 d1 d0).  In the pass over hex digit q
// a butterfly touches pos = base + j*16^q, and
//   swz2(pos) = B + J(j) + (U ^ (j & 7))
// with per-thread B, U and compile-time J(j): one base register plus at most
// seven XOR-with-immediate ops cover all 16 accesses, which then use
// immediate offsets (instead of ~5 integer ops per access).
template <int Q>
struct HexAddr {
  uint32_t r0;  // shared-space byte address for j & 7 == 0, J == 0
  __device__ __forceinline__ HexAddr(uint32_t sbase, int base) {
    const int d0 = base & 15, d1 = (base >> 4) & 15, d2 = (base >> 8) & 15;
    int B, U;
    if constexpr (Q == 2) {
      B = 16 * d1 + (d0 & 8);
      U = (d0 ^ d1) & 7;
    } else if constexpr (Q == 1) {
      B = 256 * d2 + (d0 & 8);
      U = (d0 ^ d2) & 7;
    } else {
      B = 256 * d2 + 16 * d1;
      U = (d1 ^ d2) & 7;
    }
    r0 = sbase + 16u * (uint32_t)(B + U);
  }
  template <int J>
  static constexpr int imm() {
    return Q == 2 ? 16 * 256 * J : (Q == 1 ? 16 * 16 * J : 16 * (J & 8));
  }
  template <int J>
  __device__ __forceinline__ uint32_t reg() const {
    return r0 ^ (uint32_t)(16 * (J & 7));
  }
  template <int J>
  __device__ __forceinline__ cplx ld() const {
    cplx v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];\n"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"(reg<J>()), "n"(imm<J>())
                 : "memory");
    return v;
  }
  template <int J>
  __device__ __forceinline__ void st(cplx v) const {
    asm volatile("st.shared.v2.f64 [%0+%1], {%2, %3};\n" ::"r"(reg<J>()), "n"(imm<J>()),
                 "d"(v.x), "d"(v.y)
                 : "memory");
  }
};

template <class PL>
constexpr bool hex_plan() {
  if (PL::L > 4096) return false;
  for (int q = 0; q < PL::P; ++q)
    if (PL::radix[q] != 16) return false;
  return true;
}

// Marker functors: a pass whose Load / Store is SmemIO uses HexAddr addressing
// of the swizzled exchange buffer at `sbase` (shared-space byte address).
struct SmemIO {
  uint32_t sbase;
};

template <class PL>
struct Traits {
  static constexpr int hi_count(int p) { return PL::L / (PL::stride(p) * PL::radix[p]); }
  static constexpr bool hi_major(int p) { return p > 0 && p < PL::P - 1 && hi_count(p) >= 8; }
  static constexpr int warps = PL::CTA / 32;
  static constexpr int slabs = (warps + 3) / 4;
  static constexpr int cols_needed = slabs * 4 * PL::V;
  static constexpr int tmem_cols = cols_needed <= 32    ? 32
                                   : cols_needed <= 64  ? 64
                                   : cols_needed <= 128 ? 128
                                   : cols_needed <= 256 ? 256
                                                        : 512;
  static_assert(cols_needed <= 512, "accumulator does not fit in TMEM");
  static_assert(PL::V % 4 == 0, "TMEM chunks of 4 complex values");
  static constexpr int min_blocks = (PL::CTA <= 256) ? 2 : 1;
};

// Pass-0 twiddle sources deliver chunks of TW0::kChunk values (default 4).
template <class T, class = void>
struct ChunkOf {
  static constexpr int value = 4;
};
template <class T>
struct ChunkOf<T, std::void_t<decltype(T::kChunk)>> {
  static constexpr int value = T::kChunk;
};
struct NoHookT {
  __device__ __forceinline__ void operator()() const {}
};

// Twiddle sources that also hold the pass-1 twiddles (a per-thread TMEM slab)
// expose chunk1(c, w): W_{Lp}^{j lo}, j = 4c+1 .. 4c+4, of this thread's pass-1
// butterfly.
template <class T, class = void>
struct HasChunk1 : std::false_type {};
template <class T>
struct HasChunk1<T, std::void_t<decltype(&T::chunk1)>> : std::true_type {};
// Sources with kColChunks store a butterfly's twiddles in the column-major
// chunk order of r16::colj (chunk c = stage-1 column c of the radix-16), so the
// final transform's twiddled passes fold them into the first radix-4 stage.
template <class T, class = void>
struct ColChunks : std::false_type {};
template <class T>
struct ColChunks<T, std::void_t<decltype(T::kColChunks)>> : std::bool_constant<T::kColChunks> {};

// Pass-0 twiddles by recurrence: W_L^{j beta} = (W_L^beta)^j from one table
// read per butterfly (two interleaved chains, <= 8 products deep), trading
// 14 complex multiplies for 15 table reads (TMEM or L1 traffic).
template <class C>
struct Tw0RecT {
  const C *__restrict__ tw;  // W_L^e, e in [0, L)
  __device__ __forceinline__ C base(int beta) const { return __ldg(&tw[beta]); }
};
using Tw0Rec = Tw0RecT<cplx>;
template <class T>
struct is_tw0rec : std::false_type {};
template <class C>
struct is_tw0rec<Tw0RecT<C>> : std::true_type {};

template <int R, bool INV, class C>
__device__ __forceinline__ void twiddle_rec(C (&a)[R], C w1) {
  const C w2 = cmul(w1, w1);
  C wo = w1, we = w2;
#pragma unroll
  for (int j = 1; j < R; j += 2) {
    a[j] = cmul_dir<INV>(a[j], wo);
    if (j + 1 < R) a[j + 1] = cmul_dir<INV>(a[j + 1], we);
    if (j + 2 < R) wo = cmul(wo, w2);
    if (j + 3 < R) we = cmul(we, w2);
  }
}

// One pass.  FINAL=false: DIF (butterfly then twiddle), pruned to NZ nonzero
// inputs.  FINAL=true: transposed DIT of the forward transform (twiddle then
// butterfly), pruned to NO needed outputs.
// Pass-0 twiddles W_L^{j beta} (j = 1..R0-1) from the thread-major global table.
struct Tw0Global {
  const cplx *__restrict__ tw0;
  int nbut;
  int r0;
  __device__ __forceinline__ void chunk(int beta, int c, cplx *w) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = 4 * c + q + 1;
      w[q] = j < r0 ? __ldg(&tw0[(j - 1) * nbut + beta]) : make_double2(1.0, 0.0);
    }
  }
};

// `tw` holds W_TWL^e, e in [0, TWL), TWL a multiple of every pass length
// Lp >= 1 uses: the plan's full W_L table (TWL = L) or the compact W_{L/R0}
// table (TWL = L / R0), whose few KB stay L1-resident next to a full
// shared-memory carve-out (the strided reads of a W_L table touch one 128-B
// line per twiddle).
template <class PL, int p, bool INV, bool FINAL, int NZ, int NO, int TWL = PL::L, bool REC = false,
          class TW0, class Load, class Store, class C, class PreStore = NoHookT, bool HOIST = false>
__device__ __forceinline__ void pass(int t, const C *__restrict__ tw, const TW0 &tw0,
                                     Load &&load, Store &&store, PreStore pre_store = PreStore()) {
  using Tr = Traits<PL>;
  constexpr int R = PL::radix[p];
  constexpr int s = PL::stride(p);
  constexpr int Lp = s * R;
  constexpr int NBUT = PL::L / R;
  constexpr int NB = (NBUT + PL::T - 1) / PL::T;
  constexpr int H = Tr::hi_count(p);
  // hi-major order makes a warp's table reads of the pass-p twiddles broadcast;
  // with per-thread twiddle slabs (HasChunk1) the lo-major order is used, which
  // keeps the pass P-2 -> P-1 exchange inside each warp (see fft_dif).
  constexpr bool HIM = Tr::hi_major(p) && !HasChunk1<TW0>::value;
  constexpr int NIN = FINAL ? R : NZ;
  constexpr int NOUT = NO;  // DIF passes: NO < R prunes outputs (callers pass R otherwise)
  constexpr bool kCol = ColChunks<TW0>::value;
  static_assert(!kCol || R == 16 || (p != 0 && !(p == 1 && PL::P == 3)),
                "column-major twiddle chunks are laid out for radix-16 passes");
  constexpr bool kFuse = FINAL && kCol && R == 16 && PL::P == 3 && (p == 0 || p == 1) &&
                         ChunkOf<TW0>::value == 4 && !is_tw0rec<TW0>::value;
  // Pass-0 recurrence bases of a thread's NB butterflies, beta = t + i*T:
  // W_L^beta = W_L^t * W_L^{i T}, the second factor a compile-time constant,
  // so one table read serves all NB butterflies (8192 = 2 x 16^3: NB = 8).
  [[maybe_unused]] C base0 = CT<C>::make(1, 0);
  if constexpr (p == 0 && PL::P > 1 && NB > 1 && is_tw0rec<TW0>::value) base0 = tw0.base(t);
  // HOIST: issue every load of the thread's NB butterflies before the first
  // butterfly (global operands: one exposed latency per pass, not NB)
  constexpr bool kHoist = HOIST && !std::is_same_v<std::decay_t<Load>, SmemIO>;
  [[maybe_unused]] C pre[kHoist ? NB : 1][kHoist ? NIN : 1];
  if constexpr (kHoist) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int beta = t + i * PL::T;
      if (NBUT % PL::T == 0 || beta < NBUT) {
        int lo, hi;
        if constexpr (HIM) {
          hi = beta % H;
          lo = beta / H;
        } else {
          lo = beta % s;
          hi = beta / s;
        }
        const int base = hi * Lp + lo;
        sfor<NIN>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          pre[i][j] = load(i, j, base + j * s);
        });
      }
    }
  }
  // Fewer butterflies than threads inside one warp (192 = 16 x 12 on 16
  // threads): the idle threads run butterfly 0 with their stores masked
  // instead of branching around it, because the TMEM twiddle reads inside are
  // warp-collective (tcgen05.ld.sync.aligned).
  constexpr bool kPred = NBUT < PL::T && PL::T <= 32;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int beta_raw = t + i * PL::T;
    const bool live = NBUT % PL::T == 0 || beta_raw < NBUT;
    const int beta = (kPred && !live) ? 0 : beta_raw;
    if (kPred || live) {
      int lo, hi;
      if constexpr (HIM) {
        hi = beta % H;
        lo = beta / H;
      } else {
        lo = beta % s;
        hi = beta / s;
      }
      const int base = hi * Lp + lo;
      constexpr int Q = PL::P - 1 - p;
      C a[R];
      if constexpr (std::is_same_v<std::decay_t<Load>, SmemIO>) {
        const HexAddr<Q> ad(load.sbase, base);
        sfor<NIN>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          a[j] = ad.template ld<j>();
        });
      } else if constexpr (kHoist) {
        sfor<NIN>([&](auto jc) { a[decltype(jc)::value] = pre[i][decltype(jc)::value]; });
      } else {
        sfor<NIN>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          a[j] = load(i, j, base + j * s);
        });
      }
      auto twiddle = [&]() {
        if constexpr (p == 0 && PL::P > 1 && is_tw0rec<TW0>::value) {
          if constexpr (NB > 1) {
            C bi = base0;
            sfor<NB>([&](auto ic) {  // constant index: bi = base0 * W_L^{i T}
              constexpr int ii = decltype(ic)::value;
              if (ii == i) bi = twc<ii * PL::T, PL::L, false>(base0);
            });
            twiddle_rec<R, INV>(a, bi);
          } else {
            twiddle_rec<R, INV>(a, tw0.base(beta));
          }
        } else if constexpr (p == 0 && PL::P > 1) {
          // chunks of CK twiddles (j = CK*c+1 .. CK*c+CK) keep register pressure flat
          constexpr int CK = ChunkOf<TW0>::value;
          sfor<(R - 1 + CK - 1) / CK>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            C w[CK];
            tw0.chunk(beta, c, w);
            sfor<CK>([&](auto qc) {
              constexpr int q = decltype(qc)::value;
              constexpr int j = kCol ? r16::colj(c, q) : CK * c + q + 1;
              if constexpr (j > 0 && j < R) a[j] = cmul_dir<INV>(a[j], w[q]);
            });
          });
        } else if constexpr (p == 1 && PL::P == 3 && HasChunk1<TW0>::value) {
          sfor<(R - 1 + 3) / 4>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            C w[4];
            tw0.chunk1(c, w);
            sfor<4>([&](auto qc) {
              constexpr int q = decltype(qc)::value;
              constexpr int j = kCol ? r16::colj(c, q) : 4 * c + q + 1;
              if constexpr (j > 0 && j < R) a[j] = cmul_dir<INV>(a[j], w[q]);
            });
          });
        } else if constexpr (p < PL::P - 1 && REC) {
          twiddle_rec<R, INV>(a, __ldg(&tw[lo * (TWL / Lp)]));
        } else if constexpr (p < PL::P - 1) {
          // chunks of 4 loads behind a compiler fence: the scheduler may not
          // hoist all R-1 twiddles (4(R-1) registers) above the butterfly
          sfor<(R - 1 + 3) / 4>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            asm volatile("" ::: "memory");
            C w[4];
            sfor<4>([&](auto qc) {
              constexpr int j = 4 * c + decltype(qc)::value + 1;
              if constexpr (j < R) w[decltype(qc)::value] = __ldg(&tw[j * lo * (TWL / Lp)]);
            });
            sfor<4>([&](auto qc) {
              constexpr int j = 4 * c + decltype(qc)::value + 1;
              if constexpr (j < R) a[j] = cmul_dir<INV>(a[j], w[decltype(qc)::value]);
            });
          });
        }
      };
      if constexpr (kFuse) {
        // input twiddles folded into the first radix-4 stage (r16::dft16_tw_in)
        r16::dft16_tw_in<false>(a, [&](int c, C *w) {
          if constexpr (p == 0)
            tw0.chunk(beta, c, w);
          else
            tw0.chunk1(c, w);
        });
      } else if constexpr (FINAL) {
        twiddle();
        DftP<R, false, R, NO>::run(a);
      } else {
        DftP<R, INV, NZ, NO>::run(a);
        twiddle();
      }
      pre_store();
      if (kPred && !live) continue;
      if constexpr (std::is_same_v<std::decay_t<Store>, SmemIO>) {
        const HexAddr<Q> ad(store.sbase, base);
        sfor<NOUT>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          ad.template st<j>(a[j]);
        });
      } else {
        sfor<NOUT>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          store(i, j, base + j * s, a[j]);
        });
      }
    }
  }
}

template <class PL, class C, class Lambda>
__device__ __forceinline__ decltype(auto) pick_io(Lambda &l, const SmemIO &sio) {
  if constexpr (hex_plan<PL>() && sizeof(C) == 16)
    return (sio);
  else
    return (l);
}

// bar.sync as volatile asm: keeps the volatile ld/st.shared of HexAddr ordered
struct CtaSync {
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync 0;\n" ::: "memory");
  }
};

// When one product's threads sit inside a single warp (T <= 32, T | 32), its
// exchanges only need the warp's lanes ordered: products in different warps
// then run free of each other instead of in CTA lockstep.
struct WarpSync {
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.warp.sync -1;\n" ::: "memory");
  }
};

template <class PL>
using GroupSync = std::conditional_t<(PL::T <= 32 && 32 % PL::T == 0), WarpSync, CtaSync>;

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// Default entry of fft_dif: a group barrier before pass 0 (orders its stores
// after the previous transform's reads of the exchange buffer).  Any other
// Entry object is called instead right before the pass-0 stores (a split
// arrive/wait barrier whose wait then overlaps the pass-0 loads and math).
struct SyncEntry {};
// A global-operand loader wrapped in Hoisted makes fft_dif's first pass issue
// all of a thread's loads before its butterflies (fast::pass HOIST).
template <class F>
struct Hoisted {
  F f;
  __device__ __forceinline__ auto operator()(int pos) const { return f(pos); }
};
template <class T>
struct IsHoisted : std::false_type {};
template <class F>
struct IsHoisted<Hoisted<F>> : std::true_type {};

// hook() runs (on every thread) right after the barrier that follows pass 0,
// i.e. once every thread of the group has consumed the pass-0 input.
//
// WSync (if not void) replaces the group barrier before the last pass.  Valid
// when that exchange stays inside each warp: lo-major pass P-2 with
// radix[P-2] == radix[P-1] and 32 % radix[P-1] == 0 -- warp w then writes and
// reads exactly positions [32 w R, 32 (w + 1) R) (R the last radix).
template <class PL, bool INV, int NZ, int TWL = PL::L, bool REC = false, class TW0, class GLoad,
          class Sync = CtaSync, class Hook = NoHook, class WSync = void, class Entry = SyncEntry,
          class C>
__device__ __forceinline__ void fft_dif(C *sbuf, int t, const C *__restrict__ tw,
                                        const TW0 &tw0, GLoad &&gload, C (&out)[PL::V],
                                        Sync sync = Sync(), Hook hook = Hook(),
                                        WSync * = nullptr, Entry entry = Entry()) {
  constexpr bool kEntrySync = std::is_same_v<Entry, SyncEntry>;
  constexpr bool kHoistG = IsHoisted<std::decay_t<GLoad>>::value;
  auto last_sync = [&]() {
    if constexpr (std::is_void_v<WSync>)
      sync();
    else
      WSync()();
  };
  constexpr int RL = PL::Rlast;
  constexpr int R0 = PL::radix[0];
  // gload(pos), or gload(i, j, pos) for loaders that need the butterfly slot
  auto g_load = [&](int i, int j, int pos) {
    if constexpr (std::is_invocable_v<GLoad, int, int, int>)
      return gload(i, j, pos);
    else
      return gload(pos);
  };
  auto s_load_l = [&](int, int, int pos) { return sbuf[swzc<C>(pos)]; };
  auto s_store_l = [&](int, int, int pos, C v) { sbuf[swzc<C>(pos)] = v; };
  auto r_store = [&](int i, int j, int, C v) { out[i * RL + j] = v; };
  const SmemIO sio{smem_u32(sbuf)};
  auto &&s_load = pick_io<PL, C>(s_load_l, sio);
  auto &&s_store = pick_io<PL, C>(s_store_l, sio);
  static_assert(PL::P >= 2, "fast path needs at least two passes");
  if constexpr (kEntrySync) sync();
  using SL = decltype(s_load);
  using SS = decltype(s_store);
  if constexpr (kEntrySync)
    pass<PL, 0, INV, false, (NZ < R0 ? NZ : R0), R0, TWL, REC, TW0, decltype(g_load) &, SS, C,
         NoHookT, kHoistG>(t, tw, tw0, g_load, s_store);
  else
    pass<PL, 0, INV, false, (NZ < R0 ? NZ : R0), R0, TWL, REC, TW0, decltype(g_load) &, SS, C,
         Entry &>(t, tw, tw0, g_load, s_store, entry);
  sfor<PL::P - 2>([&](auto qc) {
    constexpr int q = decltype(qc)::value + 1;
    sync();
    if constexpr (q == 1) hook();
    pass<PL, q, INV, false, PL::radix[q], PL::radix[q], TWL, REC, TW0, SL, SS>(t, tw, tw0, s_load,
                                                                          s_store);
  });
  if constexpr (PL::P == 2) {
    sync();
    hook();
  } else {
    last_sync();
  }
  pass<PL, PL::P - 1, INV, false, RL, RL, TWL, REC, TW0, SL, decltype(r_store) &>(t, tw, tw0, s_load,
                                                                             r_store);
}

// WSync (if not void): the entry barrier and the pass P-1 -> P-2 exchange stay
// inside each warp (same condition as fft_dif; the entry barrier only orders
// against the previous transform's last-pass reads, which were warp-local).
template <class PL, int NO, int TWL = PL::L, bool REC = false, class TW0, class GStore,
          class Sync = CtaSync, class WSync = void, class C>
__device__ __forceinline__ void fft_final(C *sbuf, int t, const C *__restrict__ tw,
                                          const TW0 &tw0, C (&in)[PL::V], GStore &&gstore,
                                          Sync sync = Sync(), WSync * = nullptr) {
  auto warp_sync = [&]() {
    if constexpr (std::is_void_v<WSync>)
      sync();
    else
      WSync()();
  };
  constexpr int RL = PL::Rlast;
  constexpr int R0 = PL::radix[0];
  auto r_load = [&](int i, int j, int) { return in[i * RL + j]; };
  auto s_load_l = [&](int, int, int pos) { return sbuf[swzc<C>(pos)]; };
  auto s_store_l = [&](int, int, int pos, C v) { sbuf[swzc<C>(pos)] = v; };
  auto g_store = [&](int, int, int pos, C v) { gstore(pos, v); };
  const SmemIO sio{smem_u32(sbuf)};
  auto &&s_load = pick_io<PL, C>(s_load_l, sio);
  auto &&s_store = pick_io<PL, C>(s_store_l, sio);
  warp_sync();
  using SL = decltype(s_load);
  using SS = decltype(s_store);
  pass<PL, PL::P - 1, false, true, RL, RL, TWL, REC, TW0, decltype(r_load) &, SS>(t, tw, tw0, r_load,
                                                                             s_store);
  sfor<PL::P - 2>([&](auto qc) {
    constexpr int q = PL::P - 2 - decltype(qc)::value;
    if constexpr (q == PL::P - 2)
      warp_sync();
    else
      sync();
    pass<PL, q, false, true, PL::radix[q], PL::radix[q], TWL, REC, TW0, SL, SS>(t, tw, tw0, s_load,
                                                                           s_store);
  });
  sync();
  pass<PL, 0, false, true, R0, (NO < R0 ? NO : R0), TWL, REC, TW0, SL, decltype(g_store) &>(
      t, tw, tw0, s_load, g_store);
}

// Streamed operand loads bypass L1 allocation: each element is read once, and
// keeping L1 for the twiddle tables (re-read by every pass of every product)
// is what matters once the exchange buffer has claimed most of the carve-out.
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ cplx ld_stream(const cplx *p) {
  cplx v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float *p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];\n" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_stream(const float2 *p) {
  float2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// Per-thread asynchronous copies (LDGSTS) with zero fill past the operand end.
__device__ __forceinline__ void cpa16(uint32_t dst, const void *src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa8(uint32_t dst, const void *src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ cplx load_elem(const Factor &f, long long off, int pos, double scale) {
  if (pos >= f.len) return make_double2(0.0, 0.0);
  const long long k = (long long)pos * f.estride;
  if (f.kind == FK_F64) {
    const double *p = static_cast<const double *>(f.ptr) + off;
    return make_double2(ld_stream(p + k) * scale, 0.0);
  }
  const cplx *p = static_cast<const cplx *>(f.ptr) + off;
  cplx v = ld_stream(p + k);
  return make_double2(v.x * scale, v.y * scale);
}

// complex64 variant: FK_C64 / FK_F32 operands.
__device__ __forceinline__ float2 load_elem_f(const Factor &f, long long off, int pos,
                                              float scale) {
  if (pos >= f.len) return make_float2(0.f, 0.f);
  const long long k = (long long)pos * f.estride;
  if (f.kind == FK_F32) {
    const float *p = static_cast<const float *>(f.ptr) + off;
    return make_float2(ld_stream(p + k) * scale, 0.f);
  }
  const float2 *p = static_cast<const float2 *>(f.ptr) + off;
  const float2 v = ld_stream(p + k);
  return make_float2(v.x * scale, v.y * scale);
}

}  // namespace fast
}  // namespace hk
