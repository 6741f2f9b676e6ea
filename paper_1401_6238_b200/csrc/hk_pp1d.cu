// K1 producer/consumer variant for the batched H x^{m-1} workload (cfg2):
// one 512-thread CTA per SM runs two product groups in ping-pong while the
// Tensor Memory Accelerator streams the next operands into shared memory.
//
//   smem : ex[2][L] (per-group exchange) | hst[L] (h staging, shared by the
//          two groups in turn) | xst[2][XS] (per-group x staging)
//   TMEM : cols [0,256)   spectral accumulator (ifft(h) .* fft(x)^p), per thread
//          cols [256,512) the thread's first-pass twiddles W_L^{j t}, j=1..R0-1,
//          loaded once per CTA (they are identical for every product)
//   sync : mbarrier complete_tx for TMA arrivals, named barrier per group
//
// Product k of a CTA belongs to group k&1.  Group g, after the first pass of
// ifft(h_k) has consumed hst, hands hst to the TMA for h_{k+1} (the other
// group's next product); after the first pass of fft(x_k) it refills its own
// xst with x_{k+2}.  The copy engine therefore runs a full half-period ahead
// of the math, global-load latency leaves the critical path, and the two
// groups drift into the anti-phase that keeps the FP64 pipe busy while the
// other group is in a barrier.
//
// Math per product is the fast kernel's (hk_fastcore.cuh) except that the
// 1/L of the inverse transform is applied to the n_1 kept outputs instead of
// the L inputs (4x fewer multiplies; results agree to rounding).
#include <atomic>
#include <stdio.h>
#include <stdlib.h>

#include "hk_fastcore.cuh"

namespace hk {
namespace pp {

using fast::pass;
using fast::swz2;

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(addr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
// Split WAR barrier of a product group: every warp arrives (one lane, after
// the loaded values were consumed) once it has finished reading the exchange
// buffer; the next writer waits only right before its first stores.
struct WarWait {
  uint32_t addr, parity;
  bool on;
  __device__ __forceinline__ void operator()() const {
    if (on) mbar_wait(addr, parity);
  }
};
__device__ __forceinline__ void war_arrive(uint32_t addr) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(addr);
}

// Named barrier with a runtime id (one code copy serves both groups).
template <int N>
struct GroupBar {
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(N) : "memory");
  }
};

template <int ID, int N>
struct NamedSync {
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"n"(ID), "n"(N) : "memory");
  }
};

// First-pass twiddles from this thread's TMEM slab.
struct Tw0Tmem {
  uint32_t taddr;
  __device__ __forceinline__ void chunk(int, int c, cplx *w) const { tmem_ld4(taddr + 16 * c, w); }
};
// Same slab read 8 twiddles per tcgen05.ld (two waits per pass instead of four).
struct Tw0Tmem8 {
  static constexpr int kChunk = 8;
  uint32_t taddr;
  __device__ __forceinline__ void chunk(int, int c, cplx *w) const { tmem_ld8(taddr + 32 * c, w); }
};

// Both twiddle sets from TMEM: pass 0 (W_L^{j t}) and pass 1 (W_{L/R0}^{j lo}).
// A thread's twiddles depend only on its index in its group, so the two
// groups' warps that share a TMEM lane quadrant and an index share one slab.
// COL: chunks in the column-major order of r16::colj (the final transform then
// folds them into its first radix-4 stage, fast::pass kFuse).
template <bool COL>
struct Tw01TmemT {
  static constexpr bool kColChunks = COL;
  uint32_t taddr0, taddr1;
  __device__ __forceinline__ void chunk(int, int c, cplx *w) const { tmem_ld4(taddr0 + 16 * c, w); }
  __device__ __forceinline__ void chunk1(int c, cplx *w) const { tmem_ld4(taddr1 + 16 * c, w); }
};

template <class PL>
struct Layout {
  static constexpr int L = PL::L;
  static constexpr int T = PL::T;
  static_assert(PL::G == 1 && T == 256, "ping-pong kernel: one product per 256-thread group");
  static_assert(PL::L / PL::radix[0] == T, "first pass: one butterfly per thread");
};

// TWV bit 0: pass-0 twiddles by recurrence from W_L^t (else the TMEM slab);
// bit 1: pass->=1 twiddles by recurrence from one compact-table read;
// bit 3: pass-1 twiddles from TMEM too (slabs shared by the two groups).
// Product k of a CTA is item b = blockIdx.x + k * gridDim.x of the batch, at
// operand offset (b / nsub) * bstride + (b % nsub) * sstride (the two-level
// row stage runs nsub rows per item; plain batches have nsub = 1).
template <bool ROWS>
__device__ __forceinline__ long long pp_off(const Args1D &a, long long b, long long bs,
                                            long long ss) {
  if (!ROWS || a.nsub == 1) return b * bs;  // plain batches launch with nsub == 1
  // launch items and nsub fit 32 bits (checked at launch): one 32-bit division
  // instead of the emulated 64-bit one
  const unsigned ob = (unsigned)b / (unsigned)a.nsub;
  return ob * bs + ((unsigned)b - ob * (unsigned)a.nsub) * ss;
}

// XD (NZ == R0: x is a full-length row, the two-level row stage): x is not
// staged in shared memory (it would not fit next to three L buffers); pass 0
// of fft(x) issues all of a thread's global loads up front, the rows are
// prefetched into L2 one product ahead, and the other group covers the wait.
template <class PL, int NZ, int NO, int TWV>
__global__ void __launch_bounds__(2 * PL::T, 1) k_hankel_pp(const __grid_constant__ Args1D a) {
  constexpr bool REC = (TWV & 2) != 0;
  constexpr int L = PL::L, T = PL::T, V = PL::V, R0 = PL::radix[0];
  constexpr int S0 = PL::stride(0);
  constexpr bool XD = NZ >= R0;
  constexpr bool HD = (TWV & 64) != 0;  // h loaded directly (no TMA staging)
  constexpr int XS = XD ? 0 : NZ * S0;  // staged x elements
  constexpr int TW1 = L / R0;  // passes >= 1 read the compact W_{L/R0} table
  (void)Layout<PL>{};
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // full_h[0..1], full_x[0..1] (TMA arrivals); war_x[0..1], war_h[0..1] (split
  // WAR barriers of group G: h pass-2 reads -> x pass-0 stores, final pass-0
  // reads -> next h pass-0 stores; used with TW1T)
  __shared__ __align__(8) uint64_t mbar[8];
  __shared__ uint32_t tmem_slot;
  cplx *ex = reinterpret_cast<cplx *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  cplx *hst = ex + 2 * L;
  cplx *xst = hst + L;

  const int warp = threadIdx.x >> 5;
  const int g = threadIdx.x / T;
  const int t_in = threadIdx.x - g * T;
  const uint32_t mb_h0 = smem_u32(&mbar[0]), mb_x0 = smem_u32(&mbar[2]);
  const uint32_t mb_wx0 = smem_u32(&mbar[4]), mb_wh0 = smem_u32(&mbar[6]);

  // The TMA only ever writes the first h.len (x.len) staged elements: zero the
  // tails once so the first passes read the zero padding without bounds tests.
  for (int i = a.h.len + (int)threadIdx.x; i < L; i += blockDim.x) hst[i] = make_double2(0.0, 0.0);
  for (int i = (XD ? XS : a.fac[0].len) + (int)threadIdx.x; i < XS; i += blockDim.x) {
    xst[i] = make_double2(0.0, 0.0);
    xst[XS + i] = make_double2(0.0, 0.0);
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&mbar[i]), 1);
    for (int i = 4; i < 8; ++i) mbar_init(smem_u32(&mbar[i]), T / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;
  const uint32_t tacc = tmem_slot + lane_q + (uint32_t)((warp >> 2) * 64);
  constexpr bool TW1T = (TWV & 8) != 0;
  // TWV bit 7: column-major twiddle chunks, folded into the final transform's
  // first radix-4 stages; and the cube X^3 in six FP64 instructions
  constexpr bool COLW = TW1T && (TWV & 128) != 0;
  // with TW1T the pass-0 slab of the thread index t_in is shared by both groups
  // (cols 256 + 64 * ((warp >> 2) & 1)) and the pass-1 slab sits at 384 + ...
  const uint32_t ttw = tmem_slot + lane_q + 256u +
                       (uint32_t)((TW1T ? ((warp >> 2) & 1) : (warp >> 2)) * 64);
  const uint32_t ttw1 = ttw + 128u;

  if constexpr (TW1T) {
    static_assert(!(TWV & 1) && PL::P == 3, "pass-1 TMEM twiddles need the pass-0 slab too");
    if (g == 0) {
      const fast::Tw0Global g0{a.tw0, L / R0, R0};
      // pass-1 butterfly of thread t (lo-major with TMEM twiddles, see
      // fast::pass): lo = t mod stride(1), twiddles W_{L/R0}^{j lo}
      constexpr int R1 = PL::radix[1];
      const int lo1 = t_in % PL::stride(1);
      static_assert(!COLW || (R0 == 16 && PL::radix[1] == 16), "column chunks: radix-16 passes");
#pragma unroll
      for (int c = 0; c < (R0 - 1 + 3) / 4; ++c) {
        cplx w[4];
        if constexpr (COLW) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = r16::colj(c, q);
            w[q] = j > 0 ? a.tw0[(j - 1) * (L / R0) + t_in] : make_double2(1.0, 0.0);
          }
        } else {
          g0.chunk(t_in, c, w);
        }
        tmem_st4(ttw + 16 * c, w);
      }
#pragma unroll
      for (int c = 0; c < (R1 - 1 + 3) / 4; ++c) {
        cplx w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = COLW ? r16::colj(c, q) : 4 * c + q + 1;
          w[q] = (j > 0 && j < R1) ? a.tw1[(j * lo1) % TW1] : make_double2(1.0, 0.0);
        }
        tmem_st4(ttw1 + 16 * c, w);
      }
      tmem_wait_st();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  } else if constexpr (!(TWV & 1)) {
    // this thread's first-pass twiddles W_L^{j t} -> TMEM (same for every product)
    const fast::Tw0Global g0{a.tw0, L / R0, R0};
#pragma unroll
    for (int c = 0; c < (R0 - 1 + 3) / 4; ++c) {
      cplx w[4];
      g0.chunk(t_in, c, w);
      tmem_st4(ttw + 16 * c, w);
    }
    tmem_wait_st();
  }
  using TW0 = std::conditional_t<
      TW1T, Tw01TmemT<COLW>,
      std::conditional_t<(TWV & 1) != 0, fast::Tw0Rec,
                         std::conditional_t<(TWV & 4) != 0, Tw0Tmem8, Tw0Tmem>>>;
  TW0 tw0;
  if constexpr (TW1T)
    tw0 = TW0{ttw, ttw1};
  else if constexpr ((TWV & 1) != 0)
    tw0 = fast::Tw0Rec{a.tw};
  else
    tw0 = TW0{ttw};

  // Everything the loop needs is either a kernel parameter (read from the
  // constant bank at the point of use), a compile-time function of the group
  // index G, or the thread index: this keeps the 128-register budget for data.
  const long long nloc = a.batch > blockIdx.x
                             ? (a.batch - blockIdx.x + gridDim.x - 1) / gridDim.x
                             : 0;
  auto hptr = [&](long long k) {
    return static_cast<const cplx *>(a.h.ptr) +
           pp_off<XD>(a, blockIdx.x + k * gridDim.x, a.h.bstride, a.h.sstride);
  };
  auto xptr = [&](long long k) {
    return static_cast<const cplx *>(a.fac[0].ptr) +
           pp_off<XD>(a, blockIdx.x + k * gridDim.x, a.fac[0].bstride, a.fac[0].sstride);
  };
  auto h_prefetch = [&](long long k) {  // HD: generator k of this CTA into L2
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(hptr(k)),
                 "r"(((unsigned)a.h.len * 16u) & ~15u)
                 : "memory");
  };
  auto x_prefetch = [&](long long k) {  // XD: row k of this CTA into L2
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(xptr(k)),
                 "r"((unsigned)a.fac[0].len * 16u)
                 : "memory");
  };
  if (threadIdx.x == 0) {
    const uint32_t hbytes = (uint32_t)a.h.len * 16u, xbytes = (uint32_t)a.fac[0].len * 16u;
    if (nloc > 0) {
      if constexpr (HD) {
        h_prefetch(0);
        if (nloc > 1) h_prefetch(1);
      } else {
        mbar_expect_tx(mb_h0, hbytes);
        tma_load(smem_u32(hst), hptr(0), hbytes, mb_h0);
      }
      if constexpr (XD) {
        x_prefetch(0);
      } else {
        mbar_expect_tx(mb_x0, xbytes);
        tma_load(smem_u32(xst), xptr(0), xbytes, mb_x0);
      }
    }
    if (nloc > 1) {
      if constexpr (XD) {
        x_prefetch(1);
      } else {
        mbar_expect_tx(mb_x0 + 8, xbytes);
        tma_load(smem_u32(xst + XS), xptr(1), xbytes, mb_x0 + 8);
      }
    }
  }

  // lo-major pass 1 keeps the pass-1 <-> pass-2 exchanges inside each warp:
  // those barriers become warp syncs (fast::fft_dif / fft_final)
  using WS = std::conditional_t<TW1T, fast::WarpSync, void>;
  static_assert(!TW1T || (PL::radix[1] == PL::Rlast && 32 % PL::Rlast == 0),
                "warp-local exchange needs equal last two radices");
  // TWV bit 4: the two WAR barriers of a product (entries of the h and x
  // transforms) become split mbarrier arrive/wait pairs
  constexpr bool SPLIT = TW1T && (TWV & 16) != 0;
  using Entry = std::conditional_t<SPLIT, WarWait, fast::SyncEntry>;
  // TWV bit 5: both groups run ONE copy of the loop (runtime group index):
  // half the instruction footprint of the two compile-time copies
  auto run = [&](auto gc) {
    constexpr bool RT = (TWV & 32) != 0;
    const int G = RT ? g : decltype(gc)::value;
    auto h_entry = [&](int kk) {
      if constexpr (SPLIT)
        return Entry{mb_wh0 + 8 * G, (uint32_t)((kk - 1) & 1), kk > 0};
      else
        return Entry{};
    };
    auto x_entry = [&](int kk) {
      if constexpr (SPLIT)
        return Entry{mb_wx0 + 8 * G, (uint32_t)(kk & 1), true};
      else
        return Entry{};
    };
    const GroupBar<T> sync{1 + G};
    cplx *sbuf = ex + G * L;
    cplx *my_x = xst + G * XS;
    int kk = 0;
    for (long long k = G; k < nloc; k += 2, ++kk) {
      const uint32_t par = (uint32_t)(kk & 1);
      // A fresh opaque copy of the thread index per transform keeps the
      // compiler from hoisting / sharing the swizzled smem addresses of all
      // three transforms (cheap to recompute, ruinous to keep live: spills).
      auto fresh_t = [&]() {
        int x = t_in;
        asm volatile("" : "+r"(x));
        return x;
      };
      cplx v[V];
      // ---- S = ifft(h~) from staged h; release hst to the TMA for product k+1
      int t = fresh_t();
      if constexpr (HD) {
        // h straight from global (hoisted loads, L2-prefetched a product ahead)
        const cplx *hp = hptr(k);
        const int hlen = a.h.len;
        auto hl = [hp, hlen](int pos) {
          return pos < hlen ? fast::ld_stream(hp + pos) : make_double2(0.0, 0.0);
        };
        fast::fft_dif<PL, true, R0, TW1, REC>(
            sbuf, t, a.tw1, tw0, fast::Hoisted<decltype(hl)>{hl}, v, sync,
            [&]() {
              if (t == 0 && k + 2 < nloc) h_prefetch(k + 2);
            },
            (WS *)nullptr, h_entry(kk));
      } else {
        mbar_wait(mb_h0 + 8 * G, par);
        fast::fft_dif<PL, true, R0, TW1, REC>(
            sbuf, t, a.tw1, tw0, [&](int pos) { return hst[pos]; },
            v, sync, [&]() {
              if (t == 0 && k + 1 < nloc) {
                const uint32_t mb = mb_h0 + 8 * (1 - G);
                const uint32_t bytes = (uint32_t)a.h.len * 16u;
                fence_proxy_async();
                mbar_expect_tx(mb, bytes);
                tma_load(smem_u32(hst), hptr(k + 1), bytes, mb);
              }
            },
            (WS *)nullptr, h_entry(kk));
      }
      if constexpr (SPLIT) war_arrive(mb_wx0 + 8 * G);
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) tmem_st4(tacc + 16 * c, &v[4 * c]);
      // ---- X = fft(x~) from staged x; refill this group's xst with product k+2
      t = fresh_t();
      if constexpr (XD) {
        const cplx *xp = xptr(k);
        const int xlen = a.fac[0].len;
        auto xl = [xp, xlen](int pos) {
          return pos < xlen ? fast::ld_stream(xp + pos) : make_double2(0.0, 0.0);
        };
        fast::fft_dif<PL, false, NZ, TW1, REC>(
            sbuf, t, a.tw1, tw0, fast::Hoisted<decltype(xl)>{xl}, v, sync,
            [&]() {
              if (t == 0 && k + 2 < nloc) x_prefetch(k + 2);
            },
            (WS *)nullptr, x_entry(kk));
      } else {
        mbar_wait(mb_x0 + 8 * G, par);
        fast::fft_dif<PL, false, NZ, TW1, REC>(
            sbuf, t, a.tw1, tw0, [&](int pos) { return my_x[pos]; }, v,
            sync, [&]() {
              if (t == 0 && k + 2 < nloc) {
                const uint32_t mb = mb_x0 + 8 * G;
                const uint32_t bytes = (uint32_t)a.fac[0].len * 16u;
                fence_proxy_async();
                mbar_expect_tx(mb, bytes);
                tma_load(smem_u32(my_x), xptr(k + 2), bytes, mb);
              }
            },
            (WS *)nullptr, x_entry(kk));
      }
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) {
        cplx acc[4];
        tmem_ld4(tacc + 16 * c, acc);
        if (COLW && a.fac[0].power == 3) {
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] = cmul(acc[e], ccube(v[4 * c + e]));
        } else {
          for (int q = 0; q < a.fac[0].power; ++q) {
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] = cmul(acc[e], v[4 * c + e]);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) v[4 * c + e] = acc[e];
      }
      // ---- y = fft(acc)[:n_1]
      t = fresh_t();
      cplx *yk = static_cast<cplx *>(a.out) +
                 pp_off<XD>(a, blockIdx.x + k * gridDim.x, a.out_bstride, a.out_sstride);
      fast::fft_final<PL, NO, TW1, REC>(
          sbuf, t, a.tw1, tw0, v,
          [&](int pos, cplx val) {
            if (pos < a.out_len) yk[pos] = make_double2(val.x * a.scale, val.y * a.scale);
          },
          sync, (WS *)nullptr);
      if constexpr (SPLIT) war_arrive(mb_wh0 + 8 * G);
    }
  };
  if constexpr ((TWV & 32) != 0) {
    run(std::integral_constant<int, 0>{});
  } else {
    if (g == 0)
      run(std::integral_constant<int, 0>{});
    else
      run(std::integral_constant<int, 1>{});
  }

  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<512>(tmem_slot);
  }
}

template <class PL, int NZ, int NO, int TWV>
static cudaError_t launch_pp(const Args1D &a, cudaStream_t stream) {
  constexpr int XS = NZ >= PL::radix[0] ? 0 : NZ * PL::stride(0);
  const int smem = (3 * PL::L + 2 * XS) * (int)sizeof(cplx) + 128;
  static std::atomic<unsigned long long> configured{0};
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_pp<PL, NZ, NO, TWV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    configured.fetch_or(bit);
  }
  if (a.batch >= (1ll << 31) || a.nsub >= (1ll << 31)) return cudaErrorNotSupported;
  long long grid = sms[dev & 63];
  if (const char *e = getenv("HK_PP_GRID")) grid = atoi(e);
  if (grid > a.batch) grid = a.batch;
  if (grid <= 0) return cudaSuccess;
  k_hankel_pp<PL, NZ, NO, TWV><<<(unsigned)grid, 2 * PL::T, smem, stream>>>(a);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Batched short products (the 256-point row stage of the 2D block product,
// cfg4): the ping-pong structure with "units" of GP = 256 / T products per
// 256-thread group.  Each product's threads sit in one half-warp, so every
// exchange of its three transforms is a warp sync; the group meets only where
// the staging buffers change hands (after pass 0 of h and of x).
//   smem: ex[2][GP * L] | hst[GP * L] (h rows of one unit, shared in turn) |
//         xst[2][GP * XS] (x rows of this group's unit, XS = NZ * S0)
//   TMEM: cols [0, 256) accumulators; [256, 320) the pass-0 twiddles W_L^{j t}
//         (they depend on t = lane % T only: one slab for every warp)
struct WarpEntry {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.warp.sync -1;\n" ::: "memory"); }
};

// NG groups of 512/NG threads; NH h staging buffers (unit k uses hst[k % NH]
// and, once consumed, is refilled with unit k + NH for group (g + NH) % NG).
template <class PL, int NZ, int NO, int NG, int NH>
__global__ void __launch_bounds__(512, 1) k_rows_pp(const __grid_constant__ Args1D a) {
  constexpr int L = PL::L, T = PL::T, V = PL::V, R0 = PL::radix[0];
  constexpr int GT = 512 / NG;  // threads per group
  constexpr int GP = GT / T;    // products per group (one unit)
  constexpr int S0 = PL::stride(0);
  constexpr int XS = NZ * S0;
  static_assert(PL::P == 2 && 32 % T == 0 && T * GP == GT && NG % NH == 0,
                "two-pass plan, products within half-warps");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // full_h[NG], full_x[NG]: one barrier per GROUP (not per buffer), so a
  // waiter can never see a phase two completions old on a shared barrier
  __shared__ __align__(8) uint64_t mbar[2 * NG];
  __shared__ uint32_t tmem_slot;
  cplx *ex = reinterpret_cast<cplx *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  cplx *hst = ex + NG * GP * L;
  cplx *xst = hst + NH * GP * L;
  const int warp = threadIdx.x >> 5;
  const int g = threadIdx.x / GT;
  const int t_in = threadIdx.x % GT;
  const int sub = t_in / T, t = t_in % T;
  const uint32_t mb_h0 = smem_u32(&mbar[0]), mb_x0 = smem_u32(&mbar[NG]);
  // tails the TMA never writes: h rows past h.len, x rows past x.len
  for (int i = threadIdx.x; i < NH * GP * L; i += blockDim.x)
    if (i % L >= a.h.len) hst[i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < NG * GP * XS; i += blockDim.x)
    if (i % XS >= a.fac[0].len) xst[i] = make_double2(0.0, 0.0);
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2 * NG; ++i) mbar_init(smem_u32(&mbar[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;
  const uint32_t tacc = tmem_slot + lane_q + (uint32_t)((warp >> 2) * 64);
  const uint32_t ttw = tmem_slot + lane_q + 256u;
  if (warp < 4) {  // one twiddle slab per lane quadrant serves all warps
    const fast::Tw0Global g0{a.tw0, L / R0, R0};
#pragma unroll
    for (int c = 0; c < (R0 - 1 + 3) / 4; ++c) {
      cplx w[4];
      if constexpr (L == 256) {
        g0.chunk(t, c, w);
      } else {
        // plans without a thread-major first-pass table (192 = 16 x 12): W_L^{j t}
        // straight from the W_L table, once per CTA
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 4 * c + q + 1;
          w[q] = (j < R0 && t < L / R0) ? a.tw[(j * t) % L] : make_double2(1.0, 0.0);
        }
      }
      tmem_st4(ttw + 16 * c, w);
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const Tw0Tmem tw0{ttw};

  const long long nunits = (a.batch + GP - 1) / GP;
  const long long nloc = nunits > blockIdx.x ? (nunits - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto row_off = [&](long long b, long long bs, long long ss) {  // 32-bit: see launch_rows_pp
    const unsigned ob = (unsigned)b / (unsigned)a.nsub;
    return ob * bs + ((unsigned)b - ob * (unsigned)a.nsub) * ss;
  };
  struct Unit {
    long long b0;
    int nr;
  };
  auto unit_rows = [&](long long k) {  // first row and row count of unit k
    const long long b0 = (blockIdx.x + k * gridDim.x) * GP;
    return Unit{b0, (int)(a.batch - b0 < GP ? a.batch - b0 : GP)};
  };
  auto issue_h = [&](long long k) {  // unit k into hst[k % NH]
    const Unit u = unit_rows(k);
    const long long b0 = u.b0;
    const int nr = u.nr;
    const uint32_t bytes = (uint32_t)a.h.len * 16u;
    const uint32_t mb = mb_h0 + 8 * (uint32_t)(k % NG);  // the group of unit k
    cplx *dst = hst + (k % NH) * GP * L;
    mbar_expect_tx(mb, bytes * nr);
    for (int r = 0; r < nr; ++r)
      tma_load(smem_u32(dst + r * L),
               static_cast<const cplx *>(a.h.ptr) + row_off(b0 + r, a.h.bstride, a.h.sstride), bytes, mb);
  };
  auto issue_x = [&](long long k, cplx *dst, uint32_t mb) {
    const Unit u = unit_rows(k);
    const long long b0 = u.b0;
    const int nr = u.nr;
    const uint32_t bytes = (uint32_t)a.fac[0].len * 16u;
    mbar_expect_tx(mb, bytes * nr);
    for (int r = 0; r < nr; ++r)
      tma_load(smem_u32(dst + r * XS),
               static_cast<const cplx *>(a.fac[0].ptr) +
                   row_off(b0 + r, a.fac[0].bstride, a.fac[0].sstride),
               bytes, mb);
  };
  if (threadIdx.x == 0) {
    for (int k = 0; k < NH && k < nloc; ++k) issue_h(k);
    for (int k = 0; k < NG && k < nloc; ++k) issue_x(k, xst + k * GP * XS, mb_x0 + 8 * k);
  }

  const fast::WarpSync wsync;
  // staging hand-off at a group barrier after pass 0 (measured against
  // last-warp counters with fully warp-decoupled products: 922 vs 952 us, cfg4)
  // one-warp groups hand off at a warp sync (named barriers run out at 16)
  using GSync = std::conditional_t<GT == 32, fast::WarpSync, GroupBar<GT>>;
  GSync gsync;
  if constexpr (GT != 32) gsync = GSync{1 + g};
  cplx *sbuf = ex + g * GP * L + sub * L;
  cplx *my_x = xst + g * GP * XS;
  int kk = 0;
  for (long long k = g; k < nloc; k += NG, ++kk) {
    const uint32_t par = (uint32_t)(kk & 1);  // this group's kk-th unit
    const Unit un = unit_rows(k);
    const long long b0 = un.b0;
    const bool active = sub < un.nr;
    cplx v[V];
    // ---- S = ifft(h~) of this thread's row; hst goes to the TMA for unit k+1
    const cplx *hk = hst + (k % NH) * GP * L;
    mbar_wait(mb_h0 + 8 * g, par);
    fast::fft_dif<PL, true, R0>(
        sbuf, t, a.tw, tw0, [&](int pos) { return hk[sub * L + pos]; }, v, gsync,
        [&]() {
          if (k + NH < nloc && t_in == 0) {
            fence_proxy_async();
            issue_h(k + NH);
          }
        },
        (void *)nullptr, WarpEntry{});
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) tmem_st4(tacc + 16 * c, &v[4 * c]);
    // ---- X = fft(x~); this group's xst is refilled with unit k+2
    mbar_wait(mb_x0 + 8 * g, par);
    fast::fft_dif<PL, false, NZ>(
        sbuf, t, a.tw, tw0, [&](int pos) { return my_x[sub * XS + pos]; }, v, gsync,
        [&]() {
          if (k + NG < nloc && t_in == 0) {
            fence_proxy_async();
            issue_x(k + NG, my_x, mb_x0 + 8 * g);
          }
        },
        (void *)nullptr, WarpEntry{});
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) {
      cplx acc[4];
      tmem_ld4(tacc + 16 * c, acc);
      for (int q = 0; q < a.fac[0].power; ++q) {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = cmul(acc[e], v[4 * c + e]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) v[4 * c + e] = acc[e];
    }
    // ---- y = fft(acc)[:n_1] (warp-local exchanges only)
    cplx *yk = static_cast<cplx *>(a.out) + row_off(b0 + sub, a.out_bstride, a.out_sstride);
    fast::fft_final<PL, NO>(
        sbuf, t, a.tw, tw0, v,
        [&](int pos, cplx val) {
          if (active && pos < a.out_len) yk[pos] = make_double2(val.x * a.scale, val.y * a.scale);
        },
        wsync);
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<512>(tmem_slot);
  }
}

template <class PL, int NZ, int NO, int NG, int NH>
static cudaError_t launch_rows_pp(const Args1D &a, cudaStream_t stream) {
  constexpr int GP = 512 / NG / PL::T;
  constexpr int XS = NZ * PL::stride(0);
  const int smem = ((NG + NH) * GP * PL::L + NG * GP * XS) * (int)sizeof(cplx) + 128;
  static std::atomic<unsigned long long> configured{0};
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_rows_pp<PL, NZ, NO, NG, NH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    configured.fetch_or(bit);
  }
  if (a.batch >= (1ll << 31) || a.nsub >= (1ll << 31)) return cudaErrorNotSupported;
  const long long units = (a.batch + GP - 1) / GP;
  long long grid = std::min<long long>(units, sms[dev & 63]);
  if (grid <= 0) return cudaSuccess;
  k_rows_pp<PL, NZ, NO, NG, NH><<<(unsigned)grid, 512, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace pp

// 256-point batched rows (2D block row stage) on the ping-pong kernel.
static cudaError_t launch_pp_256(const Args1D &a, cudaStream_t stream) {
  if (getenv("HK_NO_PP256")) return cudaErrorNotSupported;
  if (a.mode != M_PARTIAL || a.nfac != 1 || !a.tw0 || a.nsub < 1 || a.ncombo)
    return cudaErrorNotSupported;
  const Factor &h = a.h, &x = a.fac[0];
  if (h.kind != FK_C128 || x.kind != FK_C128 || h.estride != 1 || x.estride != 1 ||
      a.out_estride != 1 || h.len > 256 || h.len <= 0 || x.len <= 0 || x.len > 64)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(h.ptr) | reinterpret_cast<uintptr_t>(x.ptr)) & 15)
    return cudaErrorNotSupported;
  using PL = Plan1D<256, 16, 16, 16>;
  const int no = (a.out_len + 15) / 16;
  // Groups of the row kernel (B200 cfg4, us): 2 x 256 threads / 1 h buffer
  // 918, 4 x 128 / 2 buffers 890, 8 x 64 / 4 buffers 840, 16 one-warp groups /
  // 8 buffers 784 (default; HK_ROWS_NG selects the others for A/B)
  const int ng = getenv("HK_ROWS_NG") ? atoi(getenv("HK_ROWS_NG")) : 16;
  if (no <= 4) {
    if (ng == 2) return pp::launch_rows_pp<PL, 4, 4, 2, 1>(a, stream);
    if (ng == 4) return pp::launch_rows_pp<PL, 4, 4, 4, 2>(a, stream);
    if (ng == 8) return pp::launch_rows_pp<PL, 4, 4, 8, 4>(a, stream);
    return pp::launch_rows_pp<PL, 4, 4, 16, 8>(a, stream);
  }
  return pp::launch_rows_pp<PL, 4, 16, 16, 8>(a, stream);
}

// 192-point batched rows (2D block row stage at the exact padded length
// 192 >= d_in = 190 instead of 256): 16 threads per product as for 256, 12
// values per thread, radix 16 then radix 12 (12 of the 16 threads run the
// radix-16 pass; every thread one radix-12 butterfly).
static cudaError_t launch_pp_192(const Args1D &a, cudaStream_t stream) {
  if (a.mode != M_PARTIAL || a.nfac != 1 || !a.tw || a.nsub < 1 || a.ncombo)
    return cudaErrorNotSupported;
  const Factor &h = a.h, &x = a.fac[0];
  if (h.kind != FK_C128 || x.kind != FK_C128 || h.estride != 1 || x.estride != 1 ||
      a.out_estride != 1 || h.len > 192 || h.len <= 0 || x.len <= 0 || x.len > 72 ||
      a.out_len > 72)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(h.ptr) | reinterpret_cast<uintptr_t>(x.ptr)) & 15)
    return cudaErrorNotSupported;
  using PL = Plan1D<192, 16, 16, 12>;
  return pp::launch_rows_pp<PL, 6, 6, 16, 8>(a, stream);
}

// Ping-pong TMA path; cudaErrorNotSupported unless the request is the plain
// batched H x^{m-1} shape it implements.
cudaError_t launch_pp_1d(int L, const Args1D &a, cudaStream_t stream) {
  if (getenv("HK_NO_PP")) return cudaErrorNotSupported;
  if (L == 256) return launch_pp_256(a, stream);
  if (L == 192 && getenv("HK_PP192")) return launch_pp_192(a, stream);
  if (L != 4096 || a.mode != M_PARTIAL || a.nfac != 1 || !a.tw0 || a.nsub < 1 || a.ncombo)
    return cudaErrorNotSupported;
  const Factor &h = a.h, &x = a.fac[0];
  if (h.kind != FK_C128 || x.kind != FK_C128 || h.estride != 1 || x.estride != 1 ||
      a.out_estride != 1)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(h.ptr) | reinterpret_cast<uintptr_t>(x.ptr)) & 15)
    return cudaErrorNotSupported;
  if (h.len > L || h.len <= 0 || x.len <= 0 || !a.tw1) return cudaErrorNotSupported;
  using PL = Plan1D<4096, 256, 16, 16, 16>;
  constexpr int s0 = PL::stride(0);
  const int nz = (x.len + s0 - 1) / s0, no = (a.out_len + s0 - 1) / s0;
  // 24: TMEM pass-0 and pass-1 twiddles + split WAR barriers (r02: 169.4 us vs
  // 170.0 for 8 and 185.6 for 2 = recurrence for pass 1, the r01 default);
  // +128: column-major twiddle chunks folded into the final transform's first
  // radix-4 stages, cube in six instructions (HK_PP_COLW=0 turns it off)
  const bool colw = !(getenv("HK_PP_COLW") && atoi(getenv("HK_PP_COLW")) == 0);
  int twv = colw ? 152 : 24;
  if (const char *e = getenv("HK_PP_TWV")) twv = atoi(e) & 255;
  if (nz == 16 && !getenv("HK_NO_PP_ROWS")) {  // full rows (two-level row stage)
    const bool one = getenv("HK_PP_ROWS_TWO") == nullptr;  // A/B: two code copies
    if (!one) return no <= 4 ? pp::launch_pp<PL, 16, 4, 24>(a, stream) : pp::launch_pp<PL, 16, 16, 24>(a, stream);
    if (colw) return no <= 4 ? pp::launch_pp<PL, 16, 4, 184>(a, stream) : pp::launch_pp<PL, 16, 16, 184>(a, stream);
    return no <= 4 ? pp::launch_pp<PL, 16, 4, 56>(a, stream) : pp::launch_pp<PL, 16, 16, 56>(a, stream);
  }
  if (nz <= 4 && no <= 4 && a.nsub == 1) {
    switch (twv) {
      case 8: return pp::launch_pp<PL, 4, 4, 8>(a, stream);
      case 24: return pp::launch_pp<PL, 4, 4, 24>(a, stream);
      case 56: return pp::launch_pp<PL, 4, 4, 56>(a, stream);
      case 88: return pp::launch_pp<PL, 4, 4, 88>(a, stream);
      case 152: return pp::launch_pp<PL, 4, 4, 152>(a, stream);
      default: return pp::launch_pp<PL, 4, 4, 2>(a, stream);
    }
  }
  return cudaErrorNotSupported;  // x staging would not fit next to three L buffers
}

}  // namespace hk
