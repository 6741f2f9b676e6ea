// K1/K2 fast path (kernel template; instantiated per FFT length in
// hk_fast_*.cu so the lengths compile in parallel): fused batched 1D Hankel
// products with a TMEM-resident spectral accumulator, pruned first/last
// passes and conflict-free, low-traffic twiddle access.
//
// Per product (reference hankel.py:140-154 via hankel.py:42-71):
//   acc  = ifft(h~)                        -> TMEM
//   for each distinct vector factor f:     (H x^{m-1}: one factor, power m-1)
//       X = fft(x~_f)   (first pass pruned to the n_f/s_0 nonzero inputs)
//       acc = acc .* X .* ... .* X         (TMEM chunk by chunk; reference order)
//   partial: y = fft(acc)[:n_1]            (transposed network, last pass pruned
//                                           to the n_1/s_0 needed outputs)
//   full:    alpha = sum(acc)              (fixed-order reduction)
//
// Differences from the generic kernel (hk_1d.cu):
//  * acc lives in TMEM, so only one length-L working set is in registers;
//  * twiddles: one table read per butterfly (pass 0: one per thread, the NB
//    butterflies' bases follow by constant factors), the R-1 powers by a
//    two-chain recurrence (fast::twiddle_rec) -- measured faster on B200 than
//    the earlier thread-major pass-0 table and per-twiddle reads;
//  * the smem swizzle XORs the low 3 position bits with bits 4-6 ^ 8-10, which
//    keeps every 8-lane phase of every pass on distinct 16 B bank groups;
//  * optional cp.async staging of the next item's pass-0 operands (STG) and
//    regrouping of small products into multi-product CTAs (Regroup).
#pragma once

#include <atomic>
#include <stdio.h>
#include <stdlib.h>

#include "hk_fastcore.cuh"

namespace hk {
namespace fast {

// Twiddles of passes >= 1 by recurrence from one table read per butterfly
// (fast::twiddle_rec); measured on B200 against per-twiddle L1 reads.
constexpr bool kRec = true;
// Pass-0 twiddles by recurrence from W_L^beta (else the thread-major table).
constexpr bool kTw0Rec = true;

// L2 prefetch (cp.async.bulk.prefetch.L2) of one operand item, if contiguous.
__device__ __forceinline__ void prefetch_item(const Factor &f, long long b, long long nsub,
                                              int kind_bytes) {
  if (f.kind == FK_SPEC || f.estride != 1 || f.len <= 0) return;
  long long ob, os;
  split_item(b, nsub, ob, os);
  const char *p = static_cast<const char *>(f.ptr) + (ob * f.bstride + os * f.sstride) * kind_bytes;
  unsigned bytes = (unsigned)f.len * (unsigned)kind_bytes;
  // 16-byte aligned start and size
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0))
               : "memory");
}

__device__ __forceinline__ void prefetch_block(const Args1D &a, long long bb, int G) {
  for (int g = 0; g < G; ++g) {
    const long long b = bb * G + g;
    if (b >= a.batch) break;
    prefetch_item(a.h, b, a.nsub, a.h.kind == FK_F64 ? 8 : 16);
    for (int f = 0; f < a.nfac; ++f)
      prefetch_item(a.fac[f], b, a.nsub, a.fac[f].kind == FK_F64 ? 8 : 16);
  }
}

// Plan with an explicit number of products per CTA (smaller CTAs leave room
// for the staging slots while keeping several CTAs resident per SM).
template <class PL, int G_>
struct Regroup : PL {
  static constexpr int G = G_;
  static constexpr int CTA = G_ * PL::T;
  static constexpr int kStagedBlocks = G_ >= 8 ? 3 : 24 / G_;  // resident CTAs with staging
  static constexpr int SMEM_BYTES = G_ * PL::L * (int)sizeof(cplx);
  static_assert(CTA % 32 == 0, "whole warps");
};

// Staging geometry: the pass-0 inputs of one thread are NB0 butterflies of R0
// (h) or NZ (first vector factor) elements at pos = beta + j * s0.
template <class PL, int NZ>
struct Stage {
  static constexpr int S0 = PL::stride(0);
  static constexpr int NB0 = (S0 + PL::T - 1) / PL::T;
  static constexpr int SH = NB0 * PL::radix[0];
  static constexpr int SX = NB0 * NZ;
  static constexpr int BYTES = (SH + SX) * PL::CTA * (int)sizeof(cplx);
};

template <class T, class = void>
struct requires_staged_blocks : std::false_type {};
template <class T>
struct requires_staged_blocks<T, std::void_t<decltype(T::kStagedBlocks)>> : std::true_type {};

template <class PL, bool STG>
constexpr int min_blocks_for() {
  if constexpr (STG) {
    if constexpr (requires_staged_blocks<PL>::value) return PL::kStagedBlocks;
    return 3;
  }
  return Traits<PL>::min_blocks;
}

// STG: the next item's pass-0 operands (h and the first vector factor, raw
// c128/f64) are copied into per-thread shared-memory slots with cp.async
// while the current item computes.  A thread only ever reads the slots it
// filled itself, so the staging needs cp.async.wait_all and no barrier; the
// copies for item k+1 are issued right after pass 0 of item k has consumed
// the slots (the hook that runs behind the first exchange barrier).
template <class PL, int NZ, int NO, bool STG = false>
__global__ void __launch_bounds__(PL::CTA, (min_blocks_for<PL, STG>()))
    k_hankel_fast(const __grid_constant__ Args1D a) {
  using Tr = Traits<PL>;
  constexpr int T = PL::T;
  constexpr int V = PL::V;
  constexpr int COLS = Tr::tmem_cols;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplx *smem = reinterpret_cast<cplx *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<COLS>(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tmem_slot;
  const uint32_t tmy = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 4 * V);

  const int g = threadIdx.x / T;
  const int t = threadIdx.x - g * T;
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  cplx *sbuf = smem + g * PL::L;
  const cplx *__restrict__ tw = a.tw;
  using TW0 = std::conditional_t<kTw0Rec, Tw0Rec, Tw0Global>;
  TW0 tw0;
  if constexpr (kTw0Rec)
    tw0 = Tw0Rec{a.tw};
  else
    tw0 = Tw0Global{a.tw0, PL::L / PL::radix[0], PL::radix[0]};
  const GroupSync<PL> gsync;
  // one product per CTA with several pass-0 butterflies per thread (8192):
  // issue all of a thread's operand loads before its butterflies
  auto hoist_if_big = [](auto f) {
    if constexpr (PL::T >= 512)
      return Hoisted<decltype(f)>{f};
    else
      return f;
  };
  const bool do_pf = a.prefetch != 0;
  if (do_pf && threadIdx.x == 0) prefetch_block(a, blockIdx.x, PL::G);

  using St = Stage<PL, NZ>;
  constexpr int R0 = PL::radix[0];
  const uint32_t stg = smem_u32(smem + PL::G * PL::L) + 16u * threadIdx.x;
  auto slot = [&](int k) { return stg + (uint32_t)(k * PL::CTA * (int)sizeof(cplx)); };
  // copy the pass-0 inputs of operand f for block bb into slots k0..
  auto stage_issue = [&](const Factor &f, long long bb, int k0, int nin, int fac_idx) {
    long long b = bb * PL::G + g;
    if (b >= a.batch) b = a.batch - 1;
    long long ob, os;
    split_item(b, a.nsub, ob, os);
    const long long col = (fac_idx >= 0 && a.ncombo) ? (long long)a.combo_col[os][fac_idx] : os;
    const long long off = ob * f.bstride + col * f.sstride;
    const bool f64 = f.kind == FK_F64;
#pragma unroll
    for (int i = 0; i < St::NB0; ++i) {
      const int beta = t + i * T;
      if (St::S0 % T == 0 || beta < St::S0) {
#pragma unroll
        for (int j = 0; j < nin; ++j) {
          const int pos = beta + j * St::S0;
          const bool ok = pos < f.len;
          const long long e = off + (ok ? (long long)pos * f.estride : 0);
          if (f64)
            cpa8(slot(k0 + i * nin + j), static_cast<const double *>(f.ptr) + e, ok);
          else
            cpa16(slot(k0 + i * nin + j), static_cast<const cplx *>(f.ptr) + e, ok);
        }
      }
    }
  };
  auto stage_read = [&](int k, bool f64, double sc) {
    double x, y;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(slot(k)) : "memory");
    if (f64) y = 0.0;
    return make_double2(x * sc, y * sc);
  };
  if constexpr (STG) {
    stage_issue(a.h, blockIdx.x, 0, R0, -1);
    stage_issue(a.fac[0], blockIdx.x, St::SH, NZ, 0);
    cpa_commit();
  }

  // persistent loop: block bb handles products bb*G .. bb*G+G-1
  for (long long bb = blockIdx.x; bb < nblk; bb += gridDim.x) {
    // Warp-synchronous groups never meet at a CTA barrier inside the FFTs; left
    // alone the scheduler lets some warps run far ahead, and the kernel ends
    // with a long tail of few resident warps.  One barrier per item bounds it.
    if constexpr (std::is_same_v<GroupSync<PL>, WarpSync>) {
      if (bb != blockIdx.x) __syncthreads();
    }
    // stream the NEXT block's inputs into L2 while this one computes
    if (do_pf && threadIdx.x == 0 && bb + gridDim.x < nblk) prefetch_block(a, bb + gridDim.x, PL::G);
    long long b = bb * PL::G + g;
    const bool active = b < a.batch;
    if (!active) b = a.batch - 1;
    long long ob, os;
    split_item(b, a.nsub, ob, os);

    cplx v[V];
    cplx *out = static_cast<cplx *>(a.out) + ob * a.out_bstride +
                (a.ncombo ? (long long)a.combo_out[os] : os * a.out_sstride);
    if (a.mode == M_SPEC_F) {  // column spectra: X = fft(x~) in internal layout
      const Factor &fa = a.fac[0];
      const long long off = ob * fa.bstride + os * fa.sstride;
      fft_dif<PL, false, PL::radix[0], PL::L, kRec>(sbuf, t, tw, tw0,
                                       [&](int pos) { return load_elem(fa, off, pos, 1.0); }, v, gsync);
      if (active) {
#pragma unroll
        for (int r = 0; r < V; ++r) out[r * T + t] = v[r];
      }
      continue;
    }
    // ---- acc = ifft(h~) (or cached spectrum) -> TMEM
    {
      const Factor &hf = a.h;
      const long long off = ob * hf.bstride + os * hf.sstride;
      if (hf.kind == FK_SPEC) {
        const cplx *sp = static_cast<const cplx *>(hf.ptr) + off;
#pragma unroll
        for (int r = 0; r < V; ++r) v[r] = __ldg(sp + r * T + t);
      } else if constexpr (STG) {
        cpa_wait_all();  // this thread's copies for the current block have landed
        const double sc = a.scale;
        const bool f64 = hf.kind == FK_F64;
        fft_dif<PL, true, PL::radix[0], PL::L, kRec>(
            sbuf, t, tw, tw0,
            [&](int i, int j, int) { return stage_read(i * R0 + j, f64, sc); }, v, gsync,
            [&]() {
              if (bb + gridDim.x < nblk) stage_issue(hf, bb + gridDim.x, 0, R0, -1);
            });
      } else {
        const double sc = a.scale;
        fft_dif<PL, true, PL::radix[0], PL::L, kRec>(
            sbuf, t, tw, tw0, hoist_if_big([&](int pos) { return load_elem(hf, off, pos, sc); }),
            v, gsync);
      }
      if (a.mode == M_SPEC_H) {
        if (active) {
#pragma unroll
          for (int r = 0; r < V; ++r) out[r * T + t] = v[r];
        }
        continue;
      }
      tmem_wait_st();  // previous product's final reads of TMEM are complete
#pragma unroll
      for (int c = 0; c < V / 4; ++c) tmem_st4(tmy + 16 * c, &v[4 * c]);
    }
    // ---- acc .*= fft(x~_f)^{p_f}
    for (int f = 0; f < a.nfac; ++f) {
      const Factor &fa = a.fac[f];
      const long long off = ob * fa.bstride +
                            (a.ncombo ? (long long)a.combo_col[os][f] : os) * fa.sstride;
      if (fa.kind == FK_SPEC) {
        const cplx *sp = static_cast<const cplx *>(fa.ptr) + off;
#pragma unroll
        for (int r = 0; r < V; ++r) v[r] = __ldg(sp + r * T + t);
      } else if (STG && f == 0) {
        const bool f64 = fa.kind == FK_F64;
        fft_dif<PL, false, NZ, PL::L, kRec>(
            sbuf, t, tw, tw0,
            [&](int i, int j, int) { return stage_read(St::SH + i * NZ + j, f64, 1.0); }, v,
            gsync, [&]() {
              if (bb + gridDim.x < nblk) stage_issue(fa, bb + gridDim.x, St::SH, NZ, 0);
              cpa_commit();
            });
      } else {
        fft_dif<PL, false, NZ, PL::L, kRec>(
            sbuf, t, tw, tw0, hoist_if_big([&](int pos) { return load_elem(fa, off, pos, 1.0); }),
            v, gsync);
      }
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) {
        cplx acc[4];
        tmem_ld4(tmy + 16 * c, acc);
        for (int k = 0; k < fa.power; ++k) {
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = cmul(acc[q], v[4 * c + q]);
        }
        tmem_st4(tmy + 16 * c, acc);
      }
    }
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) tmem_ld4(tmy + 16 * c, &v[4 * c]);

    cplx *out2 = (a.ncombo && a.combo_out2[os] >= 0)
                     ? static_cast<cplx *>(a.out) + ob * a.out_bstride + a.combo_out2[os]
                     : nullptr;
    if (a.mode == M_PARTIAL) {
      const int n1 = a.out_len;
      const long long es = a.out_estride;
      fft_final<PL, NO, PL::L, kRec>(
          sbuf, t, tw, tw0, v,
          [&](int pos, cplx val) {
            if (active && pos < n1) {
              out[pos * es] = val;
              if (out2) out2[pos * es] = val;
            }
          },
          gsync);
    } else {
      cplx s = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < V; ++r) s = cadd(s, v[r]);
      gsync();
      cplx *red = sbuf;  // this group's own exchange buffer: other groups may still be mid-FFT
      red[t] = s;
      gsync();
      if (t == 0 && active) {
        cplx tot = make_double2(0.0, 0.0);
        for (int k = 0; k < T; ++k) tot = cadd(tot, red[k]);
        out[0] = tot;
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<COLS>(tbase);
  }
}

template <class PL, int NZ, int NO, bool STG = false>
static cudaError_t launch_variant(const Args1D &a, cudaStream_t stream) {
  const int smem = PL::G * PL::L * (int)sizeof(cplx) + (STG ? Stage<PL, NZ>::BYTES : 0) + 128;
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_fast<PL, NZ, NO, STG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // Carve out just enough shared memory for the target residency; the rest
    // stays L1 for the twiddle tables.
    const int want = min_blocks_for<PL, STG>() * (smem + 2048);
    const int pct = (want * 100 + 228 * 1024 - 1) / (228 * 1024);
    e = cudaFuncSetAttribute(k_hankel_fast<PL, NZ, NO, STG>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  if (nblk <= 0) return cudaSuccess;
  static int resident[64] = {0};
  int &res = resident[dev & 63];
  if (res == 0) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hankel_fast<PL, NZ, NO, STG>, PL::CTA,
                                                  smem);
    // The occupancy API under-reports here; derive residency from the limits.
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_hankel_fast<PL, NZ, NO, STG>);
    int smem_sm = 0, regs_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int by_regs = regs_sm / (((fa.numRegs + 7) / 8 * 8) * PL::CTA);
    const int by_smem = smem_sm / (smem + (int)fa.sharedSizeBytes + 1024);
    const int by_thr = 2048 / PL::CTA;
    int mine = by_regs < by_smem ? by_regs : by_smem;
    mine = mine < by_thr ? mine : by_thr;
    if (mine > per_sm) per_sm = mine;
    res = sms * (per_sm > 0 ? per_sm : 1);
    if (const char *e = getenv("HK_DEBUG_GRID")) {
      fprintf(stderr, "[hk] fast L=%d sms=%d per_sm=%d grid=%d smem=%d\n", PL::L, sms, per_sm,
              res, smem);
      if (atoi(e) > 0) res = atoi(e);
    }
  }
  const long long grid = nblk < res ? nblk : res;
  k_hankel_fast<PL, NZ, NO, STG><<<(unsigned)grid, PL::CTA, smem, stream>>>(a);
  return cudaGetLastError();
}

// Choose the smallest instantiated pruning level covering the request.
template <int I, int N, class F>
static void hfor_impl(F &&f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    hfor_impl<I + 1, N>(f);
  }
}
template <int N, class F>
static void hfor(F &&f) { hfor_impl<0, N>(f); }

template <class PL, int... Ls>
struct Pruned {
  static constexpr int n = sizeof...(Ls);
  static constexpr int lv[n] = {Ls...};
  static int pick(int want) {
    for (int i = 0; i < n; ++i)
      if (want <= lv[i]) return i;
    return n - 1;
  }
  template <bool STG = false>
  static cudaError_t launch(const Args1D &a, cudaStream_t stream, int nz, int no) {
    const int zi = pick(nz), oi = pick(no);
    cudaError_t r = cudaErrorInvalidValue;
    hfor<n>([&](auto zc) {
      hfor<n>([&](auto oc) {
        constexpr int Z = decltype(zc)::value, O = decltype(oc)::value;
        if (Z == zi && O == oi) r = launch_variant<PL, lv[Z], lv[O], STG>(a, stream);
      });
    });
    return r;
  }
};

}  // namespace fast

// Per-length launchers (hk_fast_<L>.cu).  maxlen = longest raw vector
// operand (nonzero prefix), outl = outputs kept; they set the first-pass /
// last-pass pruning levels.
cudaError_t launch_fast_4096(const Args1D &a, cudaStream_t s, int maxlen, int outl);
cudaError_t launch_fast_6144(const Args1D &a, cudaStream_t s, int maxlen, int outl);
cudaError_t launch_fast_256(const Args1D &a, cudaStream_t s, int maxlen, int outl, bool staged);
cudaError_t launch_fast_small(int L, const Args1D &a, cudaStream_t s, int maxlen, int outl);
cudaError_t launch_fast_8192(const Args1D &a, cudaStream_t s);

}  // namespace hk
