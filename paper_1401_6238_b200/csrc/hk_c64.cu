// complex64 / float32 variant of the fused batched 1D Hankel products
// (north_star: relative error <= 1e-4 for fp32/complex64).  Same algorithm
// as the complex128 kernels (reference hankel.py:140-154 via the
// anti-circulant embedding, hankel.py:42-71), FP32 arithmetic throughout:
//   acc = ifft(h~)                 (pass 0 reads the nonzero h prefix only)
//   acc *= fft(x~_f)^{power_f}     (one transform per DISTINCT vector; the
//                                   reference's multiplication order)
//   partial: y = fft(acc)[:n_1]    (transposed network, natural-order output)
//   full:    alpha = sum(acc)      (fixed-order reduction)
// The reference itself is complex128-only (core.py:21-22); this is the
// batched-API extension SURVEY §7 step 8 / §8(b) list as HK_C64 / HK_F32.
//
// Three kernels: the generic and fast kernels below (several products per SM,
// latency hidden by occupancy) and, for the batched L = 4096 headline shape,
// the ping-pong kernel at the end of this file (two product groups per SM,
// cp.async staging a product ahead, TMEM twiddles).
//
// Design of the first two: half the bytes of a complex128 working set, so the accumulator and
// one vector spectrum both stay in registers (no TMEM needed) and the FP32
// pipe (2x the FP64 rate on B200) does the butterflies.  Latency is hidden by
// occupancy: several independent products per SM, each a CTA group of T
// threads exchanging through its own 8-byte-swizzled shared-memory buffer.
// Twiddles come from an L1-resident single-precision table computed in long
// double on the host.
#include <atomic>
#include <stdlib.h>

#include "hk_fastcore.cuh"
#include "hk_fft1d.cuh"
#include "hk_internal.h"
#include "hk_tmem.cuh"

#ifndef HK_C64_MINB
#define HK_C64_MINB 4  // resident CTAs/SM of the 256-thread fast complex64 kernel
#endif

namespace hk {

using cplxf = float2;

__device__ __forceinline__ cplxf ld_c64(const Factor &f, long long off, int pos, float scale) {
  if (pos >= f.len) return make_float2(0.f, 0.f);
  const long long k = (long long)pos * f.estride;
  if (f.kind == FK_F32) {
    const float *p = static_cast<const float *>(f.ptr) + off;
    return make_float2(__ldg(p + k) * scale, 0.f);
  }
  const cplxf *p = static_cast<const cplxf *>(f.ptr) + off;
  const cplxf v = __ldg(p + k);
  return make_float2(v.x * scale, v.y * scale);
}

// The accumulator lives in TMEM (as in the complex128 fast kernel) for plans
// with V >= 8 values per thread, so only one length-L working set is in
// registers while the next spectrum is computed; tiny plans keep it in
// registers.  Warp w owns TMEM lanes 32*(w%4).. and a 2V-column slab w/4.
template <class PL>
struct C64Tr {
  static constexpr bool tmem = PL::V >= 8 && PL::V % 4 == 0;
  static constexpr int warps = PL::CTA / 32;
  static constexpr int slabs = (warps + 3) / 4;
  static constexpr int need = slabs * 2 * PL::V;
  static constexpr int cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : 256;
  static constexpr int min_blocks = PL::CTA >= 384 ? 1 : 2;
};

template <class PL>
__global__ void __launch_bounds__(PL::CTA, (C64Tr<PL>::min_blocks))
    k_hankel_c64(const __grid_constant__ Args1D a) {
  using Tr = C64Tr<PL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplxf *smem = reinterpret_cast<cplxf *>(smem_raw);
  constexpr int T = PL::T;
  constexpr int V = PL::V;
  const int g = threadIdx.x / T;
  const int t = threadIdx.x - g * T;
  const int warp = threadIdx.x >> 5;
  cplxf *sbuf = smem + (PL::P > 1 ? g * PL::L : 0);
  const cplxf *__restrict__ tw = a.twf;
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  uint32_t tmy = 0;
  if constexpr (Tr::tmem) {
    if (warp == 0) tmem_alloc<Tr::cols>(&tmem_slot);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tmy = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 2 * V);
  }

  for (long long bb = blockIdx.x; bb < nblk; bb += gridDim.x) {
    long long b = bb * PL::G + g;
    const bool active = b < a.batch;
    if (!active) b = a.batch - 1;  // idle groups shadow a valid item; stores are masked
    long long ob, os;
    split_item(b, a.nsub, ob, os);

    cplxf acc[Tr::tmem ? 1 : V];
    cplxf v[V];
    {
      const Factor &hf = a.h;
      const float sc = (float)a.scale;
      const long long off = ob * hf.bstride + os * hf.sstride;
      fft_dif<PL, true>(sbuf, t, tw, [&](int pos) { return ld_c64(hf, off, pos, sc); }, v);
      if constexpr (Tr::tmem) {
        tmem_wait_st();  // the previous item's reads of TMEM are complete
#pragma unroll
        for (int c = 0; c < V / 4; ++c) tmem_st4f(tmy + 8 * c, &v[4 * c]);
      } else {
#pragma unroll
        for (int r = 0; r < V; ++r) acc[r] = v[r];
      }
    }
    for (int f = 0; f < a.nfac; ++f) {
      const Factor &fa = a.fac[f];
      const long long off = ob * fa.bstride + os * fa.sstride;
      fft_dif<PL, false>(sbuf, t, tw, [&](int pos) { return ld_c64(fa, off, pos, 1.f); }, v);
      if constexpr (Tr::tmem) {
        tmem_wait_st();
#pragma unroll
        for (int c = 0; c < V / 4; ++c) {
          cplxf q[4];
          tmem_ld4f(tmy + 8 * c, q);
          for (int k = 0; k < fa.power; ++k) {
#pragma unroll
            for (int i = 0; i < 4; ++i) q[i] = cmul(q[i], v[4 * c + i]);
          }
          tmem_st4f(tmy + 8 * c, q);
        }
      } else {
        for (int k = 0; k < fa.power; ++k) {
#pragma unroll
          for (int r = 0; r < V; ++r) acc[r] = cmul(acc[r], v[r]);
        }
      }
    }
    if constexpr (Tr::tmem) {
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) tmem_ld4f(tmy + 8 * c, &v[4 * c]);
    } else {
#pragma unroll
      for (int r = 0; r < V; ++r) v[r] = acc[r];
    }
    cplxf *out = static_cast<cplxf *>(a.out) + ob * a.out_bstride + os * a.out_sstride;
    if (a.mode == M_PARTIAL) {
      const int n1 = a.out_len;
      const long long es = a.out_estride;
      fft_dit_final<PL>(sbuf, t, tw, v, [&](int pos, cplxf y) {
        if (active && pos < n1) out[pos * es] = y;
      });
    } else {
      cplxf s = make_float2(0.f, 0.f);
#pragma unroll
      for (int r = 0; r < V; ++r) s = cadd(s, v[r]);
      __syncthreads();
      cplxf *red = smem + g * T;  // G*T <= G*L slots
      red[t] = s;
      __syncthreads();
      if (t == 0 && active) {
        cplxf tot = make_float2(0.f, 0.f);
        for (int k = 0; k < T; ++k) tot = cadd(tot, red[k]);
        out[0] = tot;
      }
    }
    __syncthreads();  // the exchange buffers are reused by the next item
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

// Resident CTAs on the whole GPU for a persistent grid, from the register,
// shared-memory and thread limits (the occupancy API under-reports for these
// kernels, as for the complex128 fast kernel: it returned 1 CTA/SM here).
static int resident_ctas(const void *fn, int cta, int smem, int dev) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fn);
  int sms = 0, smem_sm = 0, regs_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  int per = regs_sm / (((fa.numRegs + 7) / 8 * 8) * cta);
  const int by_smem = smem_sm / (smem + (int)fa.sharedSizeBytes + 1024);
  per = per < by_smem ? per : by_smem;
  per = per < 2048 / cta ? per : 2048 / cta;
  return sms * (per > 0 ? per : 1);
}

// ---------------------------------------------------------------------------
// Fast variant for the batched lengths (the complex128 fast kernel's engine,
// hk_fastcore.cuh, instantiated on float2): pruned first/last passes,
// recurrence twiddles from one table read per butterfly, 8-byte swizzled
// exchanges, TMEM accumulator, L2 prefetch of the next block's operands.
__device__ __forceinline__ void prefetch_f(const Factor &f, long long b, long long nsub) {
  if (f.estride != 1 || f.len <= 0) return;
  const int eb = f.kind == FK_F32 ? 4 : 8;
  long long ob, os;
  split_item(b, nsub, ob, os);
  const char *p = static_cast<const char *>(f.ptr) + (ob * f.bstride + os * f.sstride) * eb;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + (unsigned)f.len * eb + 15) &
                       ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0))
               : "memory");
}

template <class PL>
struct FastC64Tr {
  static constexpr int warps = PL::CTA / 32;
  static constexpr int slabs = (warps + 3) / 4;
  static constexpr int need = slabs * 2 * PL::V;
  static constexpr int cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : 256;
  static constexpr int min_blocks = PL::CTA >= 512 ? 1 : (PL::CTA >= 384 ? 2 : HK_C64_MINB);
};

template <class PL, int NZ, int NO>
__global__ void __launch_bounds__(PL::CTA, (FastC64Tr<PL>::min_blocks))
    k_hankel_fast_c64(const __grid_constant__ Args1D a) {
  using Tr = FastC64Tr<PL>;
  constexpr int T = PL::T;
  constexpr int V = PL::V;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplxf *smem = reinterpret_cast<cplxf *>(smem_raw);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<Tr::cols>(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmy =
      tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 2 * V);
  const int g = threadIdx.x / T;
  const int t = threadIdx.x - g * T;
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  cplxf *sbuf = smem + g * PL::L;
  const cplxf *__restrict__ tw = a.twf;
  const fast::Tw0RecT<cplxf> tw0{a.twf};
  const fast::GroupSync<PL> gsync;
  auto prefetch = [&](long long bb) {
    for (int q = 0; q < PL::G; ++q) {
      const long long b = bb * PL::G + q;
      if (b >= a.batch) break;
      prefetch_f(a.h, b, a.nsub);
      for (int f = 0; f < a.nfac; ++f) prefetch_f(a.fac[f], b, a.nsub);
    }
  };
  if (a.prefetch && threadIdx.x == 0) prefetch(blockIdx.x);

  for (long long bb = blockIdx.x; bb < nblk; bb += gridDim.x) {
    if constexpr (std::is_same_v<fast::GroupSync<PL>, fast::WarpSync>) {
      if (bb != blockIdx.x) __syncthreads();
    }
    if (a.prefetch && threadIdx.x == 0 && bb + gridDim.x < nblk) prefetch(bb + gridDim.x);
    long long b = bb * PL::G + g;
    const bool active = b < a.batch;
    if (!active) b = a.batch - 1;
    long long ob, os;
    split_item(b, a.nsub, ob, os);
    cplxf v[V];
    {
      const Factor &hf = a.h;
      const long long off = ob * hf.bstride + os * hf.sstride;
      const float sc = (float)a.scale;
      fast::fft_dif<PL, true, PL::radix[0], PL::L, true>(
          sbuf, t, tw, tw0, [&](int pos) { return fast::load_elem_f(hf, off, pos, sc); }, v,
          gsync);
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) tmem_st4f(tmy + 8 * c, &v[4 * c]);
    }
    for (int f = 0; f < a.nfac; ++f) {
      const Factor &fa = a.fac[f];
      const long long off = ob * fa.bstride + os * fa.sstride;
      fast::fft_dif<PL, false, NZ, PL::L, true>(
          sbuf, t, tw, tw0, [&](int pos) { return fast::load_elem_f(fa, off, pos, 1.f); }, v,
          gsync);
      tmem_wait_st();
#pragma unroll
      for (int c = 0; c < V / 4; ++c) {
        cplxf q[4];
        tmem_ld4f(tmy + 8 * c, q);
        for (int k = 0; k < fa.power; ++k) {
#pragma unroll
          for (int i = 0; i < 4; ++i) q[i] = cmul(q[i], v[4 * c + i]);
        }
        tmem_st4f(tmy + 8 * c, q);
      }
    }
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) tmem_ld4f(tmy + 8 * c, &v[4 * c]);
    cplxf *out = static_cast<cplxf *>(a.out) + ob * a.out_bstride + os * a.out_sstride;
    if (a.mode == M_PARTIAL) {
      const int n1 = a.out_len;
      const long long es = a.out_estride;
      fast::fft_final<PL, NO, PL::L, true>(
          sbuf, t, tw, tw0, v,
          [&](int pos, cplxf y) {
            if (active && pos < n1) out[pos * es] = y;
          },
          gsync);
    } else {
      cplxf s = make_float2(0.f, 0.f);
#pragma unroll
      for (int r = 0; r < V; ++r) s = cadd(s, v[r]);
      gsync();
      cplxf *red = sbuf;
      red[t] = s;
      gsync();
      if (t == 0 && active) {
        cplxf tot = make_float2(0.f, 0.f);
        for (int k = 0; k < T; ++k) tot = cadd(tot, red[k]);
        out[0] = tot;
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<Tr::cols>(tmem_slot);
  }
}

template <class PL, int NZ, int NO>
static cudaError_t launch_fast_c64_variant(const Args1D &a, cudaStream_t stream) {
  const int smem = PL::G * PL::L * (int)sizeof(cplxf) + 128;
  static std::atomic<unsigned long long> configured{0};
  static int resident[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_fast_c64<PL, NZ, NO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // carve out shared memory for every resident CTA (TMEM holds the accumulators)
    e = cudaFuncSetAttribute(k_hankel_fast_c64<PL, NZ, NO>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    resident[dev & 63] = resident_ctas(reinterpret_cast<const void *>(
                                           k_hankel_fast_c64<PL, NZ, NO>),
                                       PL::CTA, smem, dev);
    configured.fetch_or(bit);
  }
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  if (nblk <= 0) return cudaSuccess;
  const long long grid = nblk < resident[dev & 63] ? nblk : resident[dev & 63];
  k_hankel_fast_c64<PL, NZ, NO><<<(unsigned)grid, PL::CTA, smem, stream>>>(a);
  return cudaGetLastError();
}

// pruning levels: nonzero first-pass inputs / needed last-pass outputs per
// butterfly, rounded up to the instantiated levels {R0/4, R0/2, R0}
template <class PL>
static cudaError_t launch_fast_c64(const Args1D &a, cudaStream_t stream, int maxlen, int outl) {
  constexpr int R0 = PL::radix[0], S0 = PL::stride(0);
  constexpr int q = R0 >= 4 ? R0 / 4 : 1, h = R0 >= 2 ? R0 / 2 : 1;
  const int nz = (maxlen + S0 - 1) / S0, no = (outl + S0 - 1) / S0;
  const int zi = nz <= q ? 0 : (nz <= h ? 1 : 2), oi = no <= q ? 0 : (no <= h ? 1 : 2);
  switch (zi * 3 + oi) {
    case 0: return launch_fast_c64_variant<PL, q, q>(a, stream);
    case 1: return launch_fast_c64_variant<PL, q, h>(a, stream);
    case 2: return launch_fast_c64_variant<PL, q, R0>(a, stream);
    case 3: return launch_fast_c64_variant<PL, h, q>(a, stream);
    case 4: return launch_fast_c64_variant<PL, h, h>(a, stream);
    case 5: return launch_fast_c64_variant<PL, h, R0>(a, stream);
    case 6: return launch_fast_c64_variant<PL, R0, q>(a, stream);
    case 7: return launch_fast_c64_variant<PL, R0, h>(a, stream);
    default: return launch_fast_c64_variant<PL, R0, R0>(a, stream);
  }
}

template <class PL>
static cudaError_t launch_c64_plan(const Args1D &a, cudaStream_t stream) {
  int smem = (PL::P > 1) ? PL::G * PL::L * (int)sizeof(cplxf) : 16;
  const int red_bytes = PL::G * PL::T * (int)sizeof(cplxf);
  if (smem < red_bytes) smem = red_bytes;
  static std::atomic<unsigned long long> configured{0};
  static int resident[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_c64<PL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    resident[dev & 63] =
        resident_ctas(reinterpret_cast<const void *>(k_hankel_c64<PL>), PL::CTA, smem, dev);
    configured.fetch_or(bit);
  }
  const long long nblk = (a.batch + PL::G - 1) / PL::G;
  if (nblk <= 0) return cudaSuccess;
  const long long grid = nblk < resident[dev & 63] ? nblk : resident[dev & 63];
  k_hankel_c64<PL><<<(unsigned)grid, PL::CTA, smem, stream>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Ping-pong variant for the batched H x^{m-1} workload in complex64 (cfg2-c64):
// the structure of the complex128 headline kernel (hk_pp1d.cu) on float2.  One
// 512-thread CTA per SM runs two 256-thread product groups; each group stages
// the operands of its product after next with per-thread 8-byte cp.async into
// its OWN h and x staging buffers (odd-length complex64 rows are only 8-byte
// aligned, so the 16-byte bulk copies of the complex128 kernel do not apply)
// right after the first pass has consumed them, so global latency is a full
// product period off the critical path.  The spectral accumulator and the
// per-thread twiddles of both twiddled passes live in TMEM; pass 1 runs
// lo-major so the pass-1/pass-2 exchanges stay inside each warp.
//   smem: ex[2][L] | hs[2][L] | xs[2][XS]   (float2; 147 KB at L = 4096)
//   TMEM: cols [0,128) accumulators (32 per warp slab) | [128,192) pass-0
//         twiddles | [192,256) pass-1 twiddles (slabs shared by the two groups)
namespace ppf {

template <int N>
struct GroupBar {
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(N) : "memory");
  }
};

struct Tw01F {
  uint32_t taddr0, taddr1;
  __device__ __forceinline__ void chunk(int, int c, cplxf *w) const { tmem_ld4f(taddr0 + 8 * c, w); }
  __device__ __forceinline__ void chunk1(int c, cplxf *w) const { tmem_ld4f(taddr1 + 8 * c, w); }
};

template <class PL, int NZ, int NO, int NG>
__global__ void __launch_bounds__(NG * PL::T, 1) k_hankel_pp_c64(const __grid_constant__ Args1D a) {
  constexpr int L = PL::L, T = PL::T, V = PL::V, R0 = PL::radix[0], R1 = PL::radix[1];
  constexpr int S0 = PL::stride(0), XS = NZ * S0, TW1 = L / R0;
  constexpr int TC = NG * 64 + 128 <= 256 ? 256 : 512;  // accumulators + two twiddle slabs
  static_assert(PL::G == 1 && T == 256 && PL::P == 3 && L / R0 == T && NZ < R0,
                "one product per 256-thread group, three passes, staged x prefix");
  static_assert(R1 == PL::Rlast && 32 % PL::Rlast == 0, "warp-local last exchange");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplxf *ex = reinterpret_cast<cplxf *>(smem_raw);
  cplxf *hs = ex + NG * L;
  cplxf *xs = hs + NG * L;
  const int warp = threadIdx.x >> 5;
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  // positions the copies never write: zero once (the padding of h~ and x~)
  for (int i = threadIdx.x; i < NG * L; i += blockDim.x)
    if (i % L >= a.h.len) hs[i] = make_float2(0.f, 0.f);
  for (int i = threadIdx.x; i < NG * XS; i += blockDim.x)
    if (i % XS >= a.fac[0].len) xs[i] = make_float2(0.f, 0.f);
  if (warp == 0) tmem_alloc<TC>(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;
  const uint32_t tacc = tmem_slot + lane_q + (uint32_t)((warp >> 2) * 32);
  const uint32_t ttw = tmem_slot + lane_q + (uint32_t)(NG * 64) + (uint32_t)(((warp >> 2) & 1) * 32);
  const uint32_t ttw1 = ttw + 64u;
  if (g == 0) {  // a thread's twiddles depend only on its index in its group
    const int lo1 = t % PL::stride(1);
#pragma unroll
    for (int c = 0; c < (R0 - 1 + 3) / 4; ++c) {
      cplxf w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * c + q + 1;
        w[q] = j < R0 ? a.twf[(j * t) % L] : make_float2(1.f, 0.f);  // W_L^{j t}
      }
      tmem_st4f(ttw + 8 * c, w);
    }
#pragma unroll
    for (int c = 0; c < (R1 - 1 + 3) / 4; ++c) {
      cplxf w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * c + q + 1;  // W_{L/R0}^{j lo} = W_L^{R0 j lo}
        w[q] = j < R1 ? a.twf[((j * lo1) % TW1) * R0] : make_float2(1.f, 0.f);
      }
      tmem_st4f(ttw1 + 8 * c, w);
    }
    tmem_wait_st();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const Tw01F tw0{ttw, ttw1};

  const long long nloc =
      a.batch > blockIdx.x ? (a.batch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  cplxf *sbuf = ex + g * L, *my_h = hs + g * L, *my_x = xs + g * XS;
  const uint32_t sh = smem_u32(my_h), sx = smem_u32(my_x);
  auto issue_h = [&](long long k) {
    const cplxf *src = static_cast<const cplxf *>(a.h.ptr) +
                       (blockIdx.x + k * (long long)gridDim.x) * a.h.bstride;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int pos = t + i * T;
      if (pos < a.h.len) fast::cpa8(sh + 8u * pos, src + pos, true);
    }
  };
  auto issue_x = [&](long long k) {
    const cplxf *src = static_cast<const cplxf *>(a.fac[0].ptr) +
                       (blockIdx.x + k * (long long)gridDim.x) * a.fac[0].bstride;
#pragma unroll
    for (int i = 0; i < NZ; ++i) {
      const int pos = t + i * T;
      if (pos < a.fac[0].len) fast::cpa8(sx + 8u * pos, src + pos, true);
    }
  };
  const GroupBar<T> sync{1 + g};
  if (g < nloc) {
    issue_h(g);
    issue_x(g);
  }
  const float sc = (float)a.scale;
  for (long long k = g; k < nloc; k += NG) {
    fast::cpa_wait_all();  // this thread's copies of product k; the entry barrier covers the group
    cplxf v[V];
    fast::fft_dif<PL, true, R0, L, false>(
        sbuf, t, a.twf, tw0, [&](int pos) { return my_h[pos]; }, v, sync,
        [&]() {
          if (k + NG < nloc) issue_h(k + NG);
        },
        (fast::WarpSync *)nullptr);
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) tmem_st4f(tacc + 8 * c, &v[4 * c]);
    fast::fft_dif<PL, false, NZ, L, false>(
        sbuf, t, a.twf, tw0, [&](int pos) { return my_x[pos]; }, v, sync,
        [&]() {
          if (k + NG < nloc) issue_x(k + NG);
        },
        (fast::WarpSync *)nullptr);
    tmem_wait_st();
#pragma unroll
    for (int c = 0; c < V / 4; ++c) {
      cplxf acc[4];
      tmem_ld4f(tacc + 8 * c, acc);
      for (int q = 0; q < a.fac[0].power; ++q) {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = cmul(acc[e], v[4 * c + e]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) v[4 * c + e] = acc[e];
    }
    cplxf *yk = static_cast<cplxf *>(a.out) +
                (blockIdx.x + k * (long long)gridDim.x) * a.out_bstride;
    fast::fft_final<PL, NO, L, false>(
        sbuf, t, a.twf, tw0, v,
        [&](int pos, cplxf val) {
          if (pos < a.out_len) yk[pos] = make_float2(val.x * sc, val.y * sc);
        },
        sync, (fast::WarpSync *)nullptr);
  }
  fast::cpa_wait_all();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<TC>(tmem_slot);
  }
}

template <class PL, int NZ, int NO, int NG>
static cudaError_t launch(const Args1D &a, cudaStream_t stream) {
  const int smem = NG * (2 * PL::L + NZ * PL::stride(0)) * (int)sizeof(cplxf) + 128;
  static std::atomic<unsigned long long> configured{0};
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_hankel_pp_c64<PL, NZ, NO, NG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    configured.fetch_or(bit);
  }
  long long grid = sms[dev & 63];
  if (grid > a.batch) grid = a.batch;
  if (grid <= 0) return cudaSuccess;
  k_hankel_pp_c64<PL, NZ, NO, NG><<<(unsigned)grid, NG * PL::T, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace ppf

// cudaErrorNotSupported unless the request is the plain batched complex64
// H x^{m-1} shape of the ping-pong kernel (HK_NO_PP_C64=1 turns it off for A/B).
static cudaError_t launch_pp_c64(int L, const Args1D &a, cudaStream_t stream) {
  if (getenv("HK_NO_PP_C64")) return cudaErrorNotSupported;
  if (L != 4096 || a.mode != M_PARTIAL || a.nfac != 1 || a.nsub != 1 || a.ncombo)
    return cudaErrorNotSupported;
  const Factor &h = a.h, &x = a.fac[0];
  if (h.kind != FK_C64 || x.kind != FK_C64 || h.estride != 1 || x.estride != 1 ||
      a.out_estride != 1 || h.len <= 0 || h.len > L || x.len <= 0)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(h.ptr) | reinterpret_cast<uintptr_t>(x.ptr)) & 7)
    return cudaErrorNotSupported;
  using PL = Plan1D<4096, 256, 16, 16, 16>;
  constexpr int s0 = PL::stride(0);
  const int nz = (x.len + s0 - 1) / s0, no = (a.out_len + s0 - 1) / s0;
  // three product groups per SM (768 threads, 85 registers) against two (128
  // registers): HK_PP_C64_NG selects for A/B
  const int ng = getenv("HK_PP_C64_NG") ? atoi(getenv("HK_PP_C64_NG")) : 2;
  if (nz <= 4 && no <= 4)
    return ng == 3 ? ppf::launch<PL, 4, 4, 3>(a, stream) : ppf::launch<PL, 4, 4, 2>(a, stream);
  return cudaErrorNotSupported;
}

cudaError_t launch_c64_1d(int L, const Args1D &a, cudaStream_t stream) {
  if (!a.twf) return cudaErrorInvalidValue;
  if (a.mode != M_PARTIAL && a.mode != M_FULL) return cudaErrorNotSupported;
  static const bool generic_only = getenv("HK_C64_GENERIC") != nullptr;  // A/B switch
  if (!generic_only) {
    const cudaError_t e = launch_pp_c64(L, a, stream);
    if (e != cudaErrorNotSupported) return e;
    int maxlen = 1;
    for (int f = 0; f < a.nfac; ++f)
      if (a.fac[f].len > maxlen) maxlen = a.fac[f].len;
    const int outl = a.mode == M_PARTIAL ? a.out_len : L;
    switch (L) {
      case 4096: return launch_fast_c64<Plan1D<4096, 256, 16, 16, 16>>(a, stream, maxlen, outl);
      case 8192: return launch_fast_c64<Plan1D<8192, 512, 2, 16, 16, 16>>(a, stream, maxlen, outl);
      case 2048: return launch_fast_c64<Plan1D<2048, 128, 8, 16, 16>>(a, stream, maxlen, outl);
      case 1024: return launch_fast_c64<Plan1D<1024, 64, 4, 16, 16>>(a, stream, maxlen, outl);
      case 256: return launch_fast_c64<Plan1D<256, 16, 16, 16>>(a, stream, maxlen, outl);
      default: break;
    }
  }
  switch (L) {
#define HK_CASE(len, ...) \
  case len:              \
    return launch_c64_plan<__VA_ARGS__>(a, stream);
    HK_PLAN_LIST(HK_CASE)
#undef HK_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hk
