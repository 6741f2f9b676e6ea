// K3 / K4: two-level fused products for transforms that do not fit on chip.
//
// The length-L transform is viewed as an L1 x L2 array, element (n1, n2),
// n2 contiguous.  Two modes share every kernel:
//   * 1D (four-step, L = L1*L2 >= d_H, reference hankel.py:140-154):
//       n = n2 + L2*n1, twiddle W_L^{n2*k1} between the column and row stages;
//   * 2D (BHHB / level-2, reference block.py:136-153, fft2 over L_in x L_out):
//       n1 = outer index, n2 = inner index, no twiddle.
// Pipeline per batch chunk (workspace = rows of length L2, natural order):
//   A  (k_cols)  column DFTs over n1 of h (inverse) and of each distinct x
//                (forward), + twiddle                       -> Wh, Wx_f
//   B  (fast 1D kernel, one "product" per row k1)           -> Wq
//                ifft_row(Wh) .* fft_row(Wx)^p, then the transposed row DFT
//   C  (k_cols)  + twiddle, column DFT over k1 (the transposed forward
//                transform of the final fft), truncation    -> y
// Zero padding and truncation are validity predicates on the loads/stores;
// columns that carry no data (x's zero block, unused outputs) are skipped.
#include <atomic>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "hk_fastcore.cuh"
#include "hk_large.h"

namespace hk {
namespace large {

// Column passes >= 1 take their twiddles by recurrence from one table read
// per butterfly (fast::twiddle_rec) instead of R-1 strided table reads.
constexpr bool kColRec = true;
// Pass-0 twiddles W_L1^{j beta} by the same recurrence from W_L1^beta.
constexpr bool kColTw0Rec = true;

__device__ __forceinline__ cplx tw4step(const ColArgs &a, long long e) {
  e %= a.L;
  const cplx hi = __ldg(&a.thi[e >> 12]);
  const cplx lo = __ldg(&a.tlo[e & 4095]);
  return cmul(hi, lo);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Persistent column-tile kernel.  Tile w = (item, column block); the CTA keeps
// two smem tile buffers and streams tile w+grid in with cp.async (zero-fill
// for padding) while it transforms tile w, so global latency overlaps math.
// Resident CTAs per SM the double-buffered tiles allow (227 KB of shared
// memory); the register budget is sized so registers never cut below that.
template <class PL, int TILE>
constexpr int col_blocks() {
  constexpr int pad = TILE >= 8 ? 1 : 8 / TILE;
  constexpr int bytes = 2 * TILE * (PL::L + pad) * 16 + 1024;
  constexpr int by_smem = (227 * 1024) / bytes;
  constexpr int by_thr = 2048 / (TILE * PL::T);
  constexpr int n = by_smem < by_thr ? by_smem : by_thr;
  return n < 1 ? 1 : (n > 4 ? 4 : n);
}

template <class PL, int TILE, int STAGE>
__global__ void __launch_bounds__(TILE * PL::T, (col_blocks<PL, TILE>())) k_cols(const __grid_constant__ ColArgs a,
                                                          int tiles_per_item, long long ntiles) {
  constexpr int L1 = PL::L, T = PL::T, V = PL::V, RL = PL::Rlast, R0 = PL::radix[0];
  constexpr int PAD = TILE >= 8 ? 1 : 8 / TILE;
  constexpr int CS = L1 + PAD;  // column stride in smem (elements)
  constexpr int NT = TILE * T;
  constexpr bool INV = STAGE == ST_A_INV;
  constexpr bool PAIR = STAGE == ST_A_PAIR;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cplx *bufs = reinterpret_cast<cplx *>(smem_raw);
  const int c = threadIdx.x / T, t = threadIdx.x - (threadIdx.x / T) * T;
  const bool real_in = a.in.kind == FK_F64;

  // Rows of column n2 that exist in an operand / output: 1D layout (len >= 0)
  // element (n1, n2) is n2 + L2 n1 < len, i.e. n1 < len / L2 + (n2 < len % L2);
  // 2D layout: n1 < e1 for n2 < e2.  The 64-bit divisions run once per thread.
  struct Lim {
    int q, rem, e2;  // rows = n2 < e2 ? q + (n2 < rem) : 0
    __device__ __forceinline__ int rows(int n2) const { return n2 < e2 ? q + (n2 < rem ? 1 : 0) : 0; }
  };
  auto make_lim = [&](long long len, int e1, int e2) {
    if (len >= 0) {
      const long long q = len / a.L2;
      return Lim{(int)(q < L1 ? q : L1), q < L1 ? (int)(len - q * a.L2) : 0, a.L2};
    }
    return Lim{e1 < L1 ? e1 : L1, 0, e2};
  };
  const Lim lim_in = make_lim(a.in.len, a.in.e1, a.in.e2);
  const Lim lim_in2 = PAIR ? make_lim(a.in2.len, a.in2.e1, a.in2.e2) : Lim{0, 0, 0};
  const Lim lim_out = make_lim(a.out.len, a.out.e1, a.out.e2);
  const Lim lim_out2 = PAIR ? make_lim(a.out2.len, a.out2.e1, a.out2.e2) : Lim{0, 0, 0};

  // Pruned first / last passes (the 2D block product's vector and output
  // passes, cfg4: 64 of 192 rows).  First pass: rows >= NZP * stride(0) of the
  // operand are zero, so each pass-0 butterfly has NZP nonzero inputs and the
  // zero rows are neither copied nor read.  Last pass: only rows < NOP * L1/RL
  // of the output are kept (register j of a last-pass butterfly holds row
  // k0 + j L1/RL), so NOP of the RL outputs are computed and stored.
  constexpr int NZP0 = PL::P > 1 ? (R0 % 3 == 0 ? R0 / 3 : R0 / 4) : R0;
  constexpr int NZP = NZP0 < 1 ? R0 : NZP0;  // radix 2 first passes are not pruned
  constexpr int NOP = (PL::P > 1 && RL == 16) ? 6 : RL;
  constexpr int S0K = PL::stride(0);
  const int in_rows = lim_in.q + (lim_in.rem > 0 ? 1 : 0);    // max rows of any column
  const int out_rows = lim_out.q + (lim_out.rem > 0 ? 1 : 0);
  const bool prune_in = !PAIR && STAGE != ST_C && NZP < R0 && in_rows <= NZP * S0K;
  const bool prune_out = STAGE == ST_C && NOP < RL && out_rows <= NOP * (L1 / RL);
  const int need_rows = prune_in ? NZP * S0K : L1;  // tile rows the first pass reads

  // Tile load.  r02 ncu (cfg4 h pass): the per-element index arithmetic of the
  // generic loop (runtime divisions, 64-bit bounds and three 64-bit multiplies
  // per element, ~40 integer instructions) was 35% of the kernel.  Here the
  // loop is unrolled with compile-time element indices, the bounds are one
  // integer compare, and the address is base + n1 s1 + n2 s2.
  // Element i of a thread is idx = tid + i NT of the TILE x L1 tile (NI = V of
  // them).  Operand contiguous along n1 (in_n1_fast): idx = cc L1 + n1d; else
  // idx = n1d TILE + cc.  NT divides L1 or L1 divides NT (NT = TILE L1 / V, TILE
  // and V powers of two... or equal), so the split of idx is a per-thread
  // constant plus a compile-time function of i; item-relative offsets are
  // 32-bit (launch_cols_t checks the extent).
  constexpr int NI = (TILE * L1) / NT;
  static_assert(NI * NT == TILE * L1 && NT % TILE == 0, "whole tile per pass of the CTA");
  constexpr bool kSplit = L1 % NT == 0 || NT % L1 == 0;
  const int f_cc0 = kSplit ? (L1 % NT == 0 ? 0 : (int)threadIdx.x / L1) : 0;
  const int f_n0 = kSplit ? (L1 % NT == 0 ? (int)threadIdx.x : (int)threadIdx.x % L1) : 0;
  const int s_cc = threadIdx.x % TILE, s_n0 = threadIdx.x / TILE;
  const uint32_t is1 = (uint32_t)a.in.s1, is2 = (uint32_t)a.in.s2;
  const uint32_t is1b = PAIR ? (uint32_t)a.in2.s1 : 0u, is2b = PAIR ? (uint32_t)a.in2.s2 : 0u;
  auto issue = [&](long long w, cplx *tile) {
    // tile indices fit 32 bits (launch_cols_t): no emulated 64-bit division
    const long long item = (unsigned)w / (unsigned)tiles_per_item;
    const int c0 = (int)((unsigned)w - (unsigned)item * (unsigned)tiles_per_item) * TILE;
    const bool half_c = STAGE == ST_C && a.half;
    const int esz = real_in || PAIR ? 8 : 16;
    const char *b1 = static_cast<const char *>(a.in.ptr) + item * a.in.item_stride * esz;
    const char *b2 = PAIR ? static_cast<const char *>(a.in2.ptr) + item * a.in2.item_stride * 8
                          : nullptr;
    auto one = [&](int cc, int n1d, int rows, int rows2) {
      if (n1d >= need_rows) return;  // pruned first pass: zero rows are never read
      // Hermitian half (ST_C): rows above L1/2 are read from row L1 - n1
      const int n1 = (half_c && 2 * n1d > L1) ? L1 - n1d : n1d;
      const uint32_t n2 = (uint32_t)(c0 + cc);
      const bool ok = n1 < rows;
      const uint32_t off = ok ? (uint32_t)n1 * is1 + n2 * is2 : 0u;
      const uint32_t dst = smem_u32(tile + cc * CS + fast::swz2(n1d));
      if constexpr (PAIR) {  // z = h + i x from two real streams (1D layout)
        const bool ok2 = n1 < rows2;
        const uint32_t off2 = ok2 ? (uint32_t)n1 * is1b + n2 * is2b : 0u;
        cp_async8(dst, b1 + (size_t)off * 8, ok);
        cp_async8(dst + 8, b2 + (size_t)off2 * 8, ok2);
      } else if (real_in) {
        cp_async8(dst, b1 + (size_t)off * 8, ok);
      } else {
        cp_async16(dst, b1 + (size_t)off * 16, ok);
      }
    };
    if (a.in_n1_fast) {
      if constexpr (L1 % NT == 0) {  // a column spans K = L1 / NT passes
        constexpr int K = L1 / NT;
#pragma unroll
        for (int cc = 0; cc < TILE; ++cc) {
          const int rows = lim_in.rows(c0 + cc), rows2 = PAIR ? lim_in2.rows(c0 + cc) : 0;
#pragma unroll
          for (int k = 0; k < K; ++k) one(cc, f_n0 + k * NT, rows, rows2);
        }
      } else if constexpr (NT % L1 == 0) {  // M = NT / L1 columns per pass
        constexpr int M = NT / L1;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int cc = i * M + f_cc0;
          one(cc, f_n0, lim_in.rows(c0 + cc), PAIR ? lim_in2.rows(c0 + cc) : 0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int idx = (int)threadIdx.x + i * NT, cc = idx / L1;
          one(cc, idx - cc * L1, lim_in.rows(c0 + cc), PAIR ? lim_in2.rows(c0 + cc) : 0);
        }
      }
    } else {
      const int rows = lim_in.rows(c0 + s_cc), rows2 = PAIR ? lim_in2.rows(c0 + s_cc) : 0;
#pragma unroll
      for (int i = 0; i < NI; ++i) one(s_cc, s_n0 + i * (NT / TILE), rows, rows2);
    }
    cp_async_commit();
  };

  long long w = blockIdx.x;
  if (w < ntiles) issue(w, bufs);
  using TW0 = std::conditional_t<kColTw0Rec, fast::Tw0Rec, fast::Tw0Global>;
  TW0 tw0;
  if constexpr (kColTw0Rec)
    tw0 = fast::Tw0Rec{a.ctw};
  else
    tw0 = fast::Tw0Global{a.ctw0, L1 / R0, R0};
  for (int it = 0; w < ntiles; ++it, w += gridDim.x) {
    cplx *tile = bufs + (it & 1) * (TILE * CS);
    const long long wn = w + gridDim.x;
    if (wn < ntiles) {
      issue(wn, bufs + ((it + 1) & 1) * (TILE * CS));
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const long long item = (unsigned)w / (unsigned)tiles_per_item;
    const int c0 = (int)((unsigned)w - (unsigned)item * (unsigned)tiles_per_item) * TILE;
    const int n2 = c0 + c;
    cplx *col = tile + c * CS;
    // pass-0 input: scale, real promotion, stage-C twiddle.  The elements of a
    // pass-0 butterfly sit at pos = beta + j*s0, so their four-step twiddles
    // W_L^{n2 pos} form a geometric sequence: two table lookups per butterfly
    // and a multiply recurrence (error ~R0 ulp) instead of two lookups each.
    constexpr int S0 = PL::stride(0);
    cplx tw_cur = make_double2(1.0, 0.0), tw_step = make_double2(1.0, 0.0);
    if (STAGE == ST_C && a.twiddle) tw_step = tw4step(a, (long long)n2 * S0);
    const cplx wrow = (STAGE == ST_C && a.half) ? tw4step(a, (long long)n2 * L1)
                                                  : make_double2(1.0, 0.0);  // W_L2^{m2}
    auto in_load = [&](int, int j, int pos) {
      cplx v = col[fast::swz2(pos)];
      if constexpr (PAIR) return v;  // scale of h applied when z is split
      if (STAGE == ST_C && a.half && 2 * pos > L1) {
        v = cmul(v, wrow);  // Q(L1-k1, m2) = conj(W_L2^{m2} Q(k1, m2))
        v.y = -v.y;
      }
      if (real_in) v.y = 0.0;
      v.x *= a.in.scale;
      v.y *= a.in.scale;
      if (STAGE == ST_C && a.twiddle) {
        if (j == 0) tw_cur = tw4step(a, (long long)n2 * pos);
        v = cmul(v, tw_cur);
        tw_cur = cmul(tw_cur, tw_step);
      }
      return v;
    };
    auto s_load = [&](int, int, int pos) { return col[fast::swz2(pos)]; };
    auto s_store = [&](int, int, int pos, cplx v) { col[fast::swz2(pos)] = v; };
    cplx v[V];
    auto r_store = [&](int i, int j, int, cplx x) { v[i * RL + j] = x; };
    if constexpr (PL::P > 1) {
      if (NZP < R0 && prune_in)
        fast::pass<PL, 0, INV, false, NZP, R0>(t, a.ctw, tw0, in_load, s_store);
      else
        fast::pass<PL, 0, INV, false, R0, R0>(t, a.ctw, tw0, in_load, s_store);
      sfor<PL::P - 2>([&](auto qc) {
        constexpr int q = decltype(qc)::value + 1;
        __syncthreads();
        fast::pass<PL, q, INV, false, PL::radix[q], PL::radix[q], L1, kColRec>(t, a.ctw, tw0, s_load,
                                                                 s_store);
      });
      __syncthreads();
      if (prune_out)
        fast::pass<PL, PL::P - 1, INV, false, RL, NOP, L1, kColRec>(t, a.ctw, tw0, s_load, r_store);
      else
        fast::pass<PL, PL::P - 1, INV, false, RL, RL, L1, kColRec>(t, a.ctw, tw0, s_load, r_store);
    } else {
      fast::pass<PL, 0, INV, false, R0, R0>(t, a.ctw, tw0, in_load, r_store);
    }
    __syncthreads();
    // digit-reversed registers -> natural order (+ stage-A twiddle)
    // last-pass register j of butterfly beta holds frequency k = k(beta) + j*L1/RL
    // (j is the most significant mixed-radix digit): geometric twiddles again
    constexpr bool TW_A = STAGE != ST_C && !PAIR;  // stage-A twiddle in this loop
    const cplx tws = (TW_A && a.twiddle) ? tw4step(a, (long long)n2 * (L1 / RL))
                                         : make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < V / RL; ++i) {
      const int beta = t + i * T;
      int k0 = 0, mul = 1;
      sfor<PL::P>([&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int Rp = PL::radix[p], Sp = PL::stride(p);
        k0 += (((beta * RL) / Sp) % Rp) * mul;
        mul *= Rp;
      });
      cplx cur = (TW_A && a.twiddle) ? tw4step(a, (long long)n2 * k0)
                                     : make_double2(1.0, 0.0);
#pragma unroll
      for (int j = 0; j < RL; ++j) {
        if (prune_out && j >= NOP) break;
        const int k = k0 + j * (L1 / RL);
        cplx x = v[i * RL + j];
        if (TW_A && a.twiddle) {
          x = INV ? cmulc(x, cur) : cmul(x, cur);
          cur = cmul(cur, tws);
        }
        col[k] = x;
      }
    }
    __syncthreads();
    // coalesced tile store
    auto store_tile = [&](const Out2 &o, const Lim &lim) {
      // thread -> fixed column cc = tid % TILE, rows tid / TILE + i (NT / TILE),
      // i < NI; the shared-memory reads of half a tile are issued before its stores
      const int m2 = c0 + s_cc;
      const int rows = lim.rows(m2);
      cplx *d = static_cast<cplx *>(o.ptr) + item * o.item_stride + s_n0 * o.s1 + m2 * o.s2;
      const long long step = (long long)(NT / TILE) * o.s1;
      const cplx *src = tile + s_cc * CS + s_n0;
      constexpr int NB = NI >= 8 ? 8 : NI;
#pragma unroll
      for (int i0 = 0; i0 < NI; i0 += NB) {
        if (s_n0 + i0 * (NT / TILE) >= rows) break;
        cplx u[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i)
          if (i0 + i < NI && s_n0 + (i0 + i) * (NT / TILE) < rows) u[i] = src[(i0 + i) * (NT / TILE)];
#pragma unroll
        for (int i = 0; i < NB; ++i)
          if (i0 + i < NI && s_n0 + (i0 + i) * (NT / TILE) < rows) d[(i0 + i) * step] = u[i];
      }
    };
    if constexpr (PAIR) {
      // col[k] = Z(k) = H(k) + i X(k) with H, X the column DFTs of the real
      // h, x:  H(k) = (Z(k) + conj Z(-k)) / 2,  X(k) = (Z(k) - conj Z(-k)) / 2i,
      // H(-k) = conj H(k), X(-k) = conj X(k).  Stage A of h is the INVERSE
      // column DFT (= conj H for real h) times 1/L; both get the four-step
      // twiddle W_L^{+-n2 k}.  Thread t handles the pairs (k, L1 - k),
      // k = t, t + T, ... <= L1/2; x's values wait in registers while h's
      // tile is stored.
      // The pairs are disjoint and each is read and rewritten by one thread,
      // so h's values go back in place at once.
      constexpr int NP = (L1 / 2 + 1 + T - 1) / T;
      cplx xa[NP], xb[NP];
      const double sh = a.in.scale;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int k = t + p * T;
        if (k > L1 / 2) continue;
        const int kk = k == 0 ? 0 : L1 - k;
        const cplx A = col[k], B = col[kk];
        const cplx H = make_double2(0.5 * (A.x + B.x), 0.5 * (A.y - B.y));
        const cplx X = make_double2(0.5 * (A.y + B.y), 0.5 * (B.x - A.x));
        const cplx wk = tw4step(a, (long long)n2 * k), wkk = tw4step(a, (long long)n2 * kk);
        // inverse h: conj(H(k)) * conj(W^{n2 k}) = conj(H(k) W^{n2 k})
        const cplx hk = cmul(H, wk), hkk = cmulc(H, wkk);  // H(-k) = conj H(k)
        xa[p] = cmul(X, wk);
        xb[p] = cmul(make_double2(X.x, -X.y), wkk);
        col[k] = make_double2(hk.x * sh, -hk.y * sh);
        if (kk != k) col[kk] = make_double2(hkk.x * sh, hkk.y * sh);
      }
      __syncthreads();
      store_tile(a.out, lim_out);
      __syncthreads();
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int k = t + p * T;
        if (k > L1 / 2) continue;
        col[k] = xa[p];
        if (k != 0 && 2 * k != L1) col[L1 - k] = xb[p];  // kk == k for k = 0, L1/2
      }
      __syncthreads();
      store_tile(a.out2, lim_out2);
    } else {
      store_tile(a.out, lim_out);
    }
    __syncthreads();  // this buffer is refilled two iterations later
  }
}

// Per-item sums of per-row partial sums (tvp_full): fixed order, deterministic.
__global__ void k_rowsum(const cplx *__restrict__ part, long long rows, cplx *out, long long n) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= n) return;
  cplx s = make_double2(0.0, 0.0);
  for (long long r = 0; r < rows; ++r) s = cadd(s, part[b * rows + r]);
  out[b] = s;
}

template <class PL, int TILE, int STAGE>
static cudaError_t launch_cols_t(const ColArgs &a, long long items, int ncols,
                                 cudaStream_t stream) {
  constexpr int PAD = TILE >= 8 ? 1 : 8 / TILE;
  const int smem = 2 * TILE * (PL::L + PAD) * (int)sizeof(cplx);
  static std::atomic<unsigned long long> configured{0};
  static int resident[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_cols<PL, TILE, STAGE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // carve out enough shared memory for every resident CTA (see resident below)
    e = cudaFuncSetAttribute(k_cols<PL, TILE, STAGE>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_cols<PL, TILE, STAGE>);
    int sms = 0, smem_sm = 0, regs_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int nt = TILE * PL::T;
    int per = regs_sm / (((fa.numRegs + 7) / 8 * 8) * nt);
    per = std::min(per, smem_sm / (smem + (int)fa.sharedSizeBytes + 1024));
    per = std::min(per, 2048 / nt);
    resident[dev & 63] = sms * std::max(1, per);
    configured.fetch_or(bit);
  }
  // the tile loads address operands with 32-bit item-relative element offsets
  auto small = [&](const Op2 &op) {
    return op.s1 >= 0 && op.s2 >= 0 &&
           (long long)(PL::L - 1) * op.s1 + (long long)(a.L2 + TILE) * op.s2 < (1ll << 31);
  };
  if (!small(a.in) || (STAGE == ST_A_PAIR && !small(a.in2))) return cudaErrorNotSupported;
  const int tiles = (ncols + TILE - 1) / TILE;
  const long long ntiles = (long long)tiles * items;
  if (ntiles <= 0) return cudaSuccess;
  if (ntiles >= (1ll << 31)) return cudaErrorNotSupported;
  const long long grid = std::min<long long>(ntiles, resident[dev & 63]);
  k_cols<PL, TILE, STAGE><<<(unsigned)grid, TILE * PL::T, smem, stream>>>(a, tiles, ntiles);
  return cudaGetLastError();
}

template <int STAGE>
static cudaError_t launch_cols_stage(const ColArgs &a, long long items, int ncols,
                                     cudaStream_t stream) {
  switch (a.L1) {
#define HK_COL(len, TILE, ...) \
  case len:                    \
    return launch_cols_t<__VA_ARGS__, TILE, STAGE>(a, items, ncols, stream);
    // TILE chosen so the double-buffered tile is <= ~130 KB (TILE*L1 ~ 3072 or less)
    HK_COL(8, 64, Plan1D<8, 1, 8>)
    HK_COL(12, 64, Plan1D<12, 1, 12>)
    HK_COL(16, 64, Plan1D<16, 1, 16>)
    HK_COL(24, 64, Plan1D<24, 1, 24>)
    HK_COL(32, 64, Plan1D<32, 2, 2, 16>)
    HK_COL(48, 64, Plan1D<48, 3, 3, 16>)
    HK_COL(64, 32, Plan1D<64, 4, 4, 16>)
    HK_COL(96, 32, Plan1D<96, 6, 6, 16>)
    HK_COL(128, 16, Plan1D<128, 8, 8, 16>)
    HK_COL(192, 8, Plan1D<192, 12, 12, 16>)  // B200 cfg4: TILE 8 973 us, 16 984, 32 1058
    HK_COL(256, 8, Plan1D<256, 16, 16, 16>)
    HK_COL(384, 8, Plan1D<384, 24, 24, 16>)
    HK_COL(512, 4, Plan1D<512, 32, 2, 16, 16>)
    HK_COL(768, 4, Plan1D<768, 48, 3, 16, 16>)
    HK_COL(1024, 2, Plan1D<1024, 64, 4, 16, 16>)
    case 1536:  // HK_COL1536_TILE: A/B of the column-tile width for cfg3
      if (getenv("HK_COL1536_TILE") && atoi(getenv("HK_COL1536_TILE")) == 2)
        return launch_cols_t<Plan1D<1536, 96, 6, 16, 16>, 2, STAGE>(a, items, ncols, stream);
      if (getenv("HK_COL1536_TILE") && atoi(getenv("HK_COL1536_TILE")) == 1)
        return launch_cols_t<Plan1D<1536, 96, 6, 16, 16>, 1, STAGE>(a, items, ncols, stream);
      return launch_cols_t<Plan1D<1536, 96, 6, 16, 16>, 4, STAGE>(a, items, ncols, stream);
    HK_COL(2048, 2, Plan1D<2048, 128, 8, 16, 16>)
    // d_H beyond 2048 x 8192 = 2^24: one-column tiles of 3072 / 4096 rows
    HK_COL(3072, 1, Plan1D<3072, 192, 12, 16, 16>)
    HK_COL(4096, 1, Plan1D<4096, 256, 16, 16, 16>)
#undef HK_COL
    default:
      return cudaErrorNotSupported;
  }
}

}  // namespace large

bool supported_col_len(long long L1) {
  switch (L1) {
    case 8: case 12: case 16: case 24: case 32: case 48: case 64: case 96: case 128:
    case 192: case 256: case 384: case 512: case 768: case 1024: case 1536: case 2048:
    case 3072: case 4096:
      return true;
    default:
      return false;
  }
}

cudaError_t launch_cols(int stage, const large::ColArgs &a, long long items, int ncols,
                        cudaStream_t stream) {
  if (stage == large::ST_A_PAIR || stage == large::ST_C) {
    const cudaError_t e = launch_cols_tma(stage, a, items, ncols, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (stage) {
    case large::ST_A_PAIR: return large::launch_cols_stage<large::ST_A_PAIR>(a, items, ncols, stream);
    case large::ST_A_FWD: return large::launch_cols_stage<large::ST_A_FWD>(a, items, ncols, stream);
    case large::ST_A_INV: return large::launch_cols_stage<large::ST_A_INV>(a, items, ncols, stream);
    default: return large::launch_cols_stage<large::ST_C>(a, items, ncols, stream);
  }
}

cudaError_t launch_rowsum(const double2 *part, long long rows, double2 *out, long long n,
                          cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  large::k_rowsum<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(part, rows, out, n);
  return cudaGetLastError();
}

}  // namespace hk
