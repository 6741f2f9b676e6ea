// K4f: the 2-level block (BHHB) product as ONE on-chip 2D spectral product per
// item (reference block.py:136-144, cfg4: order 3, 64 x 64 blocks, 190 x 190
// generator, transform 192 x 192):
//
//   y = fft2( ifft2(H~) .* fft2(X~)^p )[:n, :N]
//
// A 192 x 192 complex spectrum (576 KB) does not fit one SM, so the OUTER
// frequency k_c (the contiguous dimension of H) is split into its four residue
// classes k_c = 4 m + r.  For each r the CTA holds one quarter of the spectral
// product in shared memory and adds its contribution to y:
//
//   1. S1_r[a][m] = sum_c H[a][c] W^{-c(4m+r)}: fold each row of H onto 48
//      points (sum_q H[a][n'+48q] i^{qr}, twiddle W^{-n'r}) and a 48-point
//      inverse DFT (190 rows, 3 threads each)
//   2. X1_r[i][m] = sum_j X[i][j] W^{j(4m+r)}: the same for the n x N vector
//   3. per column m: the 1D spectral product along the inner dimension,
//      Y_r[i][m] = fft_a( ifft_a(S1_r[:,m]) .* fft_a(X1_r[:,m])^p )[i < n]
//      (48 products of length 192, 12 threads each, TMEM accumulator)
//   4. y[i][j] += W^{j r} * DFT_48(Y_r[i][:])[j mod 48]  (TMEM accumulator)
//
// Every intermediate stays on chip: HBM sees H, x and y once (H is re-read
// from L2 by the residue passes).  Shared memory: S1 (48 x 192 slots, the
// exchange buffer of step 3 in place) + X1/Y (48 x 64 slots) = 192 KB.
#include <atomic>

#include "hk_fastcore.cuh"
#include "hk_large.h"

namespace hk {
namespace bhhb {

constexpr int L = 192, D = 48, NR = 4;  // transform length, folded length, residues
constexpr int XN = 64;                  // X1/Y rows (n <= 64)
constexpr int NT = 288;                 // 24 column products x 12 threads, two rounds
constexpr int NG = NT / 12;             // concurrent column products
constexpr int NROW = NT / 3;            // concurrent 48-point row DFTs
using P192 = Plan1D<192, 12, 12, 16>;
using P48 = Plan1D<48, 3, 3, 16>;
static_assert(D % NG == 0 && 3 * XN <= NT, "rounds of the column products / row DFTs");

__device__ __forceinline__ int sa_slot(int m, int a) { return m * L + (fast::swz2(a) ^ (m & 7)); }
__device__ __forceinline__ int xb_slot(int m, int i) { return m * XN + (i ^ (m & 7)); }

// natural frequency of register j of the last-pass butterfly beta (two-pass plans)
template <class PL>
__device__ __forceinline__ int k_of(int beta, int j) {
  constexpr int RL = PL::Rlast;
  int k0 = 0, mul = 1;
  sfor<PL::P>([&](auto pc) {
    constexpr int p = decltype(pc)::value;
    constexpr int Rp = PL::radix[p], Sp = PL::stride(p);
    k0 += (((beta * RL) / Sp) % Rp) * mul;
    mul *= Rp;
  });
  return k0 + j * (PL::L / RL);
}

// i^e (inverse) or (-i)^e (forward) times a
template <bool INV>
__device__ __forceinline__ cplx rot4(cplx a, int e) {
  e &= 3;
  if (!INV && (e & 1)) e ^= 2;
  switch (e) {
    case 0: return a;
    case 1: return make_double2(-a.y, a.x);
    case 2: return make_double2(-a.x, -a.y);
    default: return make_double2(a.y, -a.x);
  }
}

// In-place 48-point DFT of one row held in shared memory at slot(pos), three
// threads per row; the result is written back in natural order.  Two CTA
// barriers (uniform over the CTA: every thread calls this).
template <bool INV, class Slot>
__device__ __forceinline__ void dft48(cplx *buf, bool active, int t, const cplx *tw48, Slot slot) {
  const fast::Tw0Rec tw0{tw48};
  auto ld = [&](int, int, int pos) { return buf[slot(pos)]; };
  auto st = [&](int, int, int pos, cplx v) { buf[slot(pos)] = v; };
  if (active) fast::pass<P48, 0, INV, false, 3, 3>(t, tw48, tw0, ld, st);  // DIF in place
  __syncthreads();
  cplx v[P48::V];
  auto rs = [&](int i, int j, int, cplx x) { v[i * 16 + j] = x; };
  if (active) fast::pass<P48, 1, INV, false, 16, 16>(t, tw48, tw0, ld, rs);
  __syncthreads();
  if (active) {
#pragma unroll
    for (int j = 0; j < 16; ++j) buf[slot(k_of<P48>(t, j))] = v[j];
  }
}

__global__ void __launch_bounds__(NT) k_bhhb_fused(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  cplx *SA = reinterpret_cast<cplx *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  cplx *XB = SA + D * L;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t lane_q = (uint32_t)(32 * (warp & 3)) << 16;
  // step 3 accumulator: 16 complex per thread (9 warps: cols 0..191); step 4
  // y accumulator: 24 complex per thread (warps 0-5: cols 256..447)
  const uint32_t tacc = tmem_slot + lane_q + (uint32_t)((warp >> 2) * 64);
  const uint32_t tyacc = tmem_slot + lane_q + 256u + (uint32_t)((warp >> 2) * 96);

  // step-3 roles: column product g, thread t3; step-1/2/4 roles: row, thread t48
  const int g = tid / 12, t3 = tid - g * 12;
  const int row = tid / 3, t48 = tid - row * 3;
  const fast::Tw0Rec tw0_192{a.tw192};

  for (long long item = blockIdx.x; item < a.batch; item += gridDim.x) {
    const cplx *H = a.h + item * a.h_bstride;
    const cplx *X = a.x + item * a.x_bstride;
#pragma unroll 1
    for (int r = 0; r < NR; ++r) {
      // ---- 1a/2a: folds (coalesced along the contiguous input dimension).
      // H is read once per residue: kept in L2 (evict_last) until the last one.
      uint64_t pol;
      if (r < NR - 1)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
      else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
      auto ldh = [&](const cplx *p) {
        cplx v;
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n"
                     : "=d"(v.x), "=d"(v.y)
                     : "l"(p), "l"(pol));
        return v;
      };
      constexpr int FB = 8;  // fold elements per thread whose loads are in flight together
      const int nfold = a.din * D;
#pragma unroll 1
      for (int e0 = 0; e0 < nfold; e0 += FB * NT) {
        cplx hv[FB][4];
#pragma unroll
        for (int b = 0; b < FB; ++b) {
          const int e = e0 + b * NT + tid;
          const int ar = e / D, np = e - ar * D;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = np + D * q;
            hv[b][q] = (e < nfold && c < a.dout) ? ldh(H + (long long)ar * a.dout + c)
                                                 : make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int b = 0; b < FB; ++b) {
          const int e = e0 + b * NT + tid;
          if (e < nfold) {
            const int ar = e / D, np = e - ar * D;
            cplx s = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const cplx w = rot4<true>(hv[b][q], q * r);
              s.x += w.x;
              s.y += w.y;
            }
            SA[sa_slot(np, ar)] = cmulc(s, __ldg(&a.tw192[(np * r) % L]));  // W^{-n' r}
          }
        }
      }
      for (int e = tid; e < XN * D; e += NT) {
        const int np = e / XN, i = e - np * XN;
        cplx s = make_double2(0.0, 0.0);
        if (i < a.n) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int j = np + D * q;
            if (j < a.N) {
              const cplx w = rot4<false>(fast::ld_stream(X + i + (long long)a.n * j), q * r);
              s.x += w.x;
              s.y += w.y;
            }
          }
          s = cmul(s, __ldg(&a.tw192[(np * r) % L]));  // W^{n' r}
        }
        XB[xb_slot(np, i)] = s;
      }
      // rows a >= din of S1 are the zero padding of the column products
      for (int e = tid; e < D * (L - a.din); e += NT) {
        const int m = e / (L - a.din), ar = a.din + (e - m * (L - a.din));
        SA[sa_slot(m, ar)] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      // ---- 1b: 48-point inverse DFTs of the din rows of S1 (in place)
#pragma unroll 1
      for (int r0 = 0; r0 < a.din; r0 += NROW) {
        const int rw = r0 + row;
        dft48<true>(SA, rw < a.din, t48, a.tw48, [&](int pos) { return sa_slot(pos, rw); });
      }
      // ---- 2b: 48-point forward DFTs of the n rows of X1 (in place)
      dft48<false>(XB, row < a.n, t48, a.tw48, [&](int pos) { return xb_slot(pos, row); });
      __syncthreads();
      // ---- 3: 48 column products of length 192 (product g = column m)
#pragma unroll 1
      for (int m0 = 0; m0 < D; m0 += NG) {
        const int m = m0 + g;
        auto ldS = [&](int, int, int pos) { return SA[sa_slot(m, pos)]; };
        auto stS = [&](int, int, int pos, cplx v) { SA[sa_slot(m, pos)] = v; };
        cplx v[P192::V];
        auto rs = [&](int i, int j, int, cplx x) { v[i * 16 + j] = x; };
        // S = ifft_a(S1 column): pass 0 in place, pass 1 into registers
        fast::pass<P192, 0, true, false, 12, 12>(t3, a.tw192, tw0_192, ldS, stS);
        __syncthreads();
        fast::pass<P192, 1, true, false, 16, 16>(t3, a.tw192, tw0_192, ldS, rs);
        tmem_wait_st();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st4(tacc + 16 * c, &v[4 * c]);
        __syncthreads();  // every S1 column read: the column is the exchange buffer now
        // X = fft_a(X1 column): nonzero rows i < n (four of the twelve pass-0 inputs)
        auto ldX = [&](int, int, int pos) {
          return pos < a.n ? XB[xb_slot(m, pos)] : make_double2(0.0, 0.0);
        };
        fast::pass<P192, 0, false, false, 4, 12>(t3, a.tw192, tw0_192, ldX, stS);
        __syncthreads();
        fast::pass<P192, 1, false, false, 16, 16>(t3, a.tw192, tw0_192, ldS, rs);
        tmem_wait_st();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          cplx acc[4];
          tmem_ld4(tacc + 16 * c, acc);
          for (int q = 0; q < a.power; ++q) {
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] = cmul(acc[e], v[4 * c + e]);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) v[4 * c + e] = acc[e];
        }
        __syncthreads();  // x pass-1 reads done before the final transform writes
        // Y column = fft_a(P)[i < n]: transposed DIT, pass 1 from registers
        auto rl = [&](int i, int j, int) { return v[i * 16 + j]; };
        fast::pass<P192, 1, false, true, 16, 16>(t3, a.tw192, tw0_192, rl, stS);
        __syncthreads();
        auto stY = [&](int, int, int pos, cplx val) {
          if (pos < a.n) XB[xb_slot(m, pos)] = val;
        };
        fast::pass<P192, 0, false, true, 12, 4>(t3, a.tw192, tw0_192, ldS, stY);
        __syncthreads();
      }
      // ---- 4: y[i][j] += W^{j r} DFT_48(Y_r[i][:])[j mod 48], rows i < n.
      // Threads 0..191 (warps 0-5, warp-uniform TMEM access) run the 64 row
      // DFTs; rows >= n compute on unused slots and store nothing.
      {
        const bool act = tid < 3 * XN;
        const fast::Tw0Rec tw0_48{a.tw48};
        auto ld = [&](int, int, int pos) { return XB[xb_slot(pos, row)]; };
        auto st = [&](int, int, int pos, cplx v) { XB[xb_slot(pos, row)] = v; };
        if (act) fast::pass<P48, 0, false, false, 3, 3>(t48, a.tw48, tw0_48, ld, st);
        __syncthreads();
        if (act) {
          cplx v[16];
          auto rs = [&](int i, int j, int, cplx x) { v[i * 16 + j] = x; };
          fast::pass<P48, 1, false, false, 16, 16>(t48, a.tw48, tw0_48, ld, rs);
          // accumulator slot s < 16: j = t48 + 3 s; slot 16 + s (s < 6): j + 48,
          // valid when t48 + 3 s < 16.  Chunks of four slots through TMEM.
          cplx *Y = a.y + item * a.y_bstride;
          const double sc = a.scale;
          tmem_wait_st();
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            cplx acc[4];
            if (r == 0) {
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[e] = make_double2(0.0, 0.0);
            } else {
              tmem_ld4(tyacc + 16 * c, acc);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int slot = 4 * c + e;
              const int q = slot < 16 ? slot : slot - 16;
              const int jj = t48 + 3 * q + (slot < 16 ? 0 : D);
              const bool ok = slot < 16 || (q < 6 && t48 + 3 * q < 16);
              if (ok) {
                const cplx w = cmul(v[q], __ldg(&a.tw192[(jj * r) % L]));
                acc[e].x += w.x;
                acc[e].y += w.y;
                if (r == NR - 1 && row < a.n && jj < a.N)
                  Y[row + (long long)a.n * jj] = make_double2(acc[e].x * sc, acc[e].y * sc);
              }
            }
            if (r < NR - 1) tmem_st4(tyacc + 16 * c, acc);
          }
        }
        __syncthreads();  // S1 / X1 regions are refilled by the next residue
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<512>(tmem_slot);
  }
}

constexpr int kSmem = (D * L + D * XN) * 16 + 128;

}  // namespace bhhb

// cudaErrorNotSupported outside the shapes the fused kernel covers.
cudaError_t launch_bhhb_fused(const bhhb::Args &a, cudaStream_t stream) {
  using namespace bhhb;
  // Opt-in (HK_BHHB_FUSED=1): measured on B200 cfg4 at 1849 us against 951 us
  // for the multi-kernel two-level path -- 9 resident warps (288 threads: the
  // 168-register cap of a >256-thread CTA already spills ~600 B) leave the FP64
  // pipe at ~10%, and the four residue passes re-read H (r02 profile).
  if (!getenv("HK_BHHB_FUSED")) return cudaErrorNotSupported;
  if (a.din > L || a.dout > L || a.n > XN || a.N > XN || a.n < 1 || a.N < 1 || a.power < 1 ||
      a.power > 8 || !a.tw48 || !a.tw192)
    return cudaErrorNotSupported;
  static std::atomic<unsigned long long> configured{0};
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e =
        cudaFuncSetAttribute(k_bhhb_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    configured.fetch_or(bit);
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long grid = std::min<long long>(a.batch, sms[dev & 63]);
  k_bhhb_fused<<<(unsigned)grid, NT, kSmem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace hk
