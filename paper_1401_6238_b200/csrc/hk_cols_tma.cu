// K3t: TMA-fed column passes of the 1D four-step for the real-operand product
// (cfg3, reference hankel.py:140-147 at L = 1536 x 8192).
//
// The generic column kernel (hk_large.cu) streams its tiles with per-thread
// 8/16-byte cp.async and stores them with per-element index arithmetic; on
// cfg3 that integer work and its latency were 44% of the stall samples (ncu
// source page, r02).  Here the Tensor Memory Accelerator moves each column
// tile: ONE thread issues 2-D boxes [TILE columns x 256 rows] of the row-major
// L1 x L2 view (zero fill past the operand), an mbarrier collects the bytes,
// and the next tile's boxes land in a separate landing buffer while the
// current tile is transformed in the exchange buffer.
//
//   ST_A_PAIR: z = h + i x (real h, real x), forward column DFT, split by
//              conjugate symmetry into the stage-A outputs of h (inverse, 1/L,
//              four-step twiddle) and x (forward, twiddle); rows k <= L1/2
//              only when `half` (the Hermitian product, see hk_capi.cu).
//   ST_C:      the final column pass over the row-stage output Q, rows above
//              L1/2 synthesised from row L1 - k1 (Hermitian), truncated to y.
//
// Pass 0 reads the landing boxes with an interleaved thread mapping (lanes
// run along the TILE columns of a row first: conflict-free 8/16-byte reads of
// the packed boxes); passes >= 1 and the epilogue use the column-major mapping
// of k_cols on the swizzled exchange buffer.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

#include "hk_fastcore.cuh"
#include "hk_large.h"

namespace hk {
namespace large {

struct alignas(64) ColTma {
  CUtensorMap m_in;    // ST_A_PAIR: h (f64 [items][rows][L2]); ST_C: Q (f64 pairs)
  CUtensorMap m_in2;   // ST_A_PAIR: x
  CUtensorMap m_in4;   // m_in as [items][blocks][256 rows][L2]: all full 256-row blocks in ONE copy
  CUtensorMap m_in24;  // the same view of x
  CUtensorMap m_out;   // tma_out: stage-A output of h (or of the operand) / y
  CUtensorMap m_out2;  // tma_out, ST_A_PAIR: stage-A output of x
  ColArgs a;
  long long rows_in, rows_in2;  // full rows the maps cover (TMA zero-fills below)
  long long tail_in, tail_in2;  // valid elements of the partial row after them
  int32_t tma_out;              // 1: epilogue stores the tile with TMA (row-major staging)
  int32_t out_rows;             // rows of the output tile (stage A: e1; ST_C: len / L2)
  int32_t nat_swz;              // natural-order column layout: k ^ ((k >> 3) & nat_swz)
  int32_t nb_in, nb_in2;        // landing boxes that hold operand rows (the rest stay zero)
  int32_t fb_in, fb_in2;        // of which full 256-row blocks (one 4-D copy; < nb: one more box)
  long long c_q, c_rem;         // ST_C: out.len = c_q * L2 + c_rem
};

namespace tma {

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
__device__ __forceinline__ void load3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                       uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void load4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                       int c3, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void store3d(const CUtensorMap *map, int c0, int c1, int c2, uint32_t src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// named barrier with a runtime id over N threads (one column group)
template <int N>
struct GroupBar {
  int id;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(N) : "memory");
  }
};

}  // namespace tma

// W_L^e for 0 <= e < 2L: every call site multiplies a column index n2 < L2 + TILE
// by a row index < L1 (or by L1 itself), so one conditional subtraction
// replaces the emulated 64-bit modulo (~100 dependent instructions per call).
__device__ __forceinline__ cplx tw4(const ColArgs &a, long long e) {
  if (e >= a.L) e -= a.L;
  return cmul(__ldg(&a.thi[e >> 12]), __ldg(&a.tlo[e & 4095]));
}

// The two table reads of a W_L^e lookup without their product: issued ahead of
// a wait or barrier, multiplied after it (the loads then overlap the wait).
struct Tw4Raw {
  cplx hi, lo;
  __device__ __forceinline__ cplx get() const { return cmul(hi, lo); }
};
__device__ __forceinline__ Tw4Raw tw4_raw(const ColArgs &a, long long e) {
  if (e >= a.L) e -= a.L;
  return Tw4Raw{__ldg(&a.thi[e >> 12]), __ldg(&a.tlo[e & 4095])};
}

// Column-pass twiddles in TMEM (r02): a thread's twiddles are the same for
// every tile (pass 0: W_L1^{j beta} of its NB0 butterflies, pass 1: W_256^{j lo}),
// so they are read once from the W_L1 table and kept next to nothing else in
// TMEM -- no dependent table reads and no recurrence per tile.
template <class PL>
struct ColTw {
  static constexpr int R0 = PL::radix[0], R1 = PL::radix[1], T = PL::T;
  static constexpr int NB0 = (PL::L / R0 + T - 1) / T;  // pass-0 butterflies per thread
  static constexpr int NC0 = (R0 - 1 + 3) / 4, NC1 = (R1 - 1 + 3) / 4;
  static constexpr int SLAB = (NB0 * NC0 + NC1) * 16;  // columns per warp slab
  uint32_t taddr;
  __device__ __forceinline__ void chunk(int beta, int c, cplx *w) const {
    tmem_ld4(taddr + 16 * ((beta / T) * NC0 + c), w);
  }
  __device__ __forceinline__ void chunk1(int c, cplx *w) const {
    tmem_ld4(taddr + 16 * (NB0 * NC0 + c), w);
  }
};

template <class PL, int TILE, int STAGE>
struct TmaLayout {
  static constexpr int L1 = PL::L;
  static constexpr int BR = 256;  // box rows
  static constexpr int PAD = TILE >= 8 ? 1 : 8 / TILE;
  static constexpr int CS = L1 + PAD;
  static constexpr bool PAIR = STAGE == ST_A_PAIR;
  // ST_C lands at most L1 complex rows (all of them without `half`)
  static constexpr int LAND = PAIR ? 2 * L1 * TILE * 8 : L1 * TILE * 16;
  // TMA-store epilogue of the Hermitian pair: H rows [0, R), X rows from XOFF
  // (128-byte aligned), row-major [row][TILE] in the exchange buffer
  static constexpr int R = L1 / 2 + 1;
  static constexpr int XOFF = (R + (8 / TILE) - 1) / (8 / TILE) * (8 / TILE);
  static constexpr int EX0 = TILE * CS * 16, EX1 = (XOFF + R) * TILE * 16;
  static constexpr int EX = EX0 > EX1 ? EX0 : EX1;
  static constexpr int SMEM = LAND + EX + 128;
  static_assert(L1 % BR == 0, "column length must be a multiple of the box height");
};

// DEC: the TILE columns run as independent thread groups (named barriers per
// column); they meet only when the landing buffer is refilled, which the
// last group to finish its pass 0 triggers.  Otherwise CTA-wide barriers.
template <class PL, int TILE, int STAGE, bool DEC>
__global__ void __launch_bounds__(TILE * PL::T, 1)
    k_cols_tma(const __grid_constant__ ColTma g, int tiles_per_item, long long ntiles) {
  using LY = TmaLayout<PL, TILE, STAGE>;
  constexpr int L1 = PL::L, T = PL::T, V = PL::V, RL = PL::Rlast, R0 = PL::radix[0];
  constexpr int CS = LY::CS, BR = LY::BR, NT = TILE * T;
  constexpr bool PAIR = LY::PAIR;
  constexpr bool SC = STAGE == ST_C;
  constexpr bool INV = STAGE == ST_A_INV;
  const ColArgs &a = g.a;
  // single-operand stage A: complex (16-byte) or real (8-byte) landing rows
  const bool cin = SC || (!PAIR && a.in.kind == FK_C128);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t mbar;
  unsigned char *base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  double *land = reinterpret_cast<double *>(base);
  cplx *landc = reinterpret_cast<cplx *>(base);
  cplx *ex = reinterpret_cast<cplx *>(base + LY::LAND);
  const uint32_t mb = smem_u32(&mbar);
  __shared__ int land_rel;  // DEC: column groups done with the landing buffer
  const int cg = threadIdx.x / T;  // DEC: this thread's column group
  const tma::GroupBar<T> gbar_{1 + cg};
  auto bar = [&]() {
    if constexpr (DEC)
      gbar_();
    else
      __syncthreads();
  };

  // Tile (item, c0) into the landing buffer: ONE 4-D tensor copy moves every
  // full 256-row block of an operand ([blocks][256][TILE] lands contiguously),
  // one more 3-D box the partial block (zero fill past the operand's rows).
  // r02 ncu: the 16-24 per-block copies of a tile cost their single issuer
  // 1-2k cycles while the other warps waited at the next CTA barrier (13% of
  // the packed pass); dealt over the warps they cost every warp a descriptor
  // waterfall.  Two or three copies by one thread are cheap.
  const int nb1 = g.nb_in, nb2 = PAIR ? g.nb_in2 : 0;
  const int fb1 = g.fb_in, fb2 = PAIR ? g.fb_in2 : 0;
  auto issue = [&](int item, int c0) {
    const uint32_t esz = (PAIR || !cin) ? 8u : 16u;
    const int f = (PAIR || !cin) ? 1 : 2;  // f64 elements per operand element
    tma::mbar_expect_tx(mb, (uint32_t)(nb1 + nb2) * BR * TILE * esz);
    unsigned char *l1 = base, *l2 = base + L1 * TILE * 8;
    if (fb1 > 0) tma::load4d(smem_u32(l1), &g.m_in4, f * c0, 0, 0, item, mb);
    if (nb1 > fb1)
      tma::load3d(smem_u32(l1 + fb1 * BR * TILE * esz), &g.m_in, f * c0, fb1 * BR, item, mb);
    if constexpr (PAIR) {
      if (fb2 > 0) tma::load4d(smem_u32(l2), &g.m_in24, c0, 0, 0, item, mb);
      if (nb2 > fb2)
        tma::load3d(smem_u32(l2 + fb2 * BR * TILE * 8), &g.m_in2, c0, fb2 * BR, item, mb);
    }
  };
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    tma::mbar_init(mb, 1);
    land_rel = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if constexpr (!SC) {
    // boxes wholly past the operand's rows are never issued: their landing
    // rows are zeroed once here and only ever read
    for (int i = threadIdx.x; i < LY::LAND / 16; i += NT) landc[i] = make_double2(0.0, 0.0);
    tma::fence_proxy_async();
  }
  __syncthreads();
  // tile w = (item, tcol) advances by gridDim.x tiles without 64-bit divisions
  long long w = blockIdx.x;
  int item = (int)(blockIdx.x / (unsigned)tiles_per_item);
  int tcol = (int)(blockIdx.x % (unsigned)tiles_per_item);
  const int d_item = (int)(gridDim.x / (unsigned)tiles_per_item);
  const int d_tcol = (int)(gridDim.x % (unsigned)tiles_per_item);
  auto next_tile = [&](int &it_, int &tc_) {
    it_ += d_item;
    tc_ += d_tcol;
    if (tc_ >= tiles_per_item) {
      tc_ -= tiles_per_item;
      ++it_;
    }
  };
  if (threadIdx.x == 0 && w < ntiles) issue(item, tcol * TILE);
  // ---- twiddle slabs in TMEM (see ColTw); 12 warps: three slabs per lane quadrant
  using CT = ColTw<PL>;
  static_assert(((TILE * T / 32 + 3) / 4) * CT::SLAB <= 512, "twiddle slabs exceed TMEM");
  static_assert(PL::P == 3, "pass-1 twiddle slab assumes a three-pass column plan");
  __shared__ uint32_t tmem_slot;
  if (warp == 0) tmem_alloc<512>(&tmem_slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const CT tw0{tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * CT::SLAB)};
  {
    const int tc = threadIdx.x % T;
    const int tp = DEC ? tc : threadIdx.x / TILE;  // pass-0 thread index
#pragma unroll
    for (int i = 0; i < CT::NB0; ++i) {
      const int beta = tp + i * T;
#pragma unroll
      for (int c = 0; c < CT::NC0; ++c) {
        cplx w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 4 * c + q + 1;
          w[q] = (j < R0 && beta < L1 / R0) ? __ldg(&a.ctw[(j * beta) % L1])
                                             : make_double2(1.0, 0.0);
        }
        tmem_st4(tw0.taddr + 16 * (i * CT::NC0 + c), w);
      }
    }
    // pass 1 (lo-major with a per-thread slab, fast::pass): lo = t mod stride(1)
    constexpr int S1 = PL::stride(1), RR1 = PL::radix[1], LP1 = S1 * RR1;
    const int lo = tc % S1;
#pragma unroll
    for (int c = 0; c < CT::NC1; ++c) {
      cplx w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * c + q + 1;
        w[q] = j < RR1 ? __ldg(&a.ctw[(j * lo * (L1 / LP1)) % L1]) : make_double2(1.0, 0.0);
      }
      tmem_st4(tw0.taddr + 16 * (CT::NB0 * CT::NC0 + c), w);
    }
    tmem_wait_st();
  }

  for (int it = 0; w < ntiles; ++it, w += gridDim.x, next_tile(item, tcol)) {
    const int c0 = tcol * TILE;
    // ST_C: the four-step twiddles of this thread's pass-0 butterflies (table
    // reads that miss L1 next to 197 KB of shared memory) are requested before
    // the wait for the tile, not between the wait and the first butterfly
    constexpr int NB0 = ColTw<PL>::NB0;
    const Tw4Raw one_raw{make_double2(1.0, 0.0), make_double2(1.0, 0.0)};
    Tw4Raw rz_step = one_raw, rz_row = one_raw, rz_cur[NB0];
    if constexpr (SC) {
      const int c = DEC ? cg : threadIdx.x % TILE;
      const int tp = DEC ? (int)(threadIdx.x % T) : threadIdx.x / TILE;
      const int n2 = c0 + c;
      rz_step = tw4_raw(a, (long long)n2 * PL::stride(0));
      if (a.half) rz_row = tw4_raw(a, (long long)n2 * L1);  // W_L2^{n2}
#pragma unroll
      for (int i = 0; i < NB0; ++i) {
        const int beta = tp + i * T;
        rz_cur[i] = beta < L1 / R0 ? tw4_raw(a, (long long)n2 * beta) : rz_step;
      }
    }
    tma::mbar_wait(mb, (uint32_t)(it & 1));
    cplx pz_step = rz_step.get(), pz_row = rz_row.get(), pz_cur[NB0];
#pragma unroll
    for (int i = 0; i < NB0; ++i) pz_cur[i] = rz_cur[i].get();
    if (g.tma_out) {  // the previous tile's TMA stores have read the exchange buffer
      if (threadIdx.x == 0) tma::bulk_wait_read();
      if constexpr (SC) __syncthreads();
    }
    if constexpr (!SC) {
      // partial last rows of the operands (the maps cover full rows only);
      // DEC: threads 0 and 1 of each column group patch that column
      const int tf = DEC ? (threadIdx.x % T) * TILE + cg : (int)threadIdx.x;
      const bool fixer = DEC ? (threadIdx.x % T) < 2 : threadIdx.x < 2 * TILE;
      if (fixer) {
        const int c = DEC ? cg : tf % TILE;
        const bool second = DEC ? (threadIdx.x % T) == 1 : tf >= TILE;
        const long long rows = second ? g.rows_in2 : g.rows_in;
        const long long tail = second ? g.tail_in2 : g.tail_in;
        if ((PAIR || !second) && tail > 0 && rows < L1) {
          const Op2 &op = second ? a.in2 : a.in;
          const int n2 = c0 + c;
          const long long e = item * op.item_stride + rows * a.L2 + n2;
          if (cin) {
            landc[rows * TILE + c] = n2 < tail ? static_cast<const cplx *>(op.ptr)[e]
                                               : make_double2(0.0, 0.0);
          } else {
            land[((second ? L1 : 0) + rows) * TILE + c] =
                n2 < tail ? static_cast<const double *>(op.ptr)[e] : 0.0;
          }
        }
      }
      bar();
    }
    // ---- pass 0 from the landing boxes (interleaved mapping; DEC: the group's column)
    {
      const int c = DEC ? cg : threadIdx.x % TILE;
      const int tp = DEC ? (int)(threadIdx.x % T) : threadIdx.x / TILE;
      cplx *col = ex + c * CS;
      cplx tw_cur = make_double2(1.0, 0.0);
      const cplx tw_step = pz_step, wrow = pz_row;
      auto in_load = [&](int i, int j, int pos) {
        if constexpr (PAIR) {
          return make_double2(land[pos * TILE + c], land[(L1 + pos) * TILE + c]);
        } else if constexpr (!SC) {
          const double sc = a.in.scale;
          if (cin) {
            const cplx v = landc[pos * TILE + c];
            return make_double2(v.x * sc, v.y * sc);
          }
          return make_double2(land[pos * TILE + c] * sc, 0.0);
        } else {
          cplx v;
          if (a.half && 2 * pos > L1) {
            // Q(L1-k1, m2) = conj(W_L2^{m2} Q(k1, m2))
            v = cmul(landc[(L1 - pos) * TILE + c], wrow);
            v.y = -v.y;
          } else {
            v = landc[pos * TILE + c];
          }
          v.x *= a.in.scale;
          v.y *= a.in.scale;
          if (j == 0) tw_cur = pz_cur[i];  // W_L^{n2 beta}: pos = beta + j S0
          v = cmul(v, tw_cur);
          tw_cur = cmul(tw_cur, tw_step);
          return v;
        }
      };
      auto s_store = [&](int, int, int pos, cplx v) { col[fast::swz2(pos)] = v; };
      fast::pass<PL, 0, INV, false, R0, R0>(tp, a.ctw, tw0, in_load, s_store);
    }
    bar();
    // the landing buffer is consumed: stream the next tile in behind the math
    if constexpr (DEC) {
      if (threadIdx.x % T == 0) {  // the last column group to get here refills
        __threadfence_block();
        if (atomicAdd(&land_rel, 1) == TILE - 1) {
          land_rel = 0;
          __threadfence_block();
          if (w + gridDim.x < ntiles) {
            int ni = item, nc = tcol;
            next_tile(ni, nc);
            tma::fence_proxy_async();
            issue(ni, nc * TILE);
          }
        }
      }
    } else if (threadIdx.x == 0 && w + gridDim.x < ntiles) {
      int ni = item, nc = tcol;
      next_tile(ni, nc);
      tma::fence_proxy_async();
      issue(ni, nc * TILE);
    }
    const int c = threadIdx.x / T, t = threadIdx.x - (threadIdx.x / T) * T;
    const int n2 = c0 + c;
    cplx *col = ex + c * CS;
    auto s_load = [&](int, int, int pos) { return col[fast::swz2(pos)]; };
    auto s_store = [&](int, int, int pos, cplx v) { col[fast::swz2(pos)] = v; };
    cplx v[V];
    auto r_store = [&](int i, int j, int, cplx x) { v[i * RL + j] = x; };
    sfor<PL::P - 2>([&](auto qc) {
      constexpr int q = decltype(qc)::value + 1;
      fast::pass<PL, q, INV, false, PL::radix[q], PL::radix[q], L1, true>(t, a.ctw, tw0, s_load,
                                                                         s_store);
      bar();
    });
    // ST_C keeps only rows k < out_rows of y: when they fit in the first NOC
    // outputs of every last-pass butterfly (k = k0 + j L1/RL, j < NOC), the
    // pruned last pass computes NOC of the RL outputs
    constexpr int NOC = 6;
    const bool prune = SC && !g.tma_out && g.out_rows <= NOC * (L1 / RL);
    if (prune)
      fast::pass<PL, PL::P - 1, INV, false, RL, NOC, L1, true>(t, a.ctw, tw0, s_load, r_store);
    else
      fast::pass<PL, PL::P - 1, INV, false, RL, RL, L1, true>(t, a.ctw, tw0, s_load, r_store);
    bar();
    // digit-reversed registers -> natural order: register j of butterfly beta
    // holds frequency k = k(beta) + j * L1 / RL; single-operand stage A also
    // applies the four-step twiddle W_L^{-+n2 k} (geometric in j)
    // natural-order positions are XOR-swizzled (bank conflicts of the
    // digit-reversed writes at L1 = 3072: 8 wavefronts per warp store -> 4)
    const int nswz = g.nat_swz;
    auto nat = [nswz](int k) { return k ^ ((k >> 3) & nswz); };
    constexpr bool TW_A = !PAIR && !SC;
    const cplx tws = TW_A ? tw4(a, (long long)n2 * (L1 / RL)) : make_double2(1.0, 0.0);
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
      cplx cur = TW_A ? tw4(a, (long long)n2 * k0) : make_double2(1.0, 0.0);
#pragma unroll
      for (int j = 0; j < RL; ++j) {
        if (SC && prune && j >= NOC) break;
        cplx x = v[i * RL + j];
        if constexpr (TW_A) {
          x = INV ? cmulc(x, cur) : cmul(x, cur);
          cur = cmul(cur, tws);
        }
        const int k = k0 + j * (L1 / RL);
        if (g.tma_out)
          ex[k * TILE + c] = x;  // row-major staging for the TMA store
        else
          col[nat(k)] = x;
      }
    }
    // PAIR: the split's twiddles are requested before the barrier, not after it
    Tw4Raw rs_wk = one_raw, rs_step = one_raw;
    if constexpr (PAIR) {
      if (!g.tma_out) {
        rs_wk = tw4_raw(a, (long long)n2 * t);
        rs_step = tw4_raw(a, (long long)n2 * T);
      }
    }
    bar();
    const cplx ps_wk = rs_wk.get(), ps_step = rs_step.get();
    if (g.tma_out) {
      // ---- TMA-store epilogue
      if constexpr (PAIR) {
        constexpr int R = LY::R, XO = LY::XOFF, NP = (R + T - 1) / T;
        cplx za[NP], zb[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int k = t + p * T;
          if (k < R) {
            za[p] = ex[k * TILE + c];
            zb[p] = ex[(k == 0 ? 0 : L1 - k) * TILE + c];
          }
        }
        __syncthreads();
        const double sh = a.in.scale;
        cplx wk = tw4(a, (long long)n2 * t);
        const cplx wstep = tw4(a, (long long)n2 * T);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int k = t + p * T;
          if (k < R) {
            const cplx A = za[p], B = zb[p];
            const cplx H = make_double2(0.5 * (A.x + B.x), 0.5 * (A.y - B.y));
            const cplx X = make_double2(0.5 * (A.y + B.y), 0.5 * (B.x - A.x));
            const cplx hk = cmul(H, wk), xk = cmul(X, wk);
            ex[k * TILE + c] = make_double2(hk.x * sh, -hk.y * sh);
            ex[(XO + k) * TILE + c] = xk;
          }
          wk = cmul(wk, wstep);
        }
      }
      tma::fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int rows = g.out_rows;
        const int inner = 2 * c0;
        for (int r0 = 0; r0 < rows; r0 += BR) {
          tma::store3d(&g.m_out, inner, r0, (int)item, smem_u32(ex + r0 * TILE));
          if constexpr (PAIR)
            tma::store3d(&g.m_out2, inner, r0, (int)item, smem_u32(ex + (LY::XOFF + r0) * TILE));
        }
        tma::bulk_commit();
      }
      continue;  // the next tile waits for these reads before reusing ex
    }
    if constexpr (PAIR) {
      // Z(k) = H(k) + i X(k):  H(k) = (Z(k) + conj Z(-k)) / 2,
      // X(k) = (Z(k) - conj Z(-k)) / 2i; h takes the inverse (conj H, 1/L)
      // and both the four-step twiddle W_L^{+-n2 k}.  Twiddles by recurrence:
      // W^{n2 (t + pT)} = W^{n2 t} (W^{n2 T})^p, W^{n2 (L1 - k)} = W_L2^{n2} conj W^{n2 k}.
      constexpr int NP = (L1 / 2 + 1 + T - 1) / T;
      cplx xa[NP], xb[NP];
      const double sh = a.in.scale;
      const int rows_out = a.out.e1;  // L1/2 + 1 with `half`, else L1
      // rows above L1/2 are never stored for the Hermitian product: skip their
      // twiddles and products (3 of the 6 complex multiplies per pair)
      const bool upper = rows_out > L1 / 2 + 1;
      cplx wk = ps_wk;
      const cplx wstep = ps_step;
      const cplx wl1 = upper ? tw4(a, (long long)n2 * L1) : make_double2(1.0, 0.0);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int k = t + p * T;
        if (k <= L1 / 2) {
          const int kk = k == 0 ? 0 : L1 - k;
          const cplx A = col[nat(k)], B = col[nat(kk)];
          const cplx H = make_double2(0.5 * (A.x + B.x), 0.5 * (A.y - B.y));
          const cplx X = make_double2(0.5 * (A.y + B.y), 0.5 * (B.x - A.x));
          const cplx hk = cmul(H, wk);
          xa[p] = cmul(X, wk);
          col[nat(k)] = make_double2(hk.x * sh, -hk.y * sh);
          if (upper) {
            const cplx wkk = k == 0 ? wk : cmulc(wl1, wk);
            const cplx hkk = cmulc(H, wkk);
            xb[p] = cmul(make_double2(X.x, -X.y), wkk);
            if (kk != k) col[nat(kk)] = make_double2(hkk.x * sh, hkk.y * sh);
          }
        }
        wk = cmul(wk, wstep);
      }
      bar();
      // thread -> fixed column cc = tid % TILE, rows r0, r0 + NT/TILE, ...
      auto store_rows = [&](const Out2 &o) {
        const int cc = DEC ? cg : threadIdx.x % TILE;
        if (c0 + cc >= a.L2) return;
        constexpr int RS = DEC ? T : NT / TILE;
        const cplx *src = ex + cc * CS;
        cplx *d = static_cast<cplx *>(o.ptr) + item * o.item_stride + c0 + cc;
        const long long step = (long long)RS * o.s1;
        int r = DEC ? (int)(threadIdx.x % T) : threadIdx.x / TILE;
        d += r * o.s1;
        for (; r < rows_out; r += RS, d += step) *d = src[nat(r)];
      };
      store_rows(a.out);
      bar();
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int k = t + p * T;
        if (k > L1 / 2) continue;
        col[nat(k)] = xa[p];
        if (upper && k != 0 && 2 * k != L1) col[nat(L1 - k)] = xb[p];
      }
      bar();
      store_rows(a.out2);
    } else if constexpr (!SC) {
      const Out2 &o = a.out;
      const int rows = o.e1 < L1 ? o.e1 : L1;
      const int cc = DEC ? cg : threadIdx.x % TILE;
      if (c0 + cc < o.e2) {
        constexpr int RS = DEC ? T : NT / TILE;
        const cplx *src = ex + cc * CS;
        int r = DEC ? (int)(threadIdx.x % T) : threadIdx.x / TILE;
        cplx *d = static_cast<cplx *>(o.ptr) + item * o.item_stride + c0 + cc + r * o.s1;
        for (; r < rows; r += RS, d += (long long)RS * o.s1) *d = src[nat(r)];
      }
    } else {
      // y(m2 + L2 k) for the rows k with m2 + L2 k < len: column n2 has
      // c_q + (n2 < c_rem) of them (out.len = c_q L2 + c_rem, split on the host)
      const Out2 &o = a.out;
      auto nrows = [&](int n2c) {
        const long long kr = g.c_q + (n2c < g.c_rem ? 1 : 0);
        return (int)(kr < L1 ? kr : L1);
      };
      const int cc = DEC ? cg : threadIdx.x % TILE;
      if (c0 + cc < a.L2) {
        const int rows = nrows(c0 + cc);
        constexpr int RS = DEC ? T : NT / TILE;
        const cplx *src = ex + cc * CS;
        int r = DEC ? (int)(threadIdx.x % T) : threadIdx.x / TILE;
        cplx *d = static_cast<cplx *>(o.ptr) + item * o.item_stride + (c0 + cc) * o.s2 + r * o.s1;
        for (; r < rows; r += RS, d += (long long)RS * o.s1) *d = src[nat(r)];
      }
    }
    bar();  // exchange buffer reused by the next tile's pass 0
  }
  if (g.tma_out && threadIdx.x == 0) tma::bulk_wait();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc<512>(tmem_slot);
  }
}

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// f64 view [items][rows][inner] with row stride `rs` and item stride `is`
// (elements); box [bx, 256, 1].
static bool encode(CUtensorMap *m, const void *ptr, long long inner, long long rows,
                   long long items, long long rs, long long is, int bx) {
  EncodeFn fn = encode_fn();
  if (!fn || rows <= 0 || inner <= 0) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (rs * 8) % 16 || (is * 8) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)(items > 0 ? items : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(rs * 8), (cuuint64_t)((is > 0 ? is : rs * rows) * 8)};
  cuuint32_t box[3] = {(cuuint32_t)bx, 256u, 1u};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void *>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The first `fb` full 256-row blocks of the same view as a 4-D tensor
// [items][fb][256][inner], box [bx, 256, fb, 1]: one copy per tile and operand.
static bool encode4(CUtensorMap *m, const void *ptr, long long inner, int fb, long long items,
                    long long rs, long long is, int bx) {
  EncodeFn fn = encode_fn();
  if (!fn || fb <= 0 || fb > 256 || inner <= 0) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (rs * 8) % 16 || (is * 8) % 16) return false;
  cuuint64_t dims[4] = {(cuuint64_t)inner, 256u, (cuuint64_t)fb, (cuuint64_t)(items > 0 ? items : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)(rs * 8), (cuuint64_t)(256 * rs * 8),
                           (cuuint64_t)((is > 0 ? is : rs * 256 * fb) * 8)};
  cuuint32_t box[4] = {(cuuint32_t)bx, 256u, (cuuint32_t)fb, 1u};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class PL, int TILE, int STAGE, bool DEC>
static cudaError_t launch_t2(ColTma &g, long long items, int ncols, cudaStream_t stream);

// DEC (independent column groups, HK_COL_DEC=1) measured slower on B200 cfg3:
// 433 vs 378 us -- per-column pass-0 reads of the packed landing rows and
// per-column 16-byte row stores cost more than the CTA barriers they remove.
template <class PL, int TILE, int STAGE>
static cudaError_t launch_t(ColTma &g, long long items, int ncols, cudaStream_t stream) {
  const bool dec = !g.tma_out && getenv("HK_COL_DEC") && atoi(getenv("HK_COL_DEC")) == 1;
  return dec ? launch_t2<PL, TILE, STAGE, true>(g, items, ncols, stream)
             : launch_t2<PL, TILE, STAGE, false>(g, items, ncols, stream);
}

template <class PL, int TILE, int STAGE, bool DEC>
static cudaError_t launch_t2(ColTma &g, long long items, int ncols, cudaStream_t stream) {
  g.nat_swz = PL::L == 3072 ? 7 : 0;
  if (const char *e = getenv("HK_COL_NATSWZ")) g.nat_swz = atoi(e) & 7;
  using LY = TmaLayout<PL, TILE, STAGE>;
  static std::atomic<unsigned long long> configured{0};
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k_cols_tma<PL, TILE, STAGE, DEC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, LY::SMEM);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    configured.fetch_or(bit);
  }
  const int tiles = (ncols + TILE - 1) / TILE;
  const long long ntiles = (long long)tiles * items;
  if (ntiles <= 0) return cudaSuccess;
  const long long grid = std::min<long long>(ntiles, sms[dev & 63]);
  k_cols_tma<PL, TILE, STAGE, DEC><<<(unsigned)grid, TILE * PL::T, LY::SMEM, stream>>>(g, tiles, ntiles);
  return cudaGetLastError();
}

}  // namespace large

namespace large {
template <class PL, int TILE>
static cudaError_t launch_cols_tma_t(int stage, const ColArgs &a, long long items, int ncols,
                                     cudaStream_t stream) {
  ColTma g{};
  g.a = a;
  const long long L2 = a.L2;
  auto full_rows = [&](const Op2 &op, long long *rows, long long *tail) {
    *rows = std::min<long long>(a.L1, op.len / L2);
    *tail = op.len - *rows * L2;
    return *rows > 0 && *tail < L2;
  };
  // landing boxes (256 rows) that hold operand rows, the partial last row included
  auto boxes = [&](long long rows, long long tail) {
    const long long r = std::min<long long>(a.L1, rows + (tail > 0 ? 1 : 0));
    return (int)((r + 255) / 256);
  };
  if (stage == ST_A_PAIR) {
    const Op2 &h = a.in, &x = a.in2;
    if (h.kind != FK_F64 || x.kind != FK_F64 || h.s1 != L2 || h.s2 != 1 || x.s1 != L2 ||
        x.s2 != 1 || h.len < 0 || x.len < 0 || a.out.s2 != 1 || a.out2.s2 != 1)
      return cudaErrorNotSupported;
    if (!full_rows(h, &g.rows_in, &g.tail_in) || !full_rows(x, &g.rows_in2, &g.tail_in2))
      return cudaErrorNotSupported;
    if (!encode(&g.m_in, h.ptr, L2, g.rows_in, items, L2, h.item_stride, TILE) ||
        !encode(&g.m_in2, x.ptr, L2, g.rows_in2, items, L2, x.item_stride, TILE))
      return cudaErrorNotSupported;
    // TMA stores of the Hermitian half (rows 0..L1/2 of both outputs)
    const Out2 &o1 = a.out, &o2 = a.out2;
    g.out_rows = o1.e1;
    g.tma_out = getenv("HK_COLTMA_STORE") && o1.e1 == a.L1 / 2 + 1 && o2.e1 == o1.e1 &&
                o1.e2 == L2 && o2.e2 == L2 && o1.len < 0 && o2.len < 0 &&
                encode(&g.m_out, o1.ptr, 2 * L2, o1.e1, items, 2 * o1.s1, 2 * o1.item_stride,
                       2 * TILE) &&
                encode(&g.m_out2, o2.ptr, 2 * L2, o2.e1, items, 2 * o2.s1, 2 * o2.item_stride,
                       2 * TILE);
    g.nb_in = boxes(g.rows_in, g.tail_in);
    g.nb_in2 = boxes(g.rows_in2, g.tail_in2);
    g.fb_in = (int)(g.rows_in / 256);
    g.fb_in2 = (int)(g.rows_in2 / 256);
    if ((g.fb_in > 0 && !encode4(&g.m_in4, h.ptr, L2, g.fb_in, items, L2, h.item_stride, TILE)) ||
        (g.fb_in2 > 0 && !encode4(&g.m_in24, x.ptr, L2, g.fb_in2, items, L2, x.item_stride, TILE)))
      return cudaErrorNotSupported;
    return launch_t<PL, TILE, ST_A_PAIR>(g, items, ncols, stream);
  }
  if (stage == ST_A_FWD || stage == ST_A_INV) {
    const Op2 &op = a.in;
    const bool cx = op.kind == FK_C128;
    if ((!cx && op.kind != FK_F64) || op.s1 != L2 || op.s2 != 1 || op.len < 0 || a.out.s2 != 1 ||
        a.out.len >= 0 || a.in_n1_fast)
      return cudaErrorNotSupported;
    if (!full_rows(op, &g.rows_in, &g.tail_in)) return cudaErrorNotSupported;
    const int f = cx ? 2 : 1;
    if (!encode(&g.m_in, op.ptr, f * L2, g.rows_in, items, f * L2, f * op.item_stride, f * TILE))
      return cudaErrorNotSupported;
    const Out2 &o = a.out;
    g.out_rows = std::min<int>(o.e1, a.L1);
    g.tma_out = getenv("HK_COLTMA_STORE") &&
                encode(&g.m_out, o.ptr, 2 * (long long)o.e2, g.out_rows, items, 2 * o.s1,
                       2 * o.item_stride, 2 * TILE);
    g.nb_in = boxes(g.rows_in, g.tail_in);
    g.fb_in = (int)(g.rows_in / 256);
    if (g.fb_in > 0 &&
        !encode4(&g.m_in4, op.ptr, f * L2, g.fb_in, items, f * L2, f * op.item_stride, f * TILE))
      return cudaErrorNotSupported;
    return stage == ST_A_FWD ? launch_t<PL, TILE, ST_A_FWD>(g, items, ncols, stream)
                             : launch_t<PL, TILE, ST_A_INV>(g, items, ncols, stream);
  }
  if (stage == ST_C) {
    const Op2 &q = a.in;
    if (q.kind != FK_C128 || q.s1 != L2 || q.s2 != 1 || q.len >= 0 || q.e2 < ncols)
      return cudaErrorNotSupported;
    const long long rows = a.half ? a.L1 / 2 + 1 : a.L1;
    if (q.e1 < rows || !encode(&g.m_in, q.ptr, 2 * L2, rows, items, 2 * L2, 2 * q.item_stride,
                               2 * TILE))
      return cudaErrorNotSupported;
    // y rows of L2 contiguous outputs: TMA stores when y is a whole number of rows
    const Out2 &o = a.out;
    g.out_rows = (int)std::min<long long>(o.len / L2, a.L1);
    g.tma_out = getenv("HK_COLTMA_STORE") && o.len > 0 && o.len % L2 == 0 && o.s2 == 1 &&
                o.s1 == L2 &&
                encode(&g.m_out, o.ptr, 2 * L2, g.out_rows, items, 2 * L2, 2 * o.item_stride,
                       2 * TILE);
    g.nb_in = (int)((a.half ? (rows + 255) / 256 * 256 : (long long)a.L1) / 256);
    g.fb_in = (int)(rows / 256);
    if (g.fb_in > 0 &&
        !encode4(&g.m_in4, q.ptr, 2 * L2, g.fb_in, items, 2 * L2, 2 * q.item_stride, 2 * TILE))
      return cudaErrorNotSupported;
    g.c_q = o.len / L2;
    g.c_rem = o.len - g.c_q * L2;
    return launch_t<PL, TILE, ST_C>(g, items, ncols, stream);
  }
  return cudaErrorNotSupported;
}
}  // namespace large

bool tma_col_len(long long L1) { return L1 == 1536 || L1 == 3072; }

// cudaErrorNotSupported unless the request is a 1D four-step column pass this
// kernel implements (L1 in {1536, 3072}, contiguous rows of length L2).
cudaError_t launch_cols_tma(int stage, const large::ColArgs &a, long long items, int ncols,
                            cudaStream_t stream) {
  using namespace large;
  if (getenv("HK_NO_COLTMA")) return cudaErrorNotSupported;
  if (!a.twiddle || items > 65535) return cudaErrorNotSupported;
  switch (a.L1) {
    case 1536: return launch_cols_tma_t<Plan1D<1536, 96, 6, 16, 16>, 4>(stage, a, items, ncols, stream);
    case 3072: return launch_cols_tma_t<Plan1D<3072, 192, 12, 16, 16>, 2>(stage, a, items, ncols, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace hk
