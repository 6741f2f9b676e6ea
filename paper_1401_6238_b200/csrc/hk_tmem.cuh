// Tensor-memory (TMEM) staging for the fused product kernels.
//
// The spectral accumulator acc = ifft(h) .* fft(x_1)^p1 .* ... (reference
// hankel.py:61-71) is the one array that must survive while another full
// length-L transform runs.  Holding it in registers doubles the register
// footprint (1 CTA/SM, spills); holding it in shared memory doubles the smem
// footprint and competes with the transform's exchange traffic on the same
// 128 B/clk datapath.  On sm_100 each SM has 256 KB of TMEM next to the tensor
// cores; tcgen05.st/ld move a warp's registers to/from its 32-lane quarter of
// TMEM without touching the LSU/shared-memory path.  We use it as a per-thread
// spill slot: warp w owns lanes 32*(w%4)..+31 and a 2*V-column slab selected
// by w/4; each thread stores its V complex doubles (2*V x 32-bit columns).
#pragma once

#include <stdint.h>

#include "hk_dft.cuh"

namespace hk {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Allocate `cols` TMEM columns (power of two >= 32) for the CTA; warp `w0` does it.
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *slot_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(slot_smem)),
               "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}

template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(COLS));
}

__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }

// 4 complex doubles = 16 consecutive 32-bit columns of this thread's lane.
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const cplx *v) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[4 * i + 0] = (uint32_t)__double2loint(v[i].x);
    r[4 * i + 1] = (uint32_t)__double2hiint(v[i].x);
    r[4 * i + 2] = (uint32_t)__double2loint(v[i].y);
    r[4 * i + 3] = (uint32_t)__double2hiint(v[i].y);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}

// Load 4 complex doubles; the wait is inside the same asm block so the
// outputs are valid when it returns (no memory clobber: TMEM is not generic
// memory, and volatile asm keeps program order among TMEM operations).
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, cplx *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i].x = __hiloint2double((int)r[4 * i + 1], (int)r[4 * i + 0]);
    v[i].y = __hiloint2double((int)r[4 * i + 3], (int)r[4 * i + 2]);
  }
}

// Load 8 complex doubles (32 columns) with one wait.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, cplx *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i].x = __hiloint2double((int)r[4 * i + 1], (int)r[4 * i + 0]);
    v[i].y = __hiloint2double((int)r[4 * i + 3], (int)r[4 * i + 2]);
  }
}

}  // namespace hk

namespace hk {

// 4 complex floats = 8 consecutive 32-bit columns (complex64 variant).
__device__ __forceinline__ void tmem_st4f(uint32_t taddr, const float2 *v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::
                   "r"(taddr),
               "r"(__float_as_uint(v[0].x)), "r"(__float_as_uint(v[0].y)),
               "r"(__float_as_uint(v[1].x)), "r"(__float_as_uint(v[1].y)),
               "r"(__float_as_uint(v[2].x)), "r"(__float_as_uint(v[2].y)),
               "r"(__float_as_uint(v[3].x)), "r"(__float_as_uint(v[3].y)));
}

__device__ __forceinline__ void tmem_ld4f(uint32_t taddr, float2 *v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
}

}  // namespace hk
