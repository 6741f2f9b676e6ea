// Microbenchmark: shared-memory vs SHFL vs TMEM data movement throughput on
// one SM (and combined), to decide which exchange paths can run concurrently.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void k(double *out, int iters) {
  __shared__ double2 buf[2048];
  __shared__ uint32_t slot;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double2 acc = make_double2(t, 0);
  uint32_t taddr = 0;
  if (MODE >= 3) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    taddr = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  }
  for (int i = 0; i < 2048; i += blockDim.x) buf[(i + t) & 2047] = make_double2(i, t);
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {  // 16 x (STS.128 + LDS.128) per thread
#pragma unroll
      for (int j = 0; j < 16; ++j) buf[(t + j * 512 + it) & 2047] = acc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        double2 v = buf[(t + j * 512 + it + 1) & 2047];
        acc.x += v.x;
      }
    }
    if (MODE == 1 || MODE == 2) {  // 64 x SHFL.32 per thread (= 16 complex doubles)
      uint32_t r[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) r[j] = __double_as_longlong(acc.x) >> (j & 31);
#pragma unroll
      for (int j = 0; j < 64; ++j) r[j] = __shfl_xor_sync(0xffffffff, r[j], (j & 15) + 1);
      uint32_t s = 0;
#pragma unroll
      for (int j = 0; j < 64; ++j) s ^= r[j];
      acc.y += s;
    }
    if (MODE == 3 || MODE == 4) {  // 64 x 32-bit to TMEM and back per thread
      uint32_t r[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = (uint32_t)(acc.x + j + c);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     ::"r"(taddr + 16 * c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n");
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                     "tcgen05.wait::ld.sync.aligned;\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(taddr + 16 * c));
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += r[j];
        acc.y += s;
      }
    }
    if (MODE == 4) {  // + smem traffic concurrently
#pragma unroll
      for (int j = 0; j < 16; ++j) buf[(t + j * 512 + it) & 2047] = acc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        double2 v = buf[(t + j * 512 + it + 1) & 2047];
        acc.x += v.x;
      }
    }
  }
  out[blockIdx.x * blockDim.x + t] = acc.x + acc.y;
  if (MODE >= 3) {
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(slot));
  }
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 512 * sizeof(double));
  const int iters = 2000;
  const char *names[] = {"smem st+ld 512B/thr", "shfl 256B/thr", "smem+shfl", "tmem st+ld 512B/thr",
                         "tmem + smem"};
  for (int mode = 0; mode < 5; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<148, 512>>>(out, iters); break;
        case 1: k<1><<<148, 512>>>(out, iters); break;
        case 2: k<2><<<148, 512>>>(out, iters); break;
        case 3: k<3><<<148, 512>>>(out, iters); break;
        case 4: k<4><<<148, 512>>>(out, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cycles = ms * 1e-3 * clk * 1e3;
    // bytes per SM per iteration
    double smem_b = 512.0 * 16 * 16 * 2, shfl_b = 512.0 * 64 * 4, tmem_b = 512.0 * 64 * 4 * 2;
    double bytes = (mode == 0 ? smem_b : mode == 1 ? shfl_b : mode == 2 ? smem_b + shfl_b
                    : mode == 3 ? tmem_b : tmem_b + smem_b) * iters;
    printf("%-22s %8.3f ms  %7.1f B/clk/SM (at %d MHz max clock)  err=%s\n", names[mode], ms,
           bytes / cycles, clk / 1000, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
