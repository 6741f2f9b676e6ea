// TMEM read vs shared-memory read throughput on B200, alone and together
// (does tcgen05.ld compete with LDS for the same per-SM bandwidth?), and
// whether DFMA chains slow down next to either stream.  One 512-thread CTA per
// SM (the cfg2 kernel's shape), bytes per SM clock reported.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench_tmem.cu -o tools/ubench_tmem
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// MODE 0: TMEM reads; 1: LDS.128 reads; 2: both in every warp; 3: half the
// warps each; 4: DFMA only; 5: DFMA + TMEM reads; 6: DFMA + LDS reads
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double *out, int iters) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 8192; i += 512) sm[i] = make_double2(i, -i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t taddr = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  const bool do_tm = MODE == 0 || MODE == 2 || MODE == 5 || (MODE == 3 && (warp & 1));
  const bool do_ld = MODE == 1 || MODE == 2 || MODE == 6 || (MODE == 3 && !(warp & 1));
  const bool do_fp = MODE >= 4;
  uint32_t acc = 0;
  double d0 = t, d1 = t + 1, d2 = t + 2, d3 = t + 3, s = 0;
  const double m = 1.0000001, c = 0.9999999;
  for (int it = 0; it < iters; ++it) {
    if (do_tm) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t r[16];
        ld16(taddr + 16 * q, r);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc ^= r[i];
      }
    }
    if (do_ld) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 v = sm[(t + 512 * q + it) & 8191];
        s += v.x - v.y;
      }
    }
    if (do_fp) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        d0 = fma(d0, m, c); d1 = fma(d1, c, m); d2 = fma(d2, m, c); d3 = fma(d3, c, m);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(slot));
  out[blockIdx.x * blockDim.x + t] = acc + s + d0 + d1 + d2 + d3;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  const int threads = 512, blocks = sms, iters = 20000, smem = 8192 * 16;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
  const char *names[] = {"TMEM ld", "LDS.128", "TMEM+LDS same warps", "TMEM/LDS split warps",
                         "DFMA only", "DFMA+TMEM ld", "DFMA+LDS.128"};
  void (*fns[])(double *, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [\n", sms, clk);
  for (int mode = 0; mode < 7; ++mode) {
    cudaFuncSetAttribute(fns[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      fns[mode]<<<blocks, threads, smem>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double cyc = ms * 1e-3 * clk * 1e3;
    const bool tm = mode == 0 || mode == 2 || mode == 5, ld = mode == 1 || mode == 2 || mode == 6;
    const double warps = (mode == 3) ? 8 : 16;
    const double tm_bytes = (tm || mode == 3) ? (double)iters * warps * 32 * 4 * 64 : 0;
    const double ld_bytes = (ld || mode == 3) ? (double)iters * warps * 32 * 16 * 16 : 0;
    const double fp = mode >= 4 ? (double)iters * 16 * 32 * 32 * 4 : 0;
    printf("  {\"mode\": \"%s\", \"ms\": %.3f, \"tmem_B_per_clk_sm\": %.1f, \"lds_B_per_clk_sm\": %.1f, "
           "\"dfma_lanes_per_clk_sm\": %.1f}%s\n",
           names[mode], ms, tm_bytes / cyc, ld_bytes / cyc, fp / cyc, mode < 6 ? "," : "");
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
  }
  printf("]}\n");
  return 0;
}
