// FP64 peaks on B200: DFMA (FP64 pipe), DMMA (mma.sync m8n8k4 f64, the
// tensor-core FP64 path) and both issued together in one kernel -- do the two
// pipes add up?  Every number is FP64 flops per second (FMA = 2 flops,
// one m8n8k4 DMMA = 2*8*8*4 = 512 flops per warp).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench_fp64.cu -o tools/ubench_fp64
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// MODE 0: DFMA only; 1: DMMA only; 2: half the warps DFMA, half DMMA;
// 3: every warp interleaves DFMA chains with DMMA; 4: DADD only
template <int MODE>
__global__ void k(double *out, int iters) {
  const int t = threadIdx.x, warp = t >> 5;
  double a0 = t, a1 = t + 1, a2 = t + 2, a3 = t + 3, a4 = t + 4, a5 = t + 5, a6 = t + 6,
         a7 = t + 7;
  const double m = 1.0000001, c = 0.9999999;
  double d0[2] = {0, 0}, d1[2] = {0, 0}, d2[2] = {0, 0}, d3[2] = {0, 0};
  double ea = 1.0 + t * 1e-9, eb = 1.0 - t * 1e-9;
  const bool do_fp = MODE == 0 || MODE == 3 || MODE == 4 || (MODE == 2 && (warp & 1) == 0);
  const bool do_mm = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (do_fp) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // 8 independent chains
        if (MODE == 4) {
          a0 += c; a1 += m; a2 += c; a3 += m; a4 += c; a5 += m; a6 += c; a7 += m;
        } else {
          a0 = fma(a0, m, c); a1 = fma(a1, c, m); a2 = fma(a2, m, c); a3 = fma(a3, c, m);
          a4 = fma(a4, m, c); a5 = fma(a5, c, m); a6 = fma(a6, m, c); a7 = fma(a7, c, m);
        }
      }
    }
    if (do_mm) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // 4 independent accumulators
        dmma(d0, ea, eb);
        dmma(d1, eb, ea);
        dmma(d2, ea, eb);
        dmma(d3, eb, ea);
      }
    }
  }
  out[blockIdx.x * blockDim.x + t] =
      a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + d0[0] + d1[1] + d2[0] + d3[1];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  const int threads = 512, blocks = sms * 2, iters = 20000;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
  const char *names[] = {"DFMA only", "DMMA only", "half warps DFMA / half DMMA",
                         "DFMA + DMMA in every warp", "DADD only"};
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [\n", sms, clk);
  for (int mode = 0; mode < 5; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<blocks, threads>>>(out, iters); break;
        case 1: k<1><<<blocks, threads>>>(out, iters); break;
        case 2: k<2><<<blocks, threads>>>(out, iters); break;
        case 3: k<3><<<blocks, threads>>>(out, iters); break;
        case 4: k<4><<<blocks, threads>>>(out, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double warps = (double)blocks * threads / 32;
    const double fp_warps = mode == 0 || mode == 3 || mode == 4 ? warps : mode == 2 ? warps / 2 : 0;
    const double mm_warps = mode == 1 || mode == 3 ? warps : mode == 2 ? warps / 2 : 0;
    const double fp_flops = fp_warps * 32 * (double)iters * 16 * 8 * (mode == 4 ? 1 : 2);
    const double mm_flops = mm_warps * (double)iters * 8 * 4 * 512;
    const double tf = (fp_flops + mm_flops) / (ms * 1e-3) / 1e12;
    const double lanes = fp_flops / (mode == 4 ? 1 : 2) / (ms * 1e-3) / (sms * clk * 1e3);
    printf("  {\"mode\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f, \"dfma_tflops\": %.2f, "
           "\"dmma_tflops\": %.2f, \"fp64_lane_ops_per_clk_per_sm\": %.1f}%s\n",
           names[mode], ms, tf, fp_flops / (ms * 1e-3) / 1e12, mm_flops / (ms * 1e-3) / 1e12,
           lanes, mode < 4 ? "," : "");
  }
  printf("]}\n");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
