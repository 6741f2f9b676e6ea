// Do FP64 math (warps 0..W/2-1) and shared-memory traffic (other warps)
// overlap on one SM?  Compare each alone with both together.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: fp64 only, 1: smem only, 2: both (split warps), 3: both in every warp
__global__ void k(double *out, int iters) {
  __shared__ double2 buf[2048];
  const int t = threadIdx.x, warp = t >> 5;
  double a0 = t, a1 = t + 1, a2 = t + 2, a3 = t + 3, a4 = 1.0000001, a5 = 0.9999999;
  double2 acc = make_double2(t, 0);
  for (int i = 0; i < 2048; i += blockDim.x) buf[(i + t) & 2047] = make_double2(i, t);
  __syncthreads();
  const bool do_fp = MODE == 0 || MODE == 3 || (MODE == 2 && warp < (int)(blockDim.x >> 6));
  const bool do_sm = MODE == 1 || MODE == 3 || (MODE == 2 && warp >= (int)(blockDim.x >> 6));
  for (int it = 0; it < iters; ++it) {
    if (do_fp) {
#pragma unroll 16
      for (int j = 0; j < 64; ++j) {  // 4 independent DFMA chains
        a0 = fma(a0, a4, a5);
        a1 = fma(a1, a5, a4);
        a2 = fma(a2, a4, a5);
        a3 = fma(a3, a5, a4);
      }
    }
    if (do_sm) {
#pragma unroll
      for (int j = 0; j < 4; ++j) buf[(t + j * 512 + it) & 2047] = acc;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 v = buf[(t + j * 512 + it + 1) & 2047];
        acc.x += v.x;
      }
    }
  }
  out[blockIdx.x * blockDim.x + t] = a0 + a1 + a2 + a3 + acc.x;
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  const char *names[] = {"fp64 only (all warps)", "smem only (all warps)", "half fp64 / half smem",
                         "fp64+smem in every warp"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<148, 512>>>(out, 4000); break;
        case 1: k<1><<<148, 512>>>(out, 4000); break;
        case 2: k<2><<<148, 512>>>(out, 4000); break;
        case 3: k<3><<<148, 512>>>(out, 4000); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("%-26s %8.3f ms\n", names[mode], ms);
  }
  return 0;
}
