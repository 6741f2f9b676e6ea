// Does an FFT-shaped instruction mix overlap FP64 arithmetic with shared-memory
// exchange traffic on one SM?  Each warp repeats: 16 x LDS.128 (volatile asm),
// a radix-16-sized block of dependent-but-parallel DADD/DFMA on the 32 loaded
// doubles, 16 x STS.128, and (optionally) a named barrier per 256-thread group.
// Modes: 0 = FP64 block only, 1 = smem only, 2 = both, 3 = both + barrier.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double *out, const double2 *__restrict__ tw, int iters) {
  extern __shared__ __align__(16) double2 buf[];  // 2 x 4096 complex
  const int t = threadIdx.x, g = t >> 8, tg = t & 255;
  const uint32_t base = smem_u32(buf + g * 4096);
  double v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = 1.0 + 1e-9 * (t + j);
  for (int i = t; i < 8192; i += 512) buf[i] = make_double2(i, -i);
  __syncthreads();
  const double c1 = 0.9238795325112867, c2 = 0.3826834323650898;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t a = base + 16u * (uint32_t)((tg * 16 + ((j + tg) & 15)) & 4095);
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2 * j]), "=d"(v[2 * j + 1]) : "r"(a));
      }
    }
    if (MODE != 1) {
      // ~200 FP64 ops: 4 butterfly stages of 32 DADDs + 2 rounds of 16 DFMA
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int h = 1 << s;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if ((j & (2 * h)) == 0) {
            const double a = v[j], b = v[j + 2 * h < 32 ? j + 2 * h : j];
            v[j] = a + b;
            if (j + 2 * h < 32) v[j + 2 * h] = a - b;
          }
#pragma unroll
        for (int j = 0; j < 32; j += 4) v[j + 1] = fma(v[j + 1], c1, v[j + 3] * c2);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = fma(v[j], c1, c2 * v[(j + 5) & 31]);
      if (MODE == 4) {  // 15 twiddle multiplies with L1-resident table loads
#pragma unroll
        for (int j = 1; j < 16; ++j) {
          const double2 w = __ldg(&tw[(j * (tg >> 4)) & 255]);
          const double re = v[2 * j], im = v[2 * j + 1];
          v[2 * j] = fma(re, w.x, -im * w.y);
          v[2 * j + 1] = fma(re, w.y, im * w.x);
        }
      }
    }
    if (MODE != 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t a = base + 16u * (uint32_t)((tg + 256 * j) & 4095);
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v[2 * j]), "d"(v[2 * j + 1]) : "memory");
      }
    }
    if (MODE >= 3) {
      if (g == 0) asm volatile("bar.sync 1, 256;" ::: "memory");
      else asm volatile("bar.sync 2, 256;" ::: "memory");
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + t] = s;
}

template <int MODE>
float run(double *out, const double2 *tw, int iters) {
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<MODE><<<148, 512, 131072>>>(out, tw, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  return ms;
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 512 * sizeof(double));
  const int iters = 4000;
  double2 *tw;
  cudaMalloc(&tw, 256 * sizeof(double2));
  cudaMemset(tw, 0, 256 * sizeof(double2));
  const float f = run<0>(out, tw, iters), m = run<1>(out, tw, iters), both = run<2>(out, tw, iters),
              bar = run<3>(out, tw, iters), twl = run<4>(out, tw, iters);
  printf("fp64 block only     %.3f ms\n", f);
  printf("smem 16ld+16st only %.3f ms\n", m);
  printf("both                %.3f ms  (sum %.3f, max %.3f)\n", both, f + m, f > m ? f : m);
  printf("both + group bar    %.3f ms\n", bar);
  printf("+ 15 twiddle cmul   %.3f ms  err=%s\n", twl, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
