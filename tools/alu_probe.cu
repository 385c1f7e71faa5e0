// Throughput probe: FMNMX3 (3-input max) vs FMNMX vs FFMA2 vs F2FP on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ float max3(float a, float b, float c) { float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float max2(float a, float b) { float r; asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
template <int MODE> __global__ void k(float* out, int iters) {
  float a[8], b = threadIdx.x * 1e-3f, c = b * 0.5f;
  for (int i = 0; i < 8; ++i) a[i] = i * 1e-4f * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = max3(a[i], b, c);
      if (MODE == 1) a[i] = max2(a[i], b);
      if (MODE == 2) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(b)); a[i] = __uint_as_float(r) ; }
      if (MODE == 3) a[i] = fmaf(a[i], 1.0001f, b);
    }
    b += 1e-7f; c -= 1e-7f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4); int iters = 8192, blocks = 148 * 4, thr = 512;
  const char* names[4] = {"FMNMX3 (max3)", "FMNMX (max2)", "F2FP bf16x2", "FFMA"};
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int m = 0; m < 4; ++m) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<blocks, thr>>>(o, iters); if (m == 1) k<1><<<blocks, thr>>>(o, iters);
      if (m == 2) k<2><<<blocks, thr>>>(o, iters); if (m == 3) k<3><<<blocks, thr>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = double(blocks) * thr * iters * 8;  // thread-ops
    printf("%-16s %.3f ms  %.1f thread-ops/clk/SM\n", names[m], ms, n / (ms * 1e-3) / 148 / (clk * 1e3));
  }
}
