// Microbenchmark: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int MODE>
__global__ void k(float* out, float x, float y, int iters) {
  float a[16];
  unsigned long long p[8];
  for (int i = 0; i < 16; ++i) a[i] = x + i + threadIdx.x;
  for (int i = 0; i < 8; ++i) p[i] = __double_as_longlong((double)(x + i));
  const unsigned long long yy = __double_as_longlong((double)y);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], y, a[(i + 1) & 15]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], yy, p[(i + 1) & 7]);
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  for (int i = 0; i < 8; ++i) s += (float)__longlong_as_double(p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (mode == 0) k<0><<<148 * 8, 256>>>(out, 1.f, 0.999f, iters); else k<1><<<148 * 8, 256>>>(out, 1.f, 0.999f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = 148.0 * 8 * 256 * (double)iters * 16;
    printf("%s: %.3f ms, %.1f TFLOP/s fp32\n", mode ? "FFMA2" : "FFMA ", ms, 2 * fmas / ms / 1e9);
  }
  return 0;
}
