// DRAM locality microbenchmark for the small-plane kernels: read 32 planes of 784 B per item,
// the planes (a) 32 batch samples of one channel (stride C * 784 B) or (b) contiguous.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/loc tools/locality_bench.cu && /tmp/loc
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ x, float* out, int items, int C, int mode) {
  float acc = 0.f;
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int it = warp; it < items; it += nw) {
    const int c = it % C, g = it / C;
    for (int j = 0; j < 32; ++j) {
      size_t plane = mode == 0 ? ((size_t)(32 * g + j) * C + c) : ((size_t)it * 32 + j);
      const float4* p = x + plane * 49;  // 784 B = 49 float4
      for (int u = lane; u < 49; u += 32) { float4 v = __ldcs(p + u); acc += v.x + v.y + v.z + v.w; }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  const int N = 128, C = 384; const size_t planes = (size_t)N * C; const size_t bytes = planes * 784;
  float4* x; float* o; cudaMalloc(&x, bytes); cudaMalloc(&o, 4); cudaMemset(x, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) for (int bpsm = 2; bpsm <= 16; bpsm *= 2) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); rd<<<148 * bpsm, 256>>>(x, o, (int)(planes / 32), C, mode); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("mode %s blocks/SM %2d: %.1f us, %.0f GB/s\n", mode ? "contiguous" : "stride C*784", bpsm, best * 1e3, bytes / best / 1e6);
  }
  return 0;
}
