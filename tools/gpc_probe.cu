// Recover the GPC partition of SM ids: CTAs of one thread-block cluster always share a GPC,
// so union-find over the %smid sets of many clusters gives the GPCs.
#include <algorithm>
#include <cstdio>
#include <map>
#include <numeric>
#include <vector>
#include <cuda_runtime.h>
__global__ void cprobe(int* out) {
  unsigned s; asm("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = s;
  // keep the CTA alive a little so clusters spread over the GPU
  long long t0 = clock64(); while (clock64() - t0 < 20000) {}
}
int find(std::vector<int>& p, int x) { while (p[x] != x) x = p[x] = p[p[x]]; return x; }
int main() {
  int* d; cudaMalloc(&d, 1 << 20);
  std::vector<int> par(256); std::iota(par.begin(), par.end(), 0);
  std::vector<int> seen(256, 0);
  cudaFuncSetAttribute(cprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) for (int rep = 0; rep < 40; ++rep) {
    cudaLaunchConfig_t cfg = {};
    int ncl = 148 / cs + rep % 7; cfg.gridDim = dim3(cs * ncl); cfg.blockDim = dim3(32);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, cprobe, d) != cudaSuccess) { printf("launch failed\n"); return 1; }
    cudaDeviceSynchronize();
    std::vector<int> c(cs * ncl); cudaMemcpy(c.data(), d, 4 * cs * ncl, cudaMemcpyDeviceToHost);
    for (int k = 0; k < ncl; ++k)
      for (int j = 0; j < cs; ++j) {
        seen[c[k * cs + j]] = 1;
        par[find(par, c[k * cs + j])] = find(par, c[k * cs]);
      }
  }
  std::map<int, std::vector<int>> comp;
  for (int s = 0; s < 256; ++s) if (seen[s]) comp[find(par, s)].push_back(s);
  printf("%zu GPC components\n", comp.size());
  for (auto& kv : comp) { printf("[%zu]", kv.second.size()); for (int x : kv.second) printf(" %d", x); printf("\n"); }
  return 0;
}
