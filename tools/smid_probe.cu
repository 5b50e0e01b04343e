// Probe the SM id layout: %smid / %nsmid per CTA, and GPC grouping via clusters of 16 (non-portable).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <set>
#include <vector>
#include <map>
#include <algorithm>
__global__ void probe(int* out) {
  unsigned s, n; asm("mov.u32 %0, %%smid;" : "=r"(s)); asm("mov.u32 %0, %%nsmid;" : "=r"(n));
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = s; out[2 * blockIdx.x + 1] = n; }
}
__global__ void __cluster_dims__(1, 1, 1) dummy() {}
__global__ void cprobe(int* out) {
  unsigned s; asm("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}
int main() {
  int* d; cudaMalloc(&d, 1 << 20);
  int nb = 148 * 4;
  probe<<<nb, 32>>>(d);
  std::vector<int> h(2 * nb); cudaMemcpy(h.data(), d, 8 * nb, cudaMemcpyDeviceToHost);
  std::set<int> ids; for (int i = 0; i < nb; ++i) ids.insert(h[2 * i]);
  printf("nsmid %d distinct smids %zu min %d max %d\n", h[1], ids.size(), *ids.begin(), *ids.rbegin());
  for (int cs : {16, 8}) {
    cudaFuncSetAttribute(cprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int ncl = 64; cfg.gridDim = dim3(cs * ncl); cfg.blockDim = dim3(32);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, cprobe, d);
    cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cluster %d: %s\n", cs, cudaGetErrorString(e)); continue; }
    std::vector<int> c(cs * ncl); cudaMemcpy(c.data(), d, 4 * cs * ncl, cudaMemcpyDeviceToHost);
    std::set<std::vector<int>> groups;
    for (int k = 0; k < ncl; ++k) { std::vector<int> g(c.begin() + k * cs, c.begin() + (k + 1) * cs); std::sort(g.begin(), g.end()); groups.insert(g); }
    printf("cluster size %d: %zu distinct groups\n", cs, groups.size());
    for (auto& g : groups) { for (int x : g) printf("%d ", x); printf("\n"); }
  }
  return 0;
}
