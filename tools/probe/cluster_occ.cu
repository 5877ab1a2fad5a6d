// How many clusters of size 2 / 4 / 8 with one ~220 KB-smem CTA per SM can be co-resident
// (cudaOccupancyMaxActiveClusters), and which SMs a cluster-4 persistent grid actually lands on.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* sm) {
  if (threadIdx.x == 0) { int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); sm[blockIdx.x] = s; }
}
int main() {
  const int smem = 226 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
