// Can a cluster-4 persistent grid (132 CTAs, ~226 KB smem each) and a cluster-2 grid on the 16 SMs it
// leaves run at the same time?  Each CTA records its SM and start / end globaltimer; kernels spin ~2 ms.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(int* sm, unsigned long long* t0, unsigned long long* t1, int base) {
  if (threadIdx.x == 0) {
    int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    sm[base + blockIdx.x] = s;
    unsigned long long a = gt();
    t0[base + blockIdx.x] = a;
    while (gt() - a < 2000000ull) {}
    t1[base + blockIdx.x] = gt();
  }
  __syncthreads();
}
int launch(int cs, int grid, int base, cudaStream_t st, int* sm, unsigned long long* t0, unsigned long long* t1) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = 226 * 1024; cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, k, sm, t0, t1, base);
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  int* sm; unsigned long long *t0, *t1;
  cudaMallocManaged(&sm, 4 * 256); cudaMallocManaged(&t0, 8 * 256); cudaMallocManaged(&t1, 8 * 256);
  cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    int e1 = launch(4, 132, 0, a, sm, t0, t1);
    int e2 = launch(2, 16, 132, b, sm, t0, t1);
    cudaDeviceSynchronize();
    unsigned long long mn = ~0ull, mx4 = 0, mn2 = ~0ull, mx2 = 0;
    for (int i = 0; i < 148; ++i) mn = t0[i] < mn ? t0[i] : mn;
    for (int i = 0; i < 132; ++i) mx4 = t1[i] > mx4 ? t1[i] : mx4;
    for (int i = 132; i < 148; ++i) { mn2 = t0[i] < mn2 ? t0[i] : mn2; mx2 = t1[i] > mx2 ? t1[i] : mx2; }
    int used[256] = {0}, dup = 0;
    for (int i = 0; i < 148; ++i) { if (used[sm[i]]) ++dup; used[sm[i]] = 1; }
    printf("rep %d: err %d %d | cluster4 ends %.3f ms | cluster2 starts %.3f ends %.3f ms | SMs reused %d\n", rep,
           e1, e2, (mx4 - mn) / 1e6, (mn2 - mn) / 1e6, (mx2 - mn) / 1e6, dup);
    printf("  cluster2 SMs:");
    for (int i = 132; i < 148; ++i) printf(" %d", sm[i]);
    printf("\n");
  }
  return 0;
}
