// Preferred-cluster semantics probe: launch 148 CTAs (1 per SM, big smem)
// with clusterDim 2 and preferredClusterDim 4; record per CTA the actual
// cluster size / rank / id, blockIdx and SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int *out) {
  extern __shared__ char smem[];
  unsigned nct, rk, cid, ncid, smid, cidy;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nct));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rk));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm volatile("mov.u32 %0, %%clusterid.y;" : "=r"(cidy));
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(ncid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) {
    int *o = out + blockIdx.x * 6;
    o[0] = nct; o[1] = rk; o[2] = cid; o[3] = ncid; o[4] = smid; o[5] = cidy;
  }
  smem[threadIdx.x] = 0;
  // keep the CTA resident a while so all 148 coexist
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
}
int main() {
  int *d; cudaMalloc(&d, 4096 * 6 * 4);
  int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int grid : {148, 296}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributePreferredClusterDimension; at[1].val.preferredClusterDim.x = 4; at[1].val.preferredClusterDim.y = 1; at[1].val.preferredClusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
    printf("grid %d launch: %s\n", grid, cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    static int h[4096 * 6];
    cudaMemcpy(h, d, grid * 6 * 4, cudaMemcpyDeviceToHost);
    int n4 = 0, n2 = 0;
    for (int b = 0; b < grid; ++b) { if (h[b*6] == 4) ++n4; else if (h[b*6] == 2) ++n2; }
    printf("CTAs in 4-clusters %d, in 2-clusters %d\n", n4, n2);
    for (int b = 0; b < grid; ++b)
      printf("blk %3d nct %d rank %d cid %3d ncid %3d cidy %d sm %3d\n", b, h[b*6], h[b*6+1], h[b*6+2], h[b*6+3], h[b*6+5], h[b*6+4]);
  }
  int n = 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(296); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
  printf("max active 4-clusters %d\n", n);
  at[0].val.clusterDim.x = 2;
  cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
  printf("max active 2-clusters %d\n", n);
  return 0;
}
