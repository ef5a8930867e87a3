// Feasibility probe: preferred cluster dimension 4 with a minimum of 2 — how
// many 4-CTA and 2-CTA clusters does a 148-CTA persistent grid get?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(int *out) {
  unsigned n, cid, smid;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) {
    out[blockIdx.x * 3 + 0] = n;
    out[blockIdx.x * 3 + 1] = cid;
    out[blockIdx.x * 3 + 2] = smid;
  }
  // keep the CTA resident long enough that all are co-resident
  long long t0 = clock64();
  while (clock64() - t0 < 20000000) {}
}

int main() {
  int *d;
  const int G = 148;
  cudaMalloc(&d, G * 3 * sizeof(int));
  cudaMemset(d, 0xff, G * 3 * sizeof(int));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributePreferredClusterDimension;
  attr[1].val.preferredClusterDim.x = 4; attr[1].val.preferredClusterDim.y = 1;
  attr[1].val.preferredClusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  int h[G * 3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int c4 = 0, c2 = 0, other = 0;
  for (int i = 0; i < G; ++i) {
    if (h[i * 3] == 4) ++c4; else if (h[i * 3] == 2) ++c2; else ++other;
  }
  printf("CTAs in 4-clusters: %d, in 2-clusters: %d, other: %d\n", c4, c2, other);
  for (int i = 0; i < G; i += 1) printf("%d:%d/%d/sm%d ", i, h[i * 3], h[i * 3 + 1], h[i * 3 + 2]);
  printf("\n");
  return 0;
}
