// Probe: a 148-CTA launch (one CTA per SM by shared memory) with regular cluster dim 2 and
// preferred cluster dim 4 -- which CTAs form 4-CTA clusters, are all co-resident, and does a
// dynamic per-cluster claim counter see every cluster.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned arrived;
__global__ void probe(int* out, unsigned long long timeout) {
  extern __shared__ unsigned char sm[];
  unsigned nct, cid, crk, smid;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nct));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crk));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  int ok = 1;
  if (threadIdx.x == 0) {
    sm[0] = 1;
    atomicAdd(&arrived, 1u);
    unsigned long long t0 = clock64();
    while (atomicAdd(&arrived, 0u) < gridDim.x) {
      if (clock64() - t0 > timeout) { ok = 0; break; }
    }
    out[blockIdx.x * 5 + 0] = nct;
    out[blockIdx.x * 5 + 1] = cid;
    out[blockIdx.x * 5 + 2] = crk;
    out[blockIdx.x * 5 + 3] = smid;
    out[blockIdx.x * 5 + 4] = ok;
  }
}
int main() {
  int* d; cudaMalloc(&d, 148 * 5 * 4 * 2);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 4; ++rep) {
    unsigned z = 0; cudaMemcpyToSymbol(arrived, &z, 4);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributePreferredClusterDimension; a[1].val.preferredClusterDim.x = 4; a[1].val.preferredClusterDim.y = 1; a[1].val.preferredClusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d, 2000000000ull);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[148 * 5]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int n4 = 0, n2 = 0, bad = 0;
    for (int b = 0; b < 148; ++b) { if (h[b*5] == 4) ++n4; else if (h[b*5] == 2) ++n2; if (!h[b*5+4]) ++bad; }
    printf("rep %d launch %s sync %s: CTAs in 4-clusters %d, in 2-clusters %d, not co-resident %d\n", rep,
           cudaGetErrorString(e), cudaGetErrorString(e2), n4, n2, bad);
    if (rep == 0)
      for (int b = 0; b < 148; ++b) printf("  blk %3d nct %d cid %3d crk %d sm %3d\n", b, h[b*5], h[b*5+1], h[b*5+2], h[b*5+3]);
  }
  return 0;
}
