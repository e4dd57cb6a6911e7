// Loopback "copy engine" probe: does a same-device cudaMemcpyAsync D2D run on the copy
// engines (DMA) or as an SM copy kernel, and does it slow a concurrent pinned H2D copy?
// (a) a 64 MB D2D copy while a blocker kernel holds every SM's thread slots for 30 ms: a copy
// that finishes long before the blocker did not need SMs; (b) H2D 64 MB alone vs concurrent
// with 8 x 64 MB of D2D copies on another stream.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024) blocker(unsigned long long ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < ns);
}
int main() {
  const size_t N = 64ull << 20;
  char *a, *b, *h;
  cudaMalloc(&a, N); cudaMalloc(&b, 8 * N);
  cudaMallocHost(&h, N);
  cudaMemset(a, 1, N);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, k0, k1;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&k0); cudaEventCreate(&k1);
  // graph memcpy node (how the loopback copy-engine chains are replayed)
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaGraphCreate(&g, 0);
  cudaGraphNode_t nd;
  cudaGraphAddMemcpyNode1D(&nd, g, nullptr, 0, b, a, N, cudaMemcpyDeviceToDevice);
  cudaGraphInstantiate(&ge, g, 0);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(k0, s1);
    blocker<<<148 * 2, 1024, 0, s1>>>(30000000ull);
    cudaEventRecord(k1, s1);
    cudaStreamWaitEvent(s0, k0, 0);
    cudaEventRecord(e0, s0);
    cudaGraphLaunch(ge, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float cms, kms;
    cudaEventElapsedTime(&cms, e0, e1);
    cudaEventElapsedTime(&kms, k0, k1);
    printf("graph D2D node 64 MB under an SM blocker: copy %.2f ms, blocker %.2f ms -> %s\n", cms, kms,
           cms < 0.5 * kms ? "copy engine" : "waited for SMs (SM copy kernel)");
    // H2D beside graph D2D copies
    cudaEventRecord(e0, s0);
    cudaMemcpyAsync(a, h, N, cudaMemcpyHostToDevice, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float h1;
    cudaEventElapsedTime(&h1, e0, e1);
    for (int i = 0; i < 8; ++i) cudaGraphLaunch(ge, s1);
    cudaEventRecord(e0, s0);
    cudaMemcpyAsync(a, h, N, cudaMemcpyHostToDevice, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float h2;
    cudaEventElapsedTime(&h2, e0, e1);
    printf("H2D 64 MB: alone %.3f ms, beside graph D2D copies %.3f ms\n", h1, h2);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(k0, s1);
    blocker<<<148 * 2, 1024, 0, s1>>>(30000000ull);
    cudaEventRecord(k1, s1);
    cudaStreamWaitEvent(s0, k0, 0);
    cudaEventRecord(e0, s0);
    cudaMemcpyAsync(b, a, N, cudaMemcpyDeviceToDevice, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float cms, kms; cudaEventElapsedTime(&cms, e0, e1); cudaEventElapsedTime(&kms, k0, k1);
    printf("D2D 64 MB under an SM blocker: copy %.2f ms, blocker %.2f ms -> %s\n", cms, kms,
           cms < 0.5 * kms ? "copy engine" : "waited for SMs (SM copy kernel)");
    // H2D alone
    cudaEventRecord(e0, s0);
    cudaMemcpyAsync(a, h, N, cudaMemcpyHostToDevice, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float h1; cudaEventElapsedTime(&h1, e0, e1);
    // H2D while D2D copies run on s1
    for (int i = 0; i < 8; ++i) cudaMemcpyAsync(b + i * N, a, N, cudaMemcpyDeviceToDevice, s1);
    cudaEventRecord(e0, s0);
    cudaMemcpyAsync(a, h, N, cudaMemcpyHostToDevice, s0);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float h2; cudaEventElapsedTime(&h2, e0, e1);
    printf("H2D 64 MB: alone %.3f ms (%.1f GB/s), beside D2D copies %.3f ms (%.1f GB/s)\n", h1, N / (h1 * 1e6), h2,
           N / (h2 * 1e6));
  }
  return 0;
}
