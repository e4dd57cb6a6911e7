// Calibration of the in-kernel clock measurement (TR_CLK trace events): one CTA spins for
// ~2 ms and reports clock64 cycles / %globaltimer ns, on an otherwise idle GPU -- the SM
// clock with no power pressure (expect ~sm_max_mhz) -- then the same while a 147-CTA FMA
// kernel loads every other SM.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(double* out, unsigned long long ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < ns);
  long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = double(c1 - c0) / double(t1 - t0) * 1e3;  // MHz
}
__global__ void burn(float* sink, int iters) {
  float a = threadIdx.x, b = 1.0001f, c = 0.9999f, d = blockIdx.x;
  for (int i = 0; i < iters; ++i) { a = fmaf(a, b, c); d = fmaf(d, c, b); }
  if (a + d == 12345.f) sink[0] = a;
}
int main() {
  double* d; cudaMalloc(&d, 8 * 148); float* s; cudaMalloc(&s, 4);
  double h[148];
  for (int rep = 0; rep < 3; ++rep) {
    spin<<<1, 32>>>(d, 2000000ull); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("idle GPU, 1 CTA: clock64 rate %.0f MHz\n", h[0]);
  }
  cudaStream_t a, b; cudaStreamCreate(&a); cudaStreamCreate(&b);
  burn<<<147 * 4, 1024, 0, a>>>(s, 2000000);
  spin<<<1, 32, 0, b>>>(d, 2000000ull);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("with an FMA load on the other SMs: clock64 rate %.0f MHz (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
