// tcgen05.mma issue-rate microbenchmark: cycles per MMA instruction, back to back with one
// commit per 16 MMAs and one batch always in flight, one CTA per SM (148), for the shapes the kernels use:
// SS 128x256x16 (1-CTA GEMM tile), SS 128x128x16 (attention S = Q K^T), TS 128x128x16 with A
// from TMEM (attention PV = P V), and SS 128x128x16 with B MN-major (V as stored).  Ideal at
// 8192 dense bf16 flop/clk/SM: 128x256x16 -> 128 cycles, 128x128x16 -> 64 cycles.
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2601_20595_b200/csrc -I include
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace ao::dev;

template <int MODE>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* out) {
  constexpr int mode = MODE;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;          // 128 x 64 bf16, SW128
  uint8_t* sB = sm + 16384;  // 256 x 64 bf16, SW128
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0 && lane == 0) {
    const uint64_t ad = make_smem_desc_sw128(smem_u32(sA)), bd = make_smem_desc_sw128(smem_u32(sB));
    const uint64_t bmn = make_smem_desc_sw128_mn(smem_u32(sB), 16384);
    const uint32_t id256 = make_idesc_bf16(128, 256), id128 = make_idesc_bf16(128, 128),
                   id128mn = make_idesc_bf16_bmn(128, 128);
    uint32_t ph[2] = {0, 0};
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if constexpr (mode == 0) mma_bf16_ss(tmem + 256, ad + uint64_t((k & 3) * 2), bd + uint64_t((k & 3) * 2), id256, 1u);
        else if constexpr (mode == 1) mma_bf16_ss(tmem + 256, ad + uint64_t((k & 3) * 2), bd + uint64_t((k & 3) * 2), id128, 1u);
        else if constexpr (mode == 2) mma_bf16_ts(tmem + 256, tmem + uint32_t((k & 7) * 8), bmn + uint64_t((k & 7) * 128), id128mn, 1u);
        else mma_bf16_ss(tmem + 256, ad + uint64_t((k & 3) * 2), bmn + uint64_t((k & 7) * 128), id128mn, 1u);
      }
      mma_commit(&bar[it & 1]);
      if (it > 0) {  // keep one batch in flight: wait for the previous batch only
        mbar_wait(&bar[(it - 1) & 1], ph[(it - 1) & 1]);
        ph[(it - 1) & 1] ^= 1;
      }
    }
    mbar_wait(&bar[(iters - 1) & 1], ph[(iters - 1) & 1]);
    long long c1 = clock64();
    atomicAdd(&out[0], (unsigned long long)(c1 - c0));
    atomicAdd(&out[1], (unsigned long long)iters * 16);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2 * sizeof(unsigned long long));
  const int smem = 16384 + 32768 + 1024 + 64;
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"SS 128x256x16", "SS 128x128x16", "TS 128x128x16 (A in TMEM, B MN-major)",
                          "SS 128x128x16 (B MN-major)"};
  const double ideal[4] = {128, 64, 64, 64};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      cudaMemset(d, 0, 2 * sizeof(unsigned long long));
      if (mode == 0) rate<0><<<148, 128, smem>>>(4000, d);
      if (mode == 1) rate<1><<<148, 128, smem>>>(4000, d);
      if (mode == 2) rate<2><<<148, 128, smem>>>(4000, d);
      if (mode == 3) rate<3><<<148, 128, smem>>>(4000, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      const double cyc = double(h[0]) / 148.0 / (double(h[1]) / 148.0);
      printf("%-40s %7.1f cycles per MMA (ideal %3.0f: %.0f %% of peak rate)  %s\n", names[mode], cyc, ideal[mode],
             100.0 * ideal[mode] / cyc, cudaGetErrorString(e));
    }
  return 0;
}
