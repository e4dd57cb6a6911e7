// TMEM port contention microbenchmark (the SP-attention bound hypothesis): cycles
// per tcgen05.ld (32x32b.x32) + wait::ld, and per tcgen05.st + wait::st, issued by 4 warps
// (one per TMEM lane quadrant) of every SM, (0) alone and (1) while warp 0 keeps the tensor
// core busy with back-to-back 128x256x16 bf16 MMAs accumulating into other TMEM columns, and
// (2) the same with 128x128 MMAs (the attention tiles' shape).  148 CTAs, one per SM.
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2601_20595_b200/csrc -I include
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace ao::dev;

__global__ void __launch_bounds__(256, 1) probe(int mode, int iters, unsigned long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;               // 128 x 64 bf16, SW128
  uint8_t* sB = sm + 16384;       // 256 x 64 bf16, SW128
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile int* stop = reinterpret_cast<volatile int*>(slot + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);  // finite bf16
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    *stop = 0;
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
  if (warp == 0) {
    if (mode > 0 && lane == 0) {
      const int N = mode == 1 ? 256 : 128;
      const uint32_t idesc = make_idesc_bf16(128, N);
      const uint64_t ad = make_smem_desc_sw128(smem_u32(sA)), bd = make_smem_desc_sw128(smem_u32(sB));
      uint32_t ph = 0;
      for (int it = 0; !*stop; ++it) {
        for (int k = 0; k < 16; ++k) mma_bf16_ss(tmem + 256, ad + uint64_t((k & 3) * 2), bd + uint64_t((k & 3) * 2), idesc, 1u);
        mma_commit(&bar[0]);
        mbar_wait(&bar[0], ph);
        ph ^= 1;
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = uint32_t(warp & 3);
    const uint32_t ta = tmem + (q * 32u << 16);
    uint32_t v[32];
    unsigned long long t_ld = 0, t_st = 0;
    for (int it = 0; it < iters; ++it) {
      long long c0 = clock64();
      tmem_ld_32x32b_x32(ta + uint32_t(it & 3) * 32, v);
      tmem_wait_ld();
      long long c1 = clock64();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += 1u;
      long long c2 = clock64();
      tmem_st_32x32b_x32(ta + 128 + uint32_t(it & 3) * 32, v);
      tmem_wait_st();
      long long c3 = clock64();
      t_ld += c1 - c0;
      t_st += c3 - c2;
    }
    if (lane == 0) {
      atomicAdd(&out[0], t_ld);
      atomicAdd(&out[1], t_st);
      atomicAdd(&out[2], (unsigned long long)iters);
    }
    asm volatile("bar.sync 1, 128;");
    if (warp == 4 && lane == 0) *stop = 1;
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
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  const int smem = 16384 + 32768 + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"no MMA", "MMA 128x256x16 back to back", "MMA 128x128x16 back to back"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(d, 0, 3 * sizeof(unsigned long long));
      probe<<<148, 256, smem>>>(mode, 20000, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[3];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      printf("%-30s tcgen05.ld x32 + wait: %7.1f cycles   tcgen05.st x32 + wait: %7.1f cycles  (%s)\n", names[mode],
             double(h[0]) / h[2], double(h[1]) / h[2], cudaGetErrorString(e));
    }
  return 0;
}
