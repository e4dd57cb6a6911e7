// red_bw.cu -- L2 write-path throughput of the ways a GEMM-RS epilogue can push fp32
// partial tiles (the RS bound): TMA tensor reduce-add (the atomic mode), TMA
// tensor store (slots mode), red.global.add.v4.f32 and st.global.v4 from registers.
// 148 CTAs x 4 warps; each warp pushes 32 x 32 fp32 boxes (4 KB) round-robin over a target
// of `mb` MiB with `depth` bulk groups in flight.  Standalone (not part of the library):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/red_bw scripts/experiments/red_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int MODE>  // 0 TMA reduce-add, 1 TMA store, 2 red.v4, 3 st.v4
__global__ void __launch_bounds__(128, 1) push(const __grid_constant__ CUtensorMap map, float* dst, int rows, int cols,
                                              int iters, int depth) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* stg = reinterpret_cast<float4*>(base + warp * 8 * 4096);
  const int nbx = cols / 32, nby = rows / 32;
  const int gw = blockIdx.x * 4 + warp, nw = gridDim.x * 4;
  int b = 0;
  for (int it = 0; it < iters; ++it) {
    const int box = (gw + it * nw) % (nbx * nby);
    const int bx = box % nbx, by = box / nbx;
    if (MODE <= 1) {
      float4* s = stg + b * 256;
      if (lane == 0) {
        if (depth == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else if (depth == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else if (depth == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) s[lane * 8 + (j ^ (lane & 7))] = make_float4(1.f, 1.f, 1.f, 1.f);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (MODE == 0)
          asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];"
                       ::"l"(&map), "r"(smem_u32(s)), "r"(bx * 32), "r"(by * 32) : "memory");
        else
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];"
                       ::"l"(&map), "r"(smem_u32(s)), "r"(bx * 32), "r"(by * 32) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      b = (b + 1) % depth;
    } else {
      // lane l: rows i*4 + l/8, 16-byte column segment l%8 of the 128-byte box rows
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float* p = dst + int64_t(by * 32 + i * 4 + (lane >> 3)) * cols + bx * 32 + (lane & 7) * 4;
        if (MODE == 2)
          asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f),
                       "f"(1.f) : "memory");
        else
          asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                       : "memory");
      }
    }
  }
  if (MODE <= 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  PFN_encode enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  const int cols = 4096;
  const int mbs[] = {16, 64, 512};
  const char* names[] = {"tma_reduce_add", "tma_store", "red_v4", "st_v4"};
  for (int mb : mbs) {
    const int rows = int((int64_t(mb) << 20) / (cols * 4));
    float* dst;
    CK(cudaMalloc(&dst, size_t(rows) * cols * 4));
    CK(cudaMemset(dst, 0, size_t(rows) * cols * 4));
    CUtensorMap map;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    const int smem = 4 * 8 * 4096 + 1024;
    for (int mode = 0; mode < 4; ++mode) {
      for (int depth : {1, 2, 4, 8}) {
        if (mode >= 2 && depth > 1) continue;
        void (*k)(CUtensorMap, float*, int, int, int, int) =
            mode == 0 ? push<0> : mode == 1 ? push<1> : mode == 2 ? push<2> : push<3>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int iters = 2000;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k<<<sms, 128, smem>>>(map, dst, rows, cols, 50, depth);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k<<<sms, 128, smem>>>(map, dst, rows, cols, iters, depth);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = double(sms) * 4 * iters * 4096;
        printf("{\"target_mib\": %d, \"op\": \"%s\", \"depth\": %d, \"GBps\": %.1f}\n", mb, names[mode], depth,
               bytes / (ms * 1e-3) / 1e9);
      }
    }
    cudaFree(dst);
  }
  return 0;
}
