// e4.cu -- transfer-backend microbenchmark kernel (SURVEY.md §8(d) "E4": peer-copy
// bandwidth vs message size and #SMs per backend, Fig.2c,d; Tab.2).
// n_ctas CTAs x 8 warps; the message is cut into chunks of chunk_bytes, chunk c is moved by
// warp c mod (8 n_ctas) with the same per-warp code the fused kernel's communication warps
// run (transfer.cuh), then the warp fences its writes to system scope as a chunk release
// would.
#include <cuda_runtime.h>

#include "kernel_args.h"
#include "ptx.cuh"
#include "transfer.cuh"

namespace ao {
namespace dev {

constexpr int kE4Warps = 8;
constexpr uint32_t kE4Buf = 12288;  // staging per buffer (as the dedicated comm CTAs)

template <int COMM>
__global__ void __launch_bounds__(kE4Warps * 32) transfer_kernel(char* dst, const char* src, int64_t bytes,
                                                                 int64_t chunk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kE4Warps * 2 * kE4Buf) + warp * 2;
  if (COMM == COMM_TMA && lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t phase_bits = 0;
  const int64_t n_chunks = (bytes + chunk - 1) / chunk;
  const int64_t gw = int64_t(blockIdx.x) * kE4Warps + warp, nw = int64_t(gridDim.x) * kE4Warps;
  for (int64_t c = gw; c < n_chunks; c += nw) {
    const int64_t off = c * chunk;
    const int64_t len = bytes - off < chunk ? bytes - off : chunk;
    if constexpr (COMM == COMM_LDST) {
      warp_copy_ldst<8>(dst + off, src + off, len, false);
      __syncwarp();
      if (lane == 0) fence_sys();
    } else {
      if (lane == 0) {
        lane0_copy_tma(dst + off, src + off, len, smem + warp * 2 * kE4Buf, kE4Buf, bars, phase_bits);
        fence_proxy_async_global();
        fence_sys();
      }
      __syncwarp();
    }
  }
}

}  // namespace dev

cudaError_t launch_transfer(int comm, char* dst, const char* src, int64_t bytes, int64_t chunk, int n_ctas,
                            cudaStream_t stream) {
  const size_t smem = dev::kE4Warps * 2 * dev::kE4Buf + dev::kE4Warps * 16 + 1024;
  if (comm == COMM_TMA) {
    static bool set = false;
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(dev::transfer_kernel<COMM_TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(smem));
      if (e != cudaSuccess) return e;
      set = true;
    }
    dev::transfer_kernel<COMM_TMA><<<n_ctas, dev::kE4Warps * 32, smem, stream>>>(dst, src, bytes, chunk);
  } else {
    dev::transfer_kernel<COMM_LDST><<<n_ctas, dev::kE4Warps * 32, 0, stream>>>(dst, src, bytes, chunk);
  }
  return cudaGetLastError();
}

}  // namespace ao
