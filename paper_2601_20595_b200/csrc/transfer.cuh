// transfer.cuh -- the in-kernel transfer backends of P:397 / Fig.7 (one warp moves one
// contiguous byte range), shared by the fused kernel's communication warps (fused.cu) and
// the backend microbenchmark (e4.cu, SURVEY.md §8(d) "E4"), so E4 measures exactly the
// code the fused ops run.
//   TMA : lane 0 streams the range through two smem staging buffers with 1-D bulk copies
//         (cp.async.bulk global -> shared -> global, the store of piece p overlapping the
//         load of piece p+1), then waits until the writes are performed.
//   LDST: all 32 lanes move 16-byte vectors, 8 loads in flight per lane before the stores.
// The caller orders the data before its release flag (fences) -- not done here.
#pragma once
#include "ptx.cuh"

namespace ao {
namespace dev {

__device__ __forceinline__ int4 ld_nc_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// LDST: every lane of the warp; `coherent_src` for peer data written during the kernel.
// U 16-byte loads per lane in flight (U * 512 bytes per warp): the copy is latency-bound at
// (bytes in flight) / (load latency), so warps with registers to spare use a larger U.
template <int U = 8>
__device__ __forceinline__ void warp_copy_ldst(char* dst, const char* src, int64_t bytes, bool coherent_src) {
  const int lane = lane_id();
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  const int64_t n = bytes / 16;
  for (int64_t base = 0; base < n; base += 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = base + u * 32 + lane;
      if (j < n) v[u] = coherent_src ? __ldcg(s + j) : ld_nc_v4(s + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = base + u * 32 + lane;
      if (j < n) st_v4(d + j, v[u]);
    }
  }
}

// TMA: lane 0 only.  `bars` = 2 mbarriers (count 1) whose phases `phase_bits` carries
// across calls; staging = 2 x buf_bytes of shared memory.  Returns with the writes performed.
__device__ __forceinline__ void lane0_copy_tma(char* dst, const char* src, int64_t bytes, uint8_t* staging,
                                               uint32_t buf_bytes, uint64_t* bars, uint32_t& phase_bits) {
  if (bytes <= 0) return;
  const int64_t npieces = (bytes + buf_bytes - 1) / buf_bytes;
  auto piece_len = [&](int64_t p) -> uint32_t {
    const int64_t rem = bytes - p * int64_t(buf_bytes);
    return uint32_t(rem < int64_t(buf_bytes) ? rem : int64_t(buf_bytes));
  };
  {
    const uint32_t n0 = piece_len(0);
    mbar_arrive_expect_tx(&bars[0], n0);
    bulk_g2s(staging, src, n0, &bars[0]);
  }
  for (int64_t p = 0; p < npieces; ++p) {
    const int b = int(p & 1);
    if (p + 1 < npieces) {
      const int nb = b ^ 1;
      bulk_wait_read<0>();  // the store that last used buffer nb has read it
      const uint32_t n1 = piece_len(p + 1);
      mbar_arrive_expect_tx(&bars[nb], n1);
      bulk_g2s(staging + nb * buf_bytes, src + (p + 1) * int64_t(buf_bytes), n1, &bars[nb]);
    }
    mbar_wait(&bars[b], (phase_bits >> b) & 1);
    phase_bits ^= (1u << b);
    bulk_s2g(dst + p * int64_t(buf_bytes), staging + b * buf_bytes, piece_len(p));
    bulk_commit();
  }
  bulk_wait<0>();  // writes performed
}

}  // namespace dev
}  // namespace ao
