// a2a.cu -- A2A-GEMM (NEXT-3) prep kernel: routing -> per-expert counts and the token
// permutation, the count exchange (every rank publishes its count row to every rank and
// acquires everyone's), and the route positions.  One CTA per rank of the launch.
//
// Definitions (Q25; oracle/a2a.py): S(s -> e) = ascending tokens of rank s with
// e in topk_idx[t, :]; expert e receives concat_s X_s[S(s -> e)]; route_pos[t, j] = row of
// (s, t) in expert topk_idx[t, j]'s block = sum_{s' < s} cnt[s'][e] + rank of t in S(s -> e).
// Flag words of a parity: chunk flags [W][maxJ] from word 0; count flags [W] and the count
// table [W][W] in the reserved tail (kernel_args.h).
#include <cuda_runtime.h>

#include "kernel_args.h"
#include "ptx.cuh"

namespace ao {
namespace dev {

constexpr int kPrepThreads = 1024;

__device__ __forceinline__ void prep_spin(const uint32_t* p, uint32_t target, const A2APrepArgs& A, int rank, int s) {
  if (ld_relaxed_sys(p) >= target) {  // relaxed polls, one acquire (see fused.cu spin_flag)
    ld_acquire_sys(p);
    return;
  }
  const uint64_t t0 = globaltimer();
  while (ld_relaxed_sys(p) < target) {
    if (globaltimer() - t0 > A.timeout_ns) {
      if (atomicCAS(&A.err->claim, 0u, 1u) == 0u) {
        A.err->rank = rank;
        A.err->cta = -100;  // prep kernel (count exchange)
        A.err->chunk = s;
        A.err->epoch = target;
        A.err->seen = ld_acquire_sys(p);
        __threadfence_system();
        st_release_sys(const_cast<uint32_t*>(&A.err->flag), 1u);
      }
      return;
    }
    __nanosleep(64);
  }
  ld_acquire_sys(p);
}

__global__ void __launch_bounds__(kPrepThreads) a2a_prep_kernel(const __grid_constant__ A2APrepArgs a) {
  const A2APrepRank& R = a.rk[blockIdx.x];
  const int W = a.W, T = a.T, k = a.topk, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cf = int(kA2ACountFlags), ctb = cf + W;  // count flags, count table (word offsets)
  __shared__ int run[AO_MAX_WORLD];         // tokens of each expert placed so far
  __shared__ int wsum[kPrepThreads / 32];
  __shared__ int tab[AO_MAX_WORLD][AO_MAX_WORLD];
  if (tid < W) run[tid] = 0;
  __syncthreads();
  // 1. per expert: stable (ascending token) positions by a block-wide exclusive scan
  for (int base = 0; base < T; base += kPrepThreads) {
    const int t = base + tid;
    int ids[AO_MAX_WORLD];
    for (int j = 0; j < k; ++j) {
      // the ABI requires k distinct expert ids in [0, W): an out-of-range or repeated id is
      // reported (AO_ERR_INVALID_ARG through the error record) and that entry is dropped
      // (route_pos = -1) instead of indexing out of bounds
      int id = t < T ? R.topk_idx[int64_t(t) * k + j] : -1;
      bool bad = t < T && (id < 0 || id >= W);
      for (int jj = 0; jj < j && !bad && t < T; ++jj) bad = id == ids[jj];
      if (bad) {
        if (atomicCAS(&a.err->claim, 0u, 1u) == 0u) {
          a.err->rank = R.rank;
          a.err->cta = kErrBadRouting;
          a.err->chunk = t;
          a.err->epoch = uint32_t(j);
          a.err->seen = uint32_t(id);
          __threadfence_system();
          st_release_sys(const_cast<uint32_t*>(&a.err->flag), 1u);
        }
        R.lpos[int64_t(t) * k + j] = -1;
        id = -1;
      }
      ids[j] = id;
    }
    for (int e = 0; e < W; ++e) {
      int jj = -1;
      for (int j = 0; j < k; ++j)
        if (ids[j] == e) jj = j;
      const bool m = jj >= 0;
      const unsigned bal = __ballot_sync(0xffffffffu, m);
      if (lane == 0) wsum[wid] = __popc(bal);
      __syncthreads();
      if (wid == 0) {
        int v = lane < kPrepThreads / 32 ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += y;
        }
        wsum[lane] = v;  // inclusive
      }
      __syncthreads();
      const int before = (wid ? wsum[wid - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
      if (m) {
        const int pos = run[e] + before;
        R.perm[int64_t(e) * T + pos] = t;
        R.lpos[int64_t(t) * k + jj] = pos;
      }
      __syncthreads();
      if (tid == 0) run[e] += wsum[kPrepThreads / 32 - 1];
      __syncthreads();
    }
  }
  // 2. publish this rank's count row to every rank, then release its count flag there
  if (tid < W * W) {
    const int q = tid / W, e = tid % W;
    R.peer_flags[q][ctb + R.rank * W + e] = uint32_t(run[e]);
  }
  __syncthreads();
  if (tid < W) {
    asm volatile("fence.sc.sys;" ::: "memory");
    st_release_sys(R.peer_flags[tid] + cf + R.rank, a.epoch);
  }
  // 3. acquire every source's count row (the whole matrix, identical on every rank)
  if (tid < W) prep_spin(R.peer_flags[R.rank] + cf + tid, a.epoch, a, R.rank, tid);
  __syncthreads();
  if (tid < W * W) tab[tid / W][tid % W] = int(__ldcg(R.peer_flags[R.rank] + ctb + tid));
  __syncthreads();
  // 4. route positions and the received row count
  for (int x = tid; x < T * k; x += kPrepThreads) {
    const int lp = R.lpos[x];
    if (lp < 0) {  // dropped (invalid) routing entry
      R.route_pos[x] = -1;
      continue;
    }
    const int e = R.topk_idx[x];
    int base = 0;
    for (int q = 0; q < R.rank; ++q) base += tab[q][e];
    R.route_pos[x] = base + lp;
  }
  if (tid == 0) {
    int r = 0;
    for (int q = 0; q < W; ++q) r += tab[q][R.rank];
    *R.recv_rows = r;
  }
}

}  // namespace dev

cudaError_t launch_a2a_prep(const A2APrepArgs& args, cudaStream_t stream) {
  dev::a2a_prep_kernel<<<args.n_group, dev::kPrepThreads, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace ao
