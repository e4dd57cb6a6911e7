// fused.cu -- the persistent fused kernel: tcgen05 GEMM mainloop + chunk waits (AG) or
// partial pushes + owner reduction (RS) + in-kernel transfer backends (TMA / LD-ST).
//
// Method (§5.2):
//  * the tile scheduler follows the planner's chunk-ordered tile list (Fig.6);
//  * a tile that consumes a chunk waits on that chunk's global-memory signal, once per
//    (worker, chunk) (minimal waits) -- producer warp, ld.acquire.sys spin;
//  * communication is issued from inside the fused kernel: co-located
//    communication warps or dedicated communication CTAs ("specialized SMs", Fig.7b/c)
//    push chunks with cp.async.bulk (TMA backend) or 16-byte ld/st (LDST backend);
//  * GEMM-RS: each finished fp32 partial tile is written into its owner's slot; the last
//    tile of a chunk releases the owner's flag.  The owner computes its own rows last; the
//    epilogue of an own tile waits for the other sources' flags of its chunks, adds their
//    partials to its TMEM accumulator in ascending source rank and stores bf16 --
//    the peer reduction fused into the epilogue (north star).
//
// Tile = BM x BN with BM = 128 * CG.  CG = 2 runs one tile on a CTA pair (cluster of 2,
// tcgen05.mma.cta_group::2, M = 256): each CTA loads its 128 rows of A and half of B's
// rows; the even CTA issues the MMA for both; each CTA's TMEM holds its 128 rows.
//
// Warp roles (1 CTA / SM):
//   warp 0      TMA producer (+ AG chunk waits)
//   warp 1      TMEM allocator + tcgen05.mma issuer (leader CTA of the pair)
//   warps 2..5  epilogue (TMEM -> registers -> smem transpose -> global; RS signals)
//   warps 6..7  AG: co-located communication warps
#include <cuda_runtime.h>

#include "kernel_args.h"
#include "ptx.cuh"
#include "transfer.cuh"

// Timing experiments (ao_debug_set "exp" bits: skip reduces, waits, ...; results invalid)
// are compiled in only with -DAO_TIMING_EXPERIMENTS=1 (AO_NVCC_FLAGS); the production
// build folds every xp() to false.
#ifndef AO_TIMING_EXPERIMENTS
#define AO_TIMING_EXPERIMENTS 0
#endif

namespace ao {
namespace dev {

__device__ __forceinline__ bool xp(const KernelArgs& a, int bit) { return AO_TIMING_EXPERIMENTS && (a.exp & bit); }

constexpr int kSubM = 128;  // rows per CTA (TMEM lanes)
constexpr int kBK = 64;
constexpr int kThreads = 256;  // AG / GEMM / A2A CTAs (and AG's dedicated comm CTAs)
// Epilogue warps per mode: GEMM-RS's epilogue (fp32 partial pushes + the owner's fused
// reduction) is the critical role, so RS CTAs run 8 (two per TMEM lane quadrant, each
// taking half of the tile's columns), the other modes 4.
template <int MODE>
struct Roles {
  static constexpr int kEpiW = MODE == 2 ? 8 : 4;        // MODE_RS == 2
  static constexpr int kCommWarp0 = 2 + kEpiW;           // first co-located comm warp
  static constexpr int kThreads = 32 * (kCommWarp0 + 2);  // + 2 comm warps (AG / A2A / GEMM-AR gather)
};
constexpr int kColocCommWarps = 2;
constexpr int kCommBufs = 2;
constexpr uint32_t kColocBufBytes = 4096;
constexpr uint32_t kStageWarpBytes = 4096;  // epilogue transpose buffer per warp (32 rows x 128 B)
constexpr uint32_t kCtaBufBytes = 12288;
constexpr int kOperandBudget = 196608;  // bytes of smem for the A/B stage ring
constexpr int kAhead = 4;  // AG (copy engine): tiles whose chunk waits the wait warp may run ahead

constexpr int kA2ABuf = 8192;        // A2A dispatch: bytes per TMA staging buffer
constexpr int kA2ABufs = 4;          // A2A dispatch: staging buffers (loads in flight)
constexpr int kA2AOperandBudget = 163840;  // A2A: one ring stage less, for the staging buffers
constexpr int kRsStg = 1;                  // RS: TMA-reduce staging buffers per epilogue warp (8 warps)
#ifndef AO_AR_PULL_U
#define AO_AR_PULL_U 32
#endif
constexpr int kArPullU = AO_AR_PULL_U;     // GEMM-AR gather: 16-byte loads in flight per lane
constexpr int kRsOperandBudget = 196608;   // RS ring (4 staging buffers + a 5-stage ring measured no faster)

// CG = CTAs per cluster: 1 (one CTA, M = 128), 2 (a CTA pair running cta_group::2 MMAs,
// M = 256) or 4 (two CTA pairs stacked along M, BM = 512, whose B rows are the same: each
// CTA loads a quarter of the tile's B rows and TMA-multicasts it to the same-position CTA
// of both pairs, so every B byte crosses the L2 -> SM crossbar once per cluster).
template <int BN, int CG, int BUDGET = kOperandBudget>
struct Cfg {
  static constexpr int kCGM = CG >= 2 ? 2 : 1;  // cta_group of the MMA
  static constexpr int kNP = CG / kCGM;          // CTA pairs sharing B (multicast) per cluster
  static constexpr int kStageA = kSubM * kBK * 2;
  static constexpr int kStageB = (BN / kCGM) * kBK * 2;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kStages = BUDGET / kStage;
  // two accumulators of BN fp32 columns; tcgen05.alloc takes a power of two >= 32
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static_assert(BN % (8 * CG) == 0 && BN <= 256 && BN >= 16, "tile N: multiple of 8 * CTAs per cluster, at most 256");
  static constexpr int kBM = kSubM * CG;
};

struct SmemLayout {
  uint32_t off_a, off_b, off_stg, off_comm, off_bar, off_slot, off_a2a, total;
};

// ---- A2A (NEXT-3) device-side schedule ---------------------------------------------------
// Built by every CTA after the count exchange (prep kernel): the count matrix, each
// expert's block offsets, the received rows, and per rank group the row blocks sorted by
// the arrival position of their latest chunk (the chunk->tile join of S:430 on ragged,
// routing-dependent chunks).
constexpr int kA2AMaxMb = 128;  // row blocks per expert (host-validated: W*T / BM)
struct A2ASched {
  int tab[AO_MAX_WORLD][AO_MAX_WORLD];   // cnt[s][e]: tokens of source s routed to expert e
  int offd[AO_MAX_WORLD][AO_MAX_WORLD];  // offd[e][s]: first row of source s's block at expert e
  int rows[AO_MAX_WORLD];                // per rank group: received rows R_e
  int nmb[AO_MAX_WORLD];                 // per rank group: row blocks
  int tprefix[AO_MAX_WORLD + 1];         // tiles before rank group g (time-sliced walk)
  int key[AO_MAX_WORLD][kA2AMaxMb];      // arrival position of a row block's latest chunk
  uint8_t order[AO_MAX_WORLD][kA2AMaxMb];  // row blocks in execution order
};

template <int BN, int CG, int BUDGET = kOperandBudget>
__host__ __device__ constexpr SmemLayout gemm_layout(bool tma_comm, bool dbl_stg, bool a2a = false) {
  using C_ = Cfg<BN, CG, BUDGET>;
  SmemLayout L{};
  L.off_a = 0;
  L.off_b = C_::kStages * C_::kStageA;
  L.off_stg = C_::kStages * C_::kStage;
  L.off_comm = L.off_stg + (dbl_stg ? 8 * kRsStg : 4) * kStageWarpBytes;  // RS: 8 warps x kRsStg buffers (TMA reduce)
  const uint32_t comm = tma_comm ? kColocCommWarps * kCommBufs * kColocBufBytes : (a2a ? kA2ABufs * kA2ABuf : 0);
  L.off_bar = L.off_comm + comm;
  const uint32_t nbars = 3 * C_::kStages + 4 + 8 * kCommBufs + 2 * kAhead;
  L.off_slot = L.off_bar + nbars * 8;
  L.off_a2a = (L.off_slot + 16 + kAhead + 15) / 16 * 16;
  L.total = L.off_a2a + (a2a ? uint32_t(sizeof(A2ASched)) : 0u) + 1024;  // + alignment slack
  return L;
}
__host__ __device__ constexpr SmemLayout comm_cta_layout() {
  SmemLayout L{};
  L.off_comm = 0;
  L.off_bar = 8 * kCommBufs * kCtaBufBytes;
  L.off_slot = L.off_bar + 8 * kCommBufs * 8;
  L.total = L.off_slot + 16 + 1024;
  return L;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Bounded spin on a flag word until it reaches `target` (an epoch).  On timeout the first
// failure is recorded in the host-mapped ErrorInfo and the wait is abandoned (no hang).
__device__ __noinline__ void spin_flag(const uint32_t* p, uint32_t target, const KernelArgs& A, int rank, int cta,
                                       int g) {
  // relaxed polls; the acquire (which invalidates the SM's L1: LDG.STRONG.SYS + CCTL.IVALL)
  // only once the value is seen (flags are monotonic epochs, so the acquire reads a value
  // >= target and synchronizes with its release)
  uint32_t v = ld_relaxed_sys(p);
  if (v >= target) {
    ld_acquire_sys(p);
    return;
  }
  const uint64_t t0 = globaltimer();
  uint32_t ns = 32;
  while (true) {
    v = ld_relaxed_sys(p);
    if (v >= target) {
      ld_acquire_sys(p);
      return;
    }
    if (globaltimer() - t0 > A.timeout_ns) {
      if (atomicCAS(&A.err->claim, 0u, 1u) == 0u) {
        A.err->rank = rank;
        A.err->cta = cta;
        A.err->chunk = g;
        A.err->epoch = target;
        A.err->seen = v;
        __threadfence_system();
        st_release_sys(const_cast<uint32_t*>(&A.err->flag), 1u);  // publish after the fields
      }
      return;
    }
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

__device__ __forceinline__ void trace_event(const KernelArgs& A, uint32_t kind, int rank, int cta, int id, uint64_t t0) {
  if (A.trace == nullptr) return;
  const uint32_t i = atomicAdd(A.trace_cursor, 1u);
  if (i < A.trace_cap) {
    TraceEvent e;
    e.t0 = t0;
    e.t1 = globaltimer();
    e.kind = kind | (A.trace_seq << 8);
    e.rank = uint32_t(rank);
    e.cta = uint32_t(cta);
    e.id = uint32_t(id);
    A.trace[i] = e;
  }
}

// Fault injection: wait at least delay/2 (+ a hash-dependent part up to delay/2) ns.
__device__ __noinline__ void inject_delay(uint32_t delay, uint32_t salt) {
  if (delay == 0) return;
  const uint64_t target = delay / 2 + (salt * 2654435761u) % (delay / 2 + 1);
  const uint64_t t0 = globaltimer();
  while (globaltimer() - t0 < target) __nanosleep(1000);
}


// ---- communication workers (AG in-kernel backends) -----------------------------------------
// Each worker is one warp; worker w handles items w, w + n_workers, ... of this rank's
// ordered item list (plan order, so early chunks go first on every worker).
template <int COMM, int U = 8>
__device__ void comm_item(const RankArgs& R, const KernelArgs& A, int i, int worker, uint8_t* staging,
                          uint32_t buf_bytes, uint64_t* bars, uint32_t& phase_bits) {
  const int lane = lane_id();
  {
    const uint64_t t_item = A.trace ? globaltimer() : 0;
    if (A.delay_ns && lane == 0) inject_delay(A.delay_ns, uint32_t(i));  // fault injection
    __syncwarp();
    const CommItem it = R.comm_items[i];
    const bool remote_src = it.kind == ITEM_PULL || it.kind == ITEM_AR_PULL;
    const char* src = (remote_src ? R.peer_data[it.peer] : R.A_shard) + it.src_off;
    char* dst = it.kind == ITEM_AR_PULL ? R.ar_out + it.dst_off
                                        : R.peer_data[it.kind == ITEM_PUSH ? it.peer : R.rank] + it.dst_off;
    if (remote_src) {
      // PULL (Lst.2): the source staged its chunk and released its ready flag;
      // AR_PULL: the owner reduced its chunk and released its "reduced" flag
      if (lane == 0) {
        const uint32_t* f = R.peer_flags[it.peer] +
                            (it.kind == ITEM_PULL ? it.g * R.n_slices + it.slice : R.n_chunks * R.W + it.g);
        spin_flag(f, R.epoch, A, R.rank, -1 - worker, it.g);
        fence_proxy_async_global();  // generic-proxy acquire -> bulk (async-proxy) reads
      }
      __syncwarp();
    }
    if constexpr (COMM == COMM_LDST) {
      warp_copy_ldst<U>(dst, src, it.bytes, remote_src);  // peer data: coherent loads
      __syncwarp();
      if (lane == 0) asm volatile("fence.sc.sys;" ::: "memory");
    } else {
      if (lane == 0 && it.bytes > 0) {
        lane0_copy_tma(dst, src, it.bytes, staging, buf_bytes, bars, phase_bits);
        fence_proxy_async_global();
        fence_sys();
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (it.kind != ITEM_AR_PULL) {
        uint32_t* f = it.kind == ITEM_PUSH ? R.peer_flags[it.peer] : R.flags;
        st_release_sys(f + it.g * R.n_slices + it.slice, R.epoch);
      }
      trace_event(A, TR_COMM, R.rank, worker, i, t_item);
    }
    __syncwarp();
  }
}

template <int COMM, int U = 8>
__device__ void comm_worker(const RankArgs& R, const KernelArgs& A, int worker, int n_workers, uint8_t* staging,
                            uint32_t buf_bytes, uint64_t* bars) {
  uint32_t phase_bits = 0;
  for (int i = worker; i < R.n_comm_items; i += n_workers)
    comm_item<COMM, U>(R, A, i, worker, staging, buf_bytes, bars, phase_bits);
}

// Time-sliced AG group (in-kernel push backends): the comm warps of every CTA serve every
// source rank's items, destination-major in the order the ranks' tiles run (each rank's
// chunks land before its turn), like the copy-engine chains of a time-sliced group.
template <int COMM, int U = 8>
__device__ void comm_worker_ts(const KernelArgs& A, int worker, int n_workers, uint8_t* staging, uint32_t buf_bytes,
                               uint64_t* bars) {
  uint32_t phase_bits = 0;
  int cnt = 0;  // items before this (destination, source) block in the global order
  for (int gi = 0; gi < A.n_group; ++gi) {
    const int e = A.rk[gi].rank;  // destination (AG push) / owner (AR pull), in execution order
    for (int gs = 0; gs < A.n_group; ++gs) {
      const RankArgs& R = A.rk[gs];
      const int o0 = R.comm_peer_off[e], o1 = R.comm_peer_off[e + 1];
      // this worker's items of the block: global indices cnt + j with (cnt + j) % n == worker
      for (int j = o0 + ((worker - cnt) % n_workers + n_workers) % n_workers; j < o1; j += n_workers)
        comm_item<COMM, U>(R, A, R.comm_by_peer[j], worker, staging, buf_bytes, bars, phase_bits);
      cnt += o1 - o0;
    }
  }
}

// ---- tile walk --------------------------------------------------------------------------
// The k-blocks [kb0, kb1) of a tile position a worker runs, and their role: 0 = the whole
// tile; stream-K tail (Q28): 1 = a tail piece (k-blocks up to the end; its fp32 partial goes
// to the plan's stream-K workspace), 2 = a head piece (k-blocks from 0; adds the tail's
// partial and stores the tile).
struct KSpan {
  int kb0, kb1, role;
};

// Calls f(R, grp, k, span) for every tile position this worker runs, in order.
// Space-sliced: positions wk, wk + n_wk, ... of its own rank group's list (Lst.1,
// P:211-216) below sk_dp, then its contiguous range of the stream-K units (position-major
// (position, k-block) pairs of positions >= sk_dp, cut into n_wk equal ranges; planner.cpp
// worker_pieces, oracle/schedule.py worker_pieces).  Time-sliced: global indices wk,
// wk + n_wk, ... of the launch's segment list (whole tiles).
template <class F>
__device__ __forceinline__ void for_tiles(const KernelArgs& a, int grp, int wk, int n_wk, int nkb, F&& f) {
  if (a.n_seg == 0) {
    const RankArgs& R = a.rk[grp];
    const int dp = R.sk_dp < R.n_tiles ? R.sk_dp : R.n_tiles;
    for (int k = wk; k < dp; k += n_wk) f(R, grp, k, KSpan{0, nkb, 0});
    if (dp < R.n_tiles) {
      const int64_t U = int64_t(R.n_tiles - dp) * nkb;
      int64_t u = U * wk / n_wk;
      const int64_t u1 = U * (wk + 1) / n_wk;
      while (u < u1) {
        const int t = int(u / nkb), kb0 = int(u % nkb);
        const int kb1 = int(u1 - u < int64_t(nkb - kb0) ? int64_t(kb0) + (u1 - u) : int64_t(nkb));
        f(R, grp, dp + t, KSpan{kb0, kb1, (kb0 == 0 && kb1 == nkb) ? 0 : (kb0 != 0 ? 1 : 2)});
        u += kb1 - kb0;
      }
    }
  } else {
    int si = 0;
    for (int i = wk; i < a.n_total; i += n_wk) {
      while (i >= a.seg[si].o + (a.seg[si].k1 - a.seg[si].k0)) ++si;
      const int g = a.seg[si].g;
      f(a.rk[g], g, a.seg[si].k0 + (i - a.seg[si].o), KSpan{0, nkb, 0});
    }
  }
}

// Time-sliced chunk waits (dependency rule 4: a tile depends on every chunk its rows
// intersect): before the first tile of this worker that needs chunk g of rank group grp,
// acquire g's flags; later tiles needing g are covered by program order.
// `got` caches the acquired chunks (bit g of got[grp], chunks g < 64; others re-checked).
struct WaitCache {
  uint64_t got[AO_MAX_WORLD];
  __device__ void reset() {
    for (int i = 0; i < AO_MAX_WORLD; ++i) got[i] = 0;
  }
  __device__ bool has(int grp, int g) const { return g < 64 && ((got[grp] >> g) & 1u); }
  __device__ void set(int grp, int g) {
    if (g < 64) got[grp] |= 1ull << g;
  }
};

// AG: the remote chunks of rows [r0, r1); returns true if it waited on anything.
__device__ __noinline__ bool ts_wait_ag(const RankArgs& R, const KernelArgs& A, WaitCache& wc, int grp, int cta,
                                        int64_t r0, int64_t r1) {
  bool waited = false;
  for (int g = int(r0 / R.crows); g <= int((r1 - 1) / R.crows); ++g) {
    if ((int64_t(g) * R.crows) / R.S == R.rank || wc.has(grp, g)) continue;
    for (int s = 0; s < R.n_slices; ++s) spin_flag(R.flags + g * R.n_slices + s, R.epoch, A, R.rank, cta, g);
    wc.set(grp, g);
    waited = true;
  }
  return waited;
}

// RS: every other source's completion flag of the chunks of own rows [r0, r1).
__device__ __noinline__ void ts_wait_rs(const RankArgs& R, const KernelArgs& A, WaitCache& wc, int grp, int cta,
                                        int64_t r0, int64_t r1) {
  for (int g = int(r0 / R.crows); g <= int((r1 - 1) / R.crows); ++g) {
    if (wc.has(grp, g)) continue;
    for (int s = 0; s < R.W; ++s)
      if (s != R.rank) spin_flag(R.flags + g * R.W + s, R.epoch, A, R.rank, cta, g);
    wc.set(grp, g);
  }
}

// RS-3: count a finished 128-row partial sub-tile (rows [sub0, sub0 + 128) of `owner`) into
// each of its chunks; the last contributor releases the owner's flag[g][rank].  Called by
// one thread after a CTA barrier of the epilogue warps; one sys-scope fence is cumulative
// over their stores / performed reduces.
__device__ __forceinline__ void rs_signal(const RankArgs& R, const KernelArgs& A, int64_t sub0, int owner) {
  // No separate sys fence: the contributing warps' reduces are performed (bulk_wait 0) or
  // their stores precede the CTA barrier, and st.release.sys below is cumulative over
  // everything that happens-before it -- the release IS the fence (measured: a
  // fence.sc.sys here cost ~10 us per launch).
  if (xp(A, 32)) asm volatile("fence.sc.sys;" ::: "memory");
  const int glo = int(sub0 / R.crows);
  const int ghi = int((sub0 + kSubM - 1) / R.crows);
  for (int g = glo; g <= ghi; ++g) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(R.counters + g) : "memory");
    if (int(old) + 1 == R.tiles_per_chunk[g]) {
      R.counters[g] = 0;
      if (A.delay_ns) inject_delay(A.delay_ns, uint32_t(g));
      st_release_sys(R.peer_flags[owner] + g * R.W + R.rank, R.epoch);
    }
  }
}

// RS: 32-column blocks of tile column nb that hold valid columns (the streamed peer
// partial boxes of an own tile).
template <int BN>
__device__ __forceinline__ int rs_blocks(int nb, int64_t N) {
  const int64_t rem = N - int64_t(nb) * BN;
  const int64_t nbx = (rem + 31) / 32;
  return int(nbx < BN / 32 ? nbx : BN / 32);
}

// A2A: build the schedule (all threads of the CTA; ends with a CTA barrier).  Rank groups
// [g_lo, g_hi) are the ones this CTA serves.  pos(s, j) = d(s) * maxJ + j with d(s) =
// (e - s) mod W: the push rotation's arrival order at expert e (own rows first, Lst.2).
__device__ __noinline__ void a2a_build(A2ASched& sm, const KernelArgs& a, int g_lo, int g_hi, int BM) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const RankArgs& R0 = a.rk[g_lo];
  const int W = R0.W, C = R0.crows, maxJ = R0.maxJ;
  const uint32_t* ct = R0.flags + kA2ACountFlags + W;  // count table (identical on every rank)
  if (tid < W * W) sm.tab[tid / W][tid % W] = int(__ldcg(ct + tid));
  __syncthreads();
  if (tid < W * W) {
    const int e = tid / W, s = tid % W;
    int o = 0;
    for (int q = 0; q < s; ++q) o += sm.tab[q][e];
    sm.offd[e][s] = o;
  }
  if (tid < g_hi - g_lo) {
    const int g = g_lo + tid, e = a.rk[g].rank;
    int r = 0;
    for (int q = 0; q < W; ++q) r += sm.tab[q][e];
    sm.rows[g] = r;
    sm.nmb[g] = (r + BM - 1) / BM;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g <= AO_MAX_WORLD; ++g) {
      sm.tprefix[g] = acc;
      if (g >= g_lo && g < g_hi) acc += sm.nmb[g] * a.rk[g].n_nb;
    }
  }
  for (int x = tid; x < (g_hi - g_lo) * kA2AMaxMb; x += nt) {
    const int g = g_lo + x / kA2AMaxMb, mb = x % kA2AMaxMb;
    if (mb >= sm.nmb[g]) continue;
    const int e = a.rk[g].rank;
    const int r0 = mb * BM, r1 = min(sm.rows[g], r0 + BM);
    int key = -1;
    for (int q = 0; q < W; ++q) {
      const int b0 = sm.offd[e][q], b1 = b0 + sm.tab[q][e];
      const int lo = max(r0, b0), hi = min(r1, b1);
      if (lo < hi) key = max(key, ((e - q + W) % W) * maxJ + (hi - 1 - b0) / C);
    }
    sm.key[g][mb] = key;
  }
  __syncthreads();
  for (int x = tid; x < (g_hi - g_lo) * kA2AMaxMb; x += nt) {  // stable rank by (key, mb)
    const int g = g_lo + x / kA2AMaxMb, mb = x % kA2AMaxMb;
    if (mb >= sm.nmb[g]) continue;
    const int k0 = sm.key[g][mb];
    int rk = 0;
    for (int m = 0; m < sm.nmb[g]; ++m) rk += (sm.key[g][m] < k0 || (sm.key[g][m] == k0 && m < mb)) ? 1 : 0;
    sm.order[g][rk] = uint8_t(mb);
  }
  __syncthreads();
}

// A2A tile k of rank group g -> (row block, column block): Triton GROUP_M over the sorted
// row-block list (P:411 intra-chunk swizzle), gm row blocks per group.
__device__ __forceinline__ int2 a2a_tile(const A2ASched& sm, const RankArgs& R, int g, int k) {
  const int nmb = sm.nmb[g], nnb = R.n_nb, gm = R.gm;
  const int per = gm * nnb;
  const int first = (k / per) * gm;
  const int size = min(nmb - first, gm);
  const int r = k % per;
  return make_int2(sm.order[g][first + r % size], r / size);
}

template <class F>
__device__ __forceinline__ void for_tiles_a2a(const KernelArgs& a, const A2ASched& sm, int grp, int wk, int n_wk, F&& f) {
  if (!a.a2a_ts) {
    const int n = sm.nmb[grp] * a.rk[grp].n_nb;
    for (int k = wk; k < n; k += n_wk) f(a.rk[grp], grp, k, KSpan{0, 0, 0});
  } else {
    int g = 0;
    for (int i = wk; i < sm.tprefix[a.n_group]; i += n_wk) {
      while (i >= sm.tprefix[g + 1]) ++g;
      f(a.rk[g], g, i - sm.tprefix[g], KSpan{0, 0, 0});
    }
  }
}

// A2A waits: every (source, chunk) flag of expert e's rows [r0, r1).
__device__ __noinline__ bool a2a_wait(const A2ASched& sm, const RankArgs& R, const KernelArgs& A, WaitCache& wc, int grp,
                                      int cta, int r0, int r1) {
  bool waited = false;
  const int W = R.W, e = R.rank;
  for (int q = 0; q < W; ++q) {
    const int b0 = sm.offd[e][q], b1 = b0 + sm.tab[q][e];
    const int lo = max(r0, b0), hi = min(r1, b1);
    if (lo >= hi) continue;
    for (int j = (lo - b0) / R.crows; j <= (hi - 1 - b0) / R.crows; ++j) {
      const int w = q * R.maxJ + j;
      if (wc.has(grp, w)) continue;
      spin_flag(R.flags + w, R.epoch, A, R.rank, cta, w);
      wc.set(grp, w);
      waited = true;
    }
  }
  return waited;
}

// A2A dispatch (comm warp): copy chunk j of source group gs's block for expert e -- a row
// gather of the routed tokens (16-byte ld/st) -- then release the expert's flag (s, j).
__device__ __noinline__ void a2a_push_chunk(const A2ASched& sm, const RankArgs& S_, const KernelArgs& A, int e, int j) {
  const int lane = lane_id();
  const int s = S_.rank, C = S_.crows;
  const int cnt = sm.tab[s][e];
  const int i0 = j * C, i1 = min(cnt, i0 + C);
  const int64_t row_bytes = S_.K * 2;
  const int n16 = int(row_bytes / 16);
  const int32_t* perm = S_.a2a_perm + int64_t(e) * S_.T;
  char* dst0 = S_.peer_data[e] + (int64_t(sm.offd[e][s]) + i0) * row_bytes;
  for (int i = i0; i < i1; ++i) {
    const int4* src = reinterpret_cast<const int4*>(S_.A_shard + int64_t(perm[i]) * row_bytes);
    int4* dst = reinterpret_cast<int4*>(dst0 + int64_t(i - i0) * row_bytes);
    constexpr int U = 8;
    for (int b = 0; b < n16; b += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = b + u * 32 + lane;
        if (x < n16) v[u] = ld_nc_v4(src + x);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = b + u * 32 + lane;
        if (x < n16) st_v4(dst + x, v[u]);
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.sc.sys;" ::: "memory");
    st_release_sys(S_.peer_flags[e] + s * S_.maxJ + j, S_.epoch);
  }
  __syncwarp();
}

// Same chunk through the TMA unit (lane 0): pieces of <= kA2ABuf bytes of the gathered
// rows, global -> smem (kA2ABufs loads in flight) -> the expert's receive buffer; then
// the flag (s, j) is released.  `par` carries the staging barriers' parities across items.
__device__ __noinline__ void a2a_push_chunk_tma(const A2ASched& sm, const RankArgs& S_, const KernelArgs& A, int e, int j,
                                                uint8_t* buf, uint64_t* bars, uint32_t& par) {
  const int s = S_.rank, C = S_.crows;
  const int cnt = sm.tab[s][e];
  const int i0 = j * C, i1 = min(cnt, i0 + C);
  const int64_t row_bytes = S_.K * 2;
  const int np = int((row_bytes + kA2ABuf - 1) / kA2ABuf);
  const int total = (i1 - i0) * np;
  const int32_t* perm = S_.a2a_perm + int64_t(e) * S_.T;
  char* dst0 = S_.peer_data[e] + (int64_t(sm.offd[e][s]) + i0) * row_bytes;
  auto piece = [&](int q, const char** src, char** dst) -> uint32_t {
    const int i = i0 + q / np, part = q % np;
    const int64_t o = int64_t(part) * kA2ABuf;
    *src = S_.A_shard + int64_t(perm[i]) * row_bytes + o;
    *dst = dst0 + int64_t(i - i0) * row_bytes + o;
    const int64_t rem = row_bytes - o;
    return uint32_t(rem < int64_t(kA2ABuf) ? rem : int64_t(kA2ABuf));
  };
  for (int q = 0; q < min(kA2ABufs, total); ++q) {
    const char* src;
    char* dst;
    const uint32_t len = piece(q, &src, &dst);
    mbar_arrive_expect_tx(&bars[q], len);
    bulk_g2s(buf + q * kA2ABuf, src, len, &bars[q]);
  }
  for (int q = 0; q < total; ++q) {
    const int b = q % kA2ABufs;
    const char* src;
    char* dst;
    const uint32_t len = piece(q, &src, &dst);
    mbar_wait(&bars[b], (par >> b) & 1u);
    par ^= 1u << b;
    bulk_s2g(dst, buf + b * kA2ABuf, len);
    bulk_commit();
    if (q + kA2ABufs < total) {
      bulk_wait_read<0>();  // the store just issued has read buffer b
      const uint32_t l2 = piece(q + kA2ABufs, &src, &dst);
      mbar_arrive_expect_tx(&bars[b], l2);
      bulk_g2s(buf + b * kA2ABuf, src, l2, &bars[b]);
    }
  }
  bulk_wait<0>();  // writes performed
  fence_proxy_async_global();
  fence_sys();
  if (A.delay_ns) inject_delay(A.delay_ns, uint32_t(s * 977 + e * 131 + j));  // fault injection
  st_release_sys(S_.peer_flags[e] + s * S_.maxJ + j, S_.epoch);
}

// AG (copy-engine pushes) and plain GEMM are bounded at 168 registers per thread (the 384-
// thread bound; launched with 256): the loopback pushes are same-device memcpys that run as
// SM kernels beside this persistent kernel and need registers left on every SM (DESIGN.md
// §8: a persistent kernel without that headroom stalled them and its chunk waits timed out).
#ifndef AO_AG_BOUND_THREADS
#define AO_AG_BOUND_THREADS 384  // 256: AG / GEMM uncapped (experiment: the cap's cost)
#endif
template <int BN, int MODE, int COMM, int CG>
__global__ void __launch_bounds__((MODE == MODE_AG || MODE == MODE_GEMM) ? AO_AG_BOUND_THREADS
                                                                      : (MODE == MODE_RS ? 384 : kThreads), 1)
    fused_kernel(const __grid_constant__ KernelArgs args) {
  static_assert((MODE != MODE_RS && MODE != MODE_A2A) || BN % 32 == 0, "RS / A2A epilogues step 32 columns");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool ts = args.n_seg > 0 || (MODE == MODE_A2A && args.a2a_ts);  // time-sliced: every GEMM CTA serves every rank
  const int gemm_ctas = ts ? args.ctas_per_rank : args.n_group * args.ctas_per_rank;

  // ------------------------------------------------------------------ dedicated comm CTA
  if (int(blockIdx.x) >= gemm_ctas) {
    if constexpr (MODE == MODE_AG && COMM != COMM_NONE) {
      const SmemLayout L = comm_cta_layout();
      uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar) + warp * kCommBufs;
      if (lane == 0) {
        for (int b = 0; b < kCommBufs; ++b) mbar_init(&bars[b], 1);
        fence_barrier_init();
      }
      __syncwarp();
      const int idx = blockIdx.x - gemm_ctas;
      const int grp = idx / args.comm_ctas_per_rank;
      const int c = idx % args.comm_ctas_per_rank;
      comm_worker<COMM>(args.rk[grp], args, c * 8 + warp, args.comm_ctas_per_rank * 8,
                        smem + L.off_comm + warp * kCommBufs * kCtaBufBytes, kCtaBufBytes, bars);
    }
    return;
  }

  // ------------------------------------------------------------------ GEMM CTA
  constexpr int kBudget = MODE == MODE_A2A ? kA2AOperandBudget : (MODE == MODE_RS ? kRsOperandBudget : kOperandBudget);
  using C_ = Cfg<BN, CG, kBudget>;
  constexpr int BM = C_::kBM;
  constexpr bool kTmaComm = (MODE == MODE_AG && COMM == COMM_TMA);
  constexpr SmemLayout L = gemm_layout<BN, CG, kBudget>(kTmaComm, MODE == MODE_RS, MODE == MODE_A2A);
  const int grp = blockIdx.x / args.ctas_per_rank;
  const int lcta = blockIdx.x % args.ctas_per_rank;  // CTA index inside the rank group
  const int wk = lcta / CG;                          // plan worker (the cluster: CTA, pair, 2 pairs)
  const int n_wk = args.ctas_per_rank / CG;
  constexpr int CGM = C_::kCGM, NP = C_::kNP;
  const uint32_t crk = (CG >= 2) ? cluster_ctarank() : 0u;  // CTA r of the cluster holds rows r*128 of the tile
  const uint32_t crank = crk & 1u;                           // position in its pair: 0 = leader (even CTA)
  const uint32_t pp = crk >> 1;                              // pair index in the cluster (CG == 4)
  const bool leader = crank == 0;
  const RankArgs& R0 = args.rk[grp];  // shapes (equal across the group: same plan hash)

  uint8_t* sA = smem + L.off_a;
  uint8_t* sB = smem + L.off_b;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* empty = full + C_::kStages;
  uint64_t* tfull = empty + C_::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* commbars = tempty + 2;
  uint64_t* pfull = commbars + 8 * kCommBufs;  // RS: ring stages carrying peer partials
  uint64_t* wrdy = pfull + C_::kStages;        // AG (CE): wait warp -> producer, per tile
  uint64_t* wfre = wrdy + kAhead;              // producer -> wait warp (slot reusable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.off_slot);
  volatile uint8_t* wwaited = smem + L.off_slot + 16;  // per slot: the wait warp acquired a flag
  // AG without in-kernel transfers: the chunk waits (ld.acquire.sys polls, microseconds each
  // under load) run in the otherwise idle warp 6, up to kAhead tiles ahead of the TMA
  // producer, which only waits on a shared-memory barrier (P:392's waits off the load path).
  constexpr bool kWaitWarp = (MODE == MODE_AG && COMM == COMM_NONE) || MODE == MODE_A2A;

  if (warp == 0 && lane == 0) {
    for (int g = ts ? 0 : grp; g < (ts ? args.n_group : grp + 1); ++g) {
      const RankArgs& R = args.rk[g];
      if (R.K > 0) {
        prefetch_tmap(&R.tmA);
        prefetch_tmap(&R.tmB);
        if (MODE == MODE_AG) prefetch_tmap(&R.tmA_loc);
      }
      if (MODE == MODE_RS && R.W > 1) prefetch_tmap(&R.tmA_loc);
    }
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < C_::kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], NP);  // CG == 4: both pairs' MMAs read this CTA's B quarter
        mbar_init(&pfull[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], Roles<MODE>::kEpiW * CGM);
      }
      for (int a = 0; a < kAhead; ++a) {
        mbar_init(&wrdy[a], 1);
        mbar_init(&wfre[a], 1);
      }
      for (int b = 0; b < 8 * kCommBufs; ++b) mbar_init(&commbars[b], 1);
      fence_barrier_init();
    }
    __syncwarp();
    if constexpr (CG >= 2) {
      tmem_alloc_cg2(tmem_slot, C_::kTmemCols);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(tmem_slot, C_::kTmemCols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if constexpr (CG >= 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  A2ASched& a2s = *reinterpret_cast<A2ASched*>(smem + L.off_a2a);
  if constexpr (MODE == MODE_A2A) a2a_build(a2s, args, ts ? 0 : grp, ts ? args.n_group : grp + 1, BM);
  // the tile walk of every role (A2A: routing-dependent list built above)
  auto walk = [&](auto&& f) {
    if constexpr (MODE == MODE_A2A)
      for_tiles_a2a(args, a2s, grp, wk, n_wk, f);
    else
      for_tiles(args, grp, wk, n_wk, int((R0.K + kBK - 1) / kBK), f);
  };
  // (row block, column block) of tile k of rank group g
  auto tile_of = [&](const RankArgs& R, int g, int k) -> int2 {
    if constexpr (MODE == MODE_A2A) {
      return a2a_tile(a2s, R, g, k);
    } else {
      const int t = R.order[k];
      return make_int2(t / R.n_nb, t - (t / R.n_nb) * R.n_nb);
    }
  };

  const int64_t K = R0.K, N = R0.N, S = R0.S, M = R0.M;
  const int nkb = int((K + kBK - 1) / kBK);

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      // L2 policy follows the tile order: with grouped / column orders an A row block is
      // reused across every column tile of its group, B tiles only by neighbours in time.
      // l2_hint: 0 A first / B last, 1 A last / B first, 2 A last / B normal, 3 both normal
      const int h = args.l2_hint & 3;
      const uint64_t pol_b = xp(args, 512) ? policy_evict_first()
                             : h == 0 ? policy_evict_last() : (h == 1 ? policy_evict_first() : policy_evict_normal());
      const uint64_t pol_a = h == 0 ? policy_evict_first() : (h == 3 ? policy_evict_normal() : policy_evict_last());
      uint32_t stage = 0, phase = 0;
      int wp = 0, we = 0;
      if constexpr (MODE != MODE_GEMM) {
        if (!ts) {
          wp = R0.wait_off[wk];
          we = R0.wait_off[wk + 1];
        }
      }
      WaitCache wc;
      wc.reset();
      uint32_t q = 0;  // this worker's tile count (wait-warp slot = q % kAhead)
      walk([&](const RankArgs& R, int grp, int k, const KSpan sp) {
        if constexpr (kWaitWarp) {
          const int j = int(q % kAhead);
          mbar_wait(&wrdy[j], (q / kAhead) & 1u);
          const bool waited = wwaited[j] != 0;
          mbar_arrive(&wfre[j]);
          ++q;
          if (waited) fence_proxy_async_global();  // generic-proxy acquire -> TMA reads
        } else if constexpr (MODE == MODE_AG) {
          bool waited = false;
          if (ts) {
            const int64_t r0 = int64_t(R.order[k] / R.n_nb) * BM;
            const uint64_t tw = args.trace ? globaltimer() : 0;
            waited = ts_wait_ag(R, args, wc, grp, lcta, r0, r0 + BM < M ? r0 + BM : M);
            if (waited) trace_event(args, TR_WAIT, R.rank, lcta, int(r0 / R.crows), tw);
          }
          while (!ts && wp < we && R.waits[wp].x == k) {
            const int g = R.waits[wp].y;
            const uint64_t tw = args.trace ? globaltimer() : 0;
            if (!(grp == 0 && wp == args.skip_wait)) {
              for (int s = 0; s < R.n_slices; ++s)
                spin_flag(R.flags + g * R.n_slices + s, R.epoch, args, R.rank, lcta, g);
            }
            trace_event(args, TR_WAIT, R.rank, lcta, g, tw);
            ++wp;
            waited = true;
          }
          if (waited) fence_proxy_async_global();  // generic-proxy arrivals -> TMA reads
        }
        const uint64_t t_load = args.trace ? globaltimer() : 0;
        const int2 tmn = tile_of(R, grp, k);
        const int mb = tmn.x, nb = tmn.y;
        const int t = mb * R.n_nb + nb;
        const CUtensorMap* mA = &R.tmA;
        int arow = mb * BM + int(crk) * kSubM;
        if constexpr (MODE == MODE_AG) {
          if (int64_t(arow) / S == R.rank) {
            mA = &R.tmA_loc;
            arow -= int(R.rank * S);
          }
        }
        // B rows of this CTA: its pair half (BN/2 rows); CG == 4: the quarter it loads and
        // multicasts to the same-position CTA of both pairs (the other quarter arrives from
        // the other pair), stacked in smem so each CTA sees its BN/2 rows contiguously
        const int brow = nb * BN + int(crank) * (BN / CGM) + int(pp) * (BN / CG);
        const uint32_t boff = pp * uint32_t(BN / CG) * 128u;
        const uint16_t bmask = uint16_t((1u << crank) | (1u << (crank + 2)));
        const int kb_lo = (MODE == MODE_AG || MODE == MODE_GEMM) ? sp.kb0 : 0;
        const int kb_hi = (MODE == MODE_AG || MODE == MODE_GEMM) ? sp.kb1 : nkb;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (CG == 4) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C_::kStage);
            tma_load_2d_2sm(sA + stage * C_::kStageA, mA, &full[stage], kb * kBK, arow, pol_a);
            tma_load_2d_2sm_mc(sB + stage * C_::kStageB + boff, &R.tmB, &full[stage], kb * kBK, brow, bmask, pol_b);
          } else if constexpr (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C_::kStage);
            tma_load_2d_2sm(sA + stage * C_::kStageA, mA, &full[stage], kb * kBK, arow, pol_a);
            tma_load_2d_2sm(sB + stage * C_::kStageB, &R.tmB, &full[stage], kb * kBK, brow, pol_b);
          } else {
            mbar_arrive_expect_tx(&full[stage], C_::kStage);
            tma_load_2d(sA + stage * C_::kStageA, mA, &full[stage], kb * kBK, arow, pol_a);
            tma_load_2d(sB + stage * C_::kStageB, &R.tmB, &full[stage], kb * kBK, brow, pol_b);
          }
          if (++stage == C_::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (MODE == MODE_RS) {
          // RS-4: an own tile's epilogue fuses the peer reduction; stream the W-1 peer
          // partials of this CTA's 128 rows through the same smem ring (32-column fp32
          // boxes) once the peers' flags for its chunks are released.
          const int64_t sub0 = int64_t(mb) * BM + int64_t(crk) * kSubM;
          if (R.W > 1 && !R.rs_atomic && sub0 / S == R.rank) {
            const uint64_t tw = args.trace ? globaltimer() : 0;
            if (ts) {
              const int64_t r0 = int64_t(mb) * BM;
              ts_wait_rs(R, args, wc, grp, lcta, r0, r0 + BM < M ? r0 + BM : M);
            }
            while (!ts && wp < we && R.waits[wp].x == k) {
              const int g = R.waits[wp].y;
              if (!(grp == 0 && wp == args.skip_wait)) {
                for (int s = 0; s < R.W; ++s)
                  if (s != R.rank) spin_flag(R.flags + g * R.W + s, R.epoch, args, R.rank, lcta, g);
              }
              ++wp;
            }
            fence_proxy_async_global();  // peers' generic-proxy stores -> TMA reads
            trace_event(args, TR_REDWAIT, R.rank, lcta, t, tw);
            const int lr0 = int(sub0 - int64_t(R.rank) * S);
            const int nvb = rs_blocks<BN>(nb, N);
            for (int cb = 0; cb < nvb; ++cb) {
              for (int s = 0; s < R.W; ++s) {
                if (s == R.rank) continue;
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&pfull[stage], kSubM * 128);  // own CTA's barrier
                tma_load_2d(sA + stage * C_::kStageA, &R.tmA_loc, &pfull[stage], nb * BN + cb * 32,
                            int(s * S) + lr0, pol_b);
                if (++stage == C_::kStages) {
                  stage = 0;
                  phase ^= 1;
                }
              }
            }
          }
        }
        trace_event(args, TR_LOAD, R.rank, lcta, t, t_load);
      });
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (leader) {
      constexpr uint32_t idesc = make_idesc_bf16(kSubM * CGM, BN);  // one pair's MMA: M = 128 * cta_group
      // full[] completes only on operand uses of a slot (RS partial stages use pfull[]),
      // so its parity is tracked per slot.
      uint32_t stage = 0, fpar = 0, acc = 0, acc_phase = 0;
      walk([&](const RankArgs& R, int grp, int k, const KSpan sp) {
        const uint64_t t_mma = args.trace ? globaltimer() : 0;
        const long long c_mma = args.trace ? clock64() : 0;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb_lo = (MODE == MODE_AG || MODE == MODE_GEMM) ? sp.kb0 : 0;
        const int kb_hi = (MODE == MODE_AG || MODE == MODE_GEMM) ? sp.kb1 : nkb;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], (fpar >> stage) & 1u);
          fpar ^= 1u << stage;
          tc_fence_after();
          if (lane == 0) {
            const uint64_t ad = make_smem_desc_sw128(smem_u32(sA + stage * C_::kStageA));
            const uint64_t bd = make_smem_desc_sw128(smem_u32(sB + stage * C_::kStageB));
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {  // +32 B per K=16 step inside the swizzle atom
              if constexpr (CG >= 2)
                mma_bf16_ss_cg2(d_tmem, ad + uint64_t(kk * 2), bd + uint64_t(kk * 2), idesc,
                                (kb != kb_lo || kk != 0) ? 1u : 0u);
              else
                mma_bf16_ss(d_tmem, ad + uint64_t(kk * 2), bd + uint64_t(kk * 2), idesc,
                            (kb != kb_lo || kk != 0) ? 1u : 0u);
            }
            // the stage is free once this pair's MMAs read it -- in every CTA that holds
            // operands of this pair (CG == 4: also the other pair's CTAs, whose B quarters
            // were multicast here)
            if constexpr (CG == 4)
              mma_commit_cg2_mask(&empty[stage], uint16_t(0xF));
            else if constexpr (CG == 2)
              mma_commit_cg2_mc(&empty[stage]);
            else
              mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C_::kStages) stage = 0;
        }
        if (lane == 0) {
          if constexpr (CG >= 2)
            mma_commit_cg2_mask(&tfull[acc], uint16_t(3u << (2 * pp)));  // this pair's CTAs
          else
            mma_commit(&tfull[acc]);
          if (args.trace) {
            const int2 tmn = tile_of(R, grp, k);
            trace_event(args, TR_MMA, R.rank, lcta, tmn.x * R.n_nb + tmn.y, t_mma);
            trace_event(args, TR_CLK, R.rank, lcta, int(clock64() - c_mma), t_mma);
          }
        }
        __syncwarp();
        if constexpr (MODE == MODE_RS) {  // ring stages carrying peer partials belong to the epilogue
          const int t = R.order[k];
          const int mb = t / R.n_nb;
          if (R.W > 1 && !R.rs_atomic && (int64_t(mb) * BM) / S == R.rank) {
            const int skip = rs_blocks<BN>(t - mb * R.n_nb, N) * (R.W - 1);
            stage = (stage + uint32_t(skip)) % C_::kStages;
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      });
    }
  } else if (warp < Roles<MODE>::kCommWarp0) {
    // ================================================================ epilogue
    // TMEM -> registers -> per-warp smem transpose -> coalesced 128-byte row segments.
    // AG/GEMM: bf16 C rows (64 columns per step).  RS: fp32 partial rows into the owner's
    // slot (32 columns per step; a peer address over NVLink, local in loopback).
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int etid = threadIdx.x - 64;
    constexpr int kEpiW = Roles<MODE>::kEpiW;
    constexpr int kEpiT = 32 * kEpiW;  // epilogue threads (named barrier 1)
    // RS: warps 2-5 take columns [0, BN/2) of the tile, warps 6-9 [BN/2, BN)
    const int half = (warp - 2) / 4;
    const int c_lo = kEpiW == 8 ? half * (BN / 2) : 0, c_hi = kEpiW == 8 ? c_lo + BN / 2 : BN;
    uint4* stg = reinterpret_cast<uint4*>(smem + L.off_stg + (warp - 2) * kStageWarpBytes);
    constexpr int CW = (MODE == MODE_RS) ? 32 : 64;  // columns per staging step (128 B per row)
    constexpr int EPS = (MODE == MODE_RS) ? 4 : 8;   // elements per 16-byte lane segment
    constexpr int EB = (MODE == MODE_RS) ? 4 : 2;    // bytes per output element
    uint32_t acc = 0, acc_phase = 0;
    uint32_t rs_stage = 0, ppar = 0;  // RS: replay of the producer's ring position, pfull parities
    int wp_e = 0, we_e = 0;           // RS ATOMIC: the epilogue walks the own-tile waits itself
    if constexpr (MODE == MODE_RS) {
      if (!ts) {
        wp_e = R0.wait_off[wk];
        we_e = R0.wait_off[wk + 1];
      }
    }
    WaitCache wc;
    if (etid == 0) wc.reset();
    walk([&](const RankArgs& R, int grp, int k, const KSpan sp) {
      const int2 tmn = tile_of(R, grp, k);
      const int mb = tmn.x, nb = tmn.y;
      const int t = mb * R.n_nb + nb;
      // rows past the end of the output are not stored (A2A: the received rows R_e)
      int64_t rlim = M;
      if constexpr (MODE == MODE_A2A) rlim = a2s.rows[grp];
      if constexpr (MODE == MODE_RS)  // operand stages of this tile (consumed by the MMA)
        rs_stage = (rs_stage + uint32_t(nkb)) % C_::kStages;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint64_t t_epi = args.trace ? globaltimer() : 0;
      const uint32_t tb = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
      const int64_t col_base = int64_t(nb) * BN;
      const int64_t sub0 = int64_t(mb) * BM + int64_t(crk) * kSubM;  // first row of this CTA's 128
      const int64_t row0 = sub0 + q * 32;                                // first row of this warp
      int owner = 0;
      bool own_tile = false;
      char* dst_base;  // byte address of (row0, col 0) of the destination matrix
      const int64_t ld_bytes = N * EB;
      if constexpr (MODE == MODE_RS) {
        owner = int(sub0 / S);
        own_tile = owner == R.rank;
        dst_base = R.rs_atomic ? R.peer_acc[owner] + (row0 - int64_t(owner) * S) * ld_bytes  // reduce-add target
                               : R.peer_data[owner] + (int64_t(R.rank) * S + (row0 - int64_t(owner) * S)) * ld_bytes;
      } else {
        dst_base = reinterpret_cast<char*>(R.C) + row0 * ld_bytes;
      }
      if constexpr (MODE == MODE_RS) {
        if (own_tile && R.rs_atomic) {
          // RS-4, ATOMIC: the peers reduce-added their partials into this rank's
          // accumulator; wait for their chunk flags, then add the accumulator to the TMEM
          // tile with coalesced loads (own value staged through smem so lane l owns rows
          // i*4 + l/8, columns 4*(l%8)..+3), store bf16, and re-arm the accumulator (zeros).
          if (etid == 0) {
            const uint64_t tw = args.trace ? globaltimer() : 0;
            if (ts && !xp(args, 4)) {
              const int64_t r0 = int64_t(mb) * BM;
              ts_wait_rs(R, args, wc, grp, lcta, r0, r0 + BM < M ? r0 + BM : M);
            }
            while (!ts && wp_e < we_e && R.waits[wp_e].x <= k) {
              const int g = R.waits[wp_e].y;
              if (!(grp == 0 && wp_e == args.skip_wait) && !xp(args, 4)) {
                for (int s = 0; s < R.W; ++s)
                  if (s != R.rank) spin_flag(R.flags + g * R.W + s, R.epoch, args, R.rank, lcta, g);
              }
              ++wp_e;
            }
            trace_event(args, TR_REDWAIT, R.rank, lcta, t, tw);
          }
          named_bar_sync(1, kEpiT);
          const int64_t lrow0 = row0 - int64_t(R.rank) * S;  // this warp's first row in C_shard
          float* accm = reinterpret_cast<float*>(R.peer_acc[R.rank]);
          __nv_bfloat16* cout = reinterpret_cast<__nv_bfloat16*>(R.C);
          const int c = lane & 7;
          float4 pa[8];
          auto load_acc = [&](int64_t col0, float4 (&dst)[8]) {
            const bool okl = col0 < N && col0 + 4 * c < N;
            const int64_t off = (lrow0 + (lane >> 3)) * N + col0 + 4 * c;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (!okl || xp(args, 2)) {
                dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
              } else if (R.rs_bf16) {  // bf16 wire: a bf16 accumulator [S, N]
                const uint2 b = __ldcg(reinterpret_cast<const uint2*>(
                    reinterpret_cast<const __nv_bfloat16*>(accm) + off + int64_t(i) * 4 * N));
                dst[i] = make_float4(__uint_as_float(b.x << 16), __uint_as_float(b.x & 0xffff0000u),
                                     __uint_as_float(b.y << 16), __uint_as_float(b.y & 0xffff0000u));
              } else {
                dst[i] = __ldcg(reinterpret_cast<const float4*>(accm + off + int64_t(i) * 4 * N));
              }
            }
          };
#pragma unroll 1
          for (int cc = c_lo; cc < c_hi; cc += 32) {
            const int64_t col0 = col_base + cc;
            if (col0 >= N) break;  // warp-uniform
            load_acc(col0, pa);  // in flight while the TMEM block is read and staged
            uint32_t v[32];
            tmem_ld_32x32b_x32(tb + cc, v);
            tmem_wait_ld();
            if (nkb == 0) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0u;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              stg[lane * 8 + (j ^ (lane & 7))] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __syncwarp();
            const bool ok = col0 + 4 * c < N;
            const int64_t base_off = (lrow0 + (lane >> 3)) * N + col0 + 4 * c;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rr = i * 4 + (lane >> 3);
              const uint4 w = stg[rr * 8 + (c ^ (rr & 7))];
              const float4 x = make_float4(pa[i].x + __uint_as_float(w.x), pa[i].y + __uint_as_float(w.y),
                                           pa[i].z + __uint_as_float(w.z), pa[i].w + __uint_as_float(w.w));
              if (ok) {
                uint2 o;
                o.x = pack_bf16x2(x.x, x.y);
                o.y = pack_bf16x2(x.z, x.w);
                *reinterpret_cast<uint2*>(cout + base_off + int64_t(i) * 4 * N) = o;
                if (R.ar)  // GEMM-AR: the reduced rows peers gather
                  *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(R.ar_red) + base_off + int64_t(i) * 4 * N) = o;
                if (xp(args, 1)) {
                } else if (R.rs_bf16) {
                  *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(accm) + base_off + int64_t(i) * 4 * N) =
                      make_uint2(0u, 0u);
                } else {
                  st_v4(reinterpret_cast<int4*>(accm + base_off + int64_t(i) * 4 * N), make_int4(0, 0, 0, 0));
                }
              }
            }
            __syncwarp();
          }
        } else if (own_tile && half == 0) {
          // (slots: the four warps of half 0 take every column -- the peer boxes stream
          // through the operand ring in one order; named barrier 2 = those 128 threads)
          // RS-4 fused reduction: the peer partials arrive as 32-column fp32 boxes in the
          // smem ring (streamed by the producer); thread = row, like the TMEM accumulator.
          // Sum in ascending source rank, own TMEM value at s == rank, store bf16.
          const int r = q * 32 + lane;  // row inside this CTA's 128-row half
          const int nvb = rs_blocks<BN>(nb, N);
          char* crow0 = reinterpret_cast<char*>(R.C) + (row0 - int64_t(R.rank) * S) * N * 2;
#pragma unroll 1
          for (int cb = 0; cb < nvb; ++cb) {
            float acc[32];
            const int nterms = R.W;  // ascending source rank; own TMEM value at s == rank
            const int own_term = R.rank;
            for (int s = 0; s < nterms; ++s) {
              if (s == own_term) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tb + cb * 32, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const float x = nkb ? __uint_as_float(v[i]) : 0.f;
                  acc[i] = s == 0 ? x : acc[i] + x;
                }
              } else {
                mbar_wait(&pfull[rs_stage], (ppar >> rs_stage) & 1u);
                ppar ^= 1u << rs_stage;
                const uint4* box = reinterpret_cast<const uint4*>(sA + rs_stage * C_::kStageA);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const uint4 w = box[r * 8 + (j ^ (r & 7))];  // TMA 128-B swizzle
                  const float x0 = __uint_as_float(w.x), x1 = __uint_as_float(w.y), x2 = __uint_as_float(w.z),
                              x3 = __uint_as_float(w.w);
                  acc[4 * j] = s == 0 ? x0 : acc[4 * j] + x0;
                  acc[4 * j + 1] = s == 0 ? x1 : acc[4 * j + 1] + x1;
                  acc[4 * j + 2] = s == 0 ? x2 : acc[4 * j + 2] + x2;
                  acc[4 * j + 3] = s == 0 ? x3 : acc[4 * j + 3] + x3;
                }
                named_bar_sync(2, 128);  // every half-0 epilogue thread has read the stage
                if (etid == 0) mbar_arrive(&empty[rs_stage]);
                if (++rs_stage == C_::kStages) rs_stage = 0;
              }
            }
            // bf16 pack, stage row `lane` (64 B) through the transpose buffer, store
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 w = make_uint4(pack_bf16x2(acc[8 * j], acc[8 * j + 1]), pack_bf16x2(acc[8 * j + 2], acc[8 * j + 3]),
                                         pack_bf16x2(acc[8 * j + 4], acc[8 * j + 5]),
                                         pack_bf16x2(acc[8 * j + 6], acc[8 * j + 7]));
              stg[lane * 4 + (j ^ ((lane >> 1) & 3))] = w;
            }
            __syncwarp();
            const int64_t col0 = col_base + cb * 32;
            const int c = lane & 3;
            const bool ok = col0 + 8 * c < N;
            char* colp = crow0 + (col0 + 8 * c) * 2;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int rr = i * 8 + (lane >> 2);
              const uint4 w = stg[rr * 4 + (c ^ ((rr >> 1) & 3))];
              if (ok) {
                st_v4(reinterpret_cast<int4*>(colp + rr * N * 2), make_int4(w.x, w.y, w.z, w.w));
                if (R.ar)  // GEMM-AR: the reduced rows peers gather
                  st_v4(reinterpret_cast<int4*>(colp - reinterpret_cast<char*>(R.C) + R.ar_red + rr * N * 2),
                        make_int4(w.x, w.y, w.z, w.w));
              }
            }
            __syncwarp();
          }
        }
      }
      // stream-K (Q28): this CTA's partial slot of a split tile position
      float4* sk_part = nullptr;
      uint32_t* sk_flag = nullptr;
      if constexpr (MODE == MODE_AG || MODE == MODE_GEMM) {
        if (sp.role != 0) {
          const int slot = (k - R.sk_dp) * CG + int(crk);
          sk_part = reinterpret_cast<float4*>(R.sk_ws) + int64_t(slot) * ((BN + 31) / 32) * 128 * 8;
          sk_flag = R.sk_flags + slot;
          if (sp.role == 2) {  // head piece: the tail piece (the next worker's first) must have landed
            if (etid == 0) spin_flag(sk_flag, R.sk_seq, args, R.rank, lcta, -2);
            named_bar_sync(1, kEpiT);
          }
        }
      }
      if (!own_tile) {
      // RS ATOMIC: the TMA unit reduce-adds each staged 32 x 32 fp32 box into the owner's
      // accumulator (two staging buffers per warp, so staging overlaps the previous reduce).
      const bool tma_red = MODE == MODE_RS && R.rs_atomic && !xp(args, 64);  // exp 64: thread red.add
      int sb = 0;
      if constexpr (MODE == MODE_AG || MODE == MODE_GEMM) {
        if (sk_part != nullptr) {
          // stream-K piece (Q28), 32 fp32 columns per step through the transpose buffer, so
          // the partial moves in coalesced 512-byte warp accesses: lane l handles rows
          // i*4 + l/8, columns 4*(l%8)..+3 of the warp's 32 x 32 block.  Tail piece: store the
          // partial ([cb][128 rows][32] fp32).  Head piece: add it, store bf16 C.
          const int c = lane & 7;
#pragma unroll 1
          for (int cb = 0; cb < (BN + 31) / 32; ++cb) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tb + cb * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              stg[lane * 8 + (j ^ (lane & 7))] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __syncwarp();
            float4* wsb = sk_part + (int64_t(cb) * 128 + q * 32) * 8;  // this warp's 32 rows of block cb
            if (sp.role == 1) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rr = i * 4 + (lane >> 3);
                const uint4 w = stg[rr * 8 + (c ^ (rr & 7))];
                __stcg(wsb + rr * 8 + c, make_float4(__uint_as_float(w.x), __uint_as_float(w.y), __uint_as_float(w.z),
                                                     __uint_as_float(w.w)));
              }
            } else {
              float4 a[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) a[i] = __ldcg(wsb + (i * 4 + (lane >> 3)) * 8 + c);
              const int64_t col = col_base + cb * 32 + 4 * c;
              const bool ok = col < N && cb * 32 + 4 * c < BN;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rr = i * 4 + (lane >> 3);
                const uint4 w = stg[rr * 8 + (c ^ (rr & 7))];
                if (ok && row0 + rr < rlim) {
                  uint2 o;
                  o.x = pack_bf16x2(__uint_as_float(w.x) + a[i].x, __uint_as_float(w.y) + a[i].y);
                  o.y = pack_bf16x2(__uint_as_float(w.z) + a[i].z, __uint_as_float(w.w) + a[i].w);
                  *reinterpret_cast<uint2*>(dst_base + rr * ld_bytes + col * EB) = o;
                }
              }
            }
            __syncwarp();
          }
        }
      }
#pragma unroll 1
      for (int cc = c_lo; cc < ((MODE == MODE_AG || MODE == MODE_GEMM) && sk_part != nullptr ? 0 : c_hi); cc += CW) {
        uint32_t v[32];
        if constexpr (MODE == MODE_RS) {
          tmem_ld_32x32b_x32(tb + cc, v);
          tmem_wait_ld();
        } else {
          uint32_t lo[32], hi[32];
          tmem_ld_32x32b_x32(tb + cc, lo);
          tmem_ld_32x32b_x32(tb + cc + 32, hi);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            v[i] = pack_bf16x2(__uint_as_float(lo[2 * i]), __uint_as_float(lo[2 * i + 1]));
            v[16 + i] = pack_bf16x2(__uint_as_float(hi[2 * i]), __uint_as_float(hi[2 * i + 1]));
          }
        }
        if (nkb == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        const int64_t col0 = col_base + cc;
        if (col0 >= N) break;  // warp-uniform
        if (tma_red && R.rs_bf16) {
          // bf16 wire (Q14, non-conforming): 64 columns per step as bf16 pairs, one 32 x 64
          // bf16 box reduce-added into the owner's bf16 accumulator; the next block of 32
          // columns is consumed here too (cc advances by 64)
          if ((cc - c_lo) & 32) continue;
          uint32_t hi[32];
          tmem_ld_32x32b_x32(tb + cc + 32, hi);
          tmem_wait_ld();
          if (nkb == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) hi[i] = 0u;
          }
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
            pk[16 + i] = pack_bf16x2(__uint_as_float(hi[2 * i]), __uint_as_float(hi[2 * i + 1]));
          }
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            stg[lane * 8 + (j ^ (lane & 7))] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_reduce_add_2d(&R.tmAcc[owner], stg, int(col0), int(row0 - int64_t(owner) * S));
            bulk_commit();
          }
          continue;
        }
        if (tma_red) {
          uint4* sg = stg + sb * (kEpiW * kStageWarpBytes / 16);
          if (lane == 0) bulk_wait_read<kRsStg - 1>();  // the reduce that last read buffer sb is done reading
          __syncwarp();
          // the TMA 128-B swizzle of a 1024-B-aligned box: 16-B chunk j of row r at j ^ (r & 7)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            sg[lane * 8 + (j ^ (lane & 7))] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          if (!xp(args, 8192)) fence_proxy_async_smem();  // generic smem writes -> async proxy (TMA) reads
          __syncwarp();
          if (lane == 0 && !(xp(args, 1024) && ((cc / CW) & 1)) && !xp(args, 16384)) {  // exp 1024/16384: half / no reduces (timing only)
            if (xp(args, 256))  // timing experiment: keep the accumulator lines in L2
              tma_reduce_add_2d_hint(&R.tmAcc[owner], sg, int(col0), int(row0 - int64_t(owner) * S),
                                     policy_evict_last());
            else
              tma_reduce_add_2d(&R.tmAcc[owner], sg, int(col0), int(row0 - int64_t(owner) * S));
          }
          if (lane == 0) bulk_commit();
          sb = (sb + 1) % kRsStg;
          continue;
        }
        // stage row `lane` (128 B) with a 16-byte XOR swizzle (conflict-free both ways)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          stg[lane * 8 + (j ^ (lane & 7))] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __syncwarp();
        const int c = lane & 7;
        // N % 8 == 0: a segment is all-valid or all-out; columns past this tile's BN (a
        // BN that is not a multiple of the step) belong to the next tile and are not stored
        const bool ok = col0 + c * EPS < N && (BN % CW == 0 || cc + c * EPS < BN);
        char* colp = dst_base + (col0 + c * EPS) * EB;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + (lane >> 3);
          const uint4 w = stg[r * 8 + (c ^ (r & 7))];
          if (ok && !xp(args, 16) && row0 + r < rlim) {
            if (MODE == MODE_RS && R.rs_atomic && !xp(args, 8))
              red_add_v4_f32(colp + r * ld_bytes, w.x, w.y, w.z, w.w);
            else
              st_v4(reinterpret_cast<int4*>(colp + r * ld_bytes), make_int4(w.x, w.y, w.z, w.w));
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG >= 2)
          mbar_arrive_leader(&tempty[acc]);
        else
          mbar_arrive(&tempty[acc]);
      }
      if (tma_red) {
        // RS-3 after the reduces are performed (the TMEM buffer is already released).
        // Deferring this to the next tile was measured slower: the owners' own tiles wait
        // on these signals.
        if (lane == 0) {
          bulk_wait<0>();              // this warp's reduces performed
          fence_proxy_async_global();  // async-proxy writes -> the generic release below
        }
        __syncwarp();
        named_bar_sync(1, kEpiT);
        if (etid == 0) rs_signal(R, args, sub0, owner);
      }
      }
      if (own_tile) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG >= 2)
            mbar_arrive_leader(&tempty[acc]);
          else
            mbar_arrive(&tempty[acc]);
        }
      }
      if ((MODE == MODE_AG || MODE == MODE_GEMM) && sp.role == 1) {
        // stream-K tail piece: every epilogue thread's partial stores precede the CTA-scope
        // barrier; the release (cumulative) publishes them to the head piece's CTA
        named_bar_sync(1, kEpiT);
        if (etid == 0) st_release_gpu(sk_flag, R.sk_seq);
      }
      if (MODE == MODE_RS && !own_tile && !(R.rs_atomic && !xp(args, 64))) {
        // RS-3 (stores / thread reduces): signal this sub-tile now.
        named_bar_sync(1, kEpiT);
        if (etid == 0) rs_signal(R, args, sub0, owner);
      }
      if (MODE == MODE_RS && own_tile && R.ar && R.W > 1) {
        // GEMM-AR: count this own sub-tile into its chunks; the last one releases the
        // owner's "reduced" flag of chunk g (word n_chunks*W + g), which peers' gather
        // warps acquire before pulling the rows (Fig.4d).
        named_bar_sync(1, kEpiT);
        if (etid == 0) {  // (release below is cumulative over the CTA's stores, as in rs_signal)
          const int glo = int(sub0 / R.crows);
          const int ghi = int((sub0 + kSubM - 1) / R.crows);
          for (int g = glo; g <= ghi; ++g) {
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(R.counters + g) : "memory");
            if (int(old) + 1 == R.tiles_per_chunk[g]) {
              R.counters[g] = 0;
              st_release_sys(R.flags + R.n_chunks * R.W + g, R.epoch);
            }
          }
        }
      }
      if (etid == 0) trace_event(args, TR_EPI, R.rank, lcta, t, t_epi);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  } else {
    // ================================================================ co-located comm warps
    if constexpr (kWaitWarp) {
      if (warp == Roles<MODE>::kCommWarp0 && lane == 0) {
        WaitCache wc;
        wc.reset();
        int wp = (ts || MODE == MODE_A2A) ? 0 : R0.wait_off[wk];
        int we = (ts || MODE == MODE_A2A) ? 0 : R0.wait_off[wk + 1];
        uint32_t q = 0;
        walk([&](const RankArgs& R, int grp, int k, const KSpan sp) {
          const int j = int(q % kAhead);
          mbar_wait(&wfre[j], ((q / kAhead) & 1u) ^ 1u);
          bool waited = false;
          if constexpr (MODE == MODE_A2A) {
            // the (source, chunk) blocks of this tile's received rows
            const int r0 = a2a_tile(a2s, R, grp, k).x * BM;
            const uint64_t tw = args.trace ? globaltimer() : 0;
            // debug mutation: CTA 0 of rank group 0 skips the waits of its skip_wait-th tile
            if (!(args.skip_wait >= 0 && blockIdx.x == 0 && grp == 0 && int(q) == args.skip_wait))
              waited = a2a_wait(a2s, R, args, wc, grp, lcta, r0, min(a2s.rows[grp], r0 + BM));
            if (waited) trace_event(args, TR_WAIT, R.rank, lcta, r0 / BM, tw);
          } else if (ts) {
            const int64_t r0 = int64_t(R.order[k] / R.n_nb) * BM;
            const uint64_t tw = args.trace ? globaltimer() : 0;
            waited = ts_wait_ag(R, args, wc, grp, lcta, r0, r0 + BM < M ? r0 + BM : M);
            if (waited) trace_event(args, TR_WAIT, R.rank, lcta, int(r0 / R.crows), tw);
          }
          while (!ts && wp < we && R.waits[wp].x == k) {
            const int g = R.waits[wp].y;
            const uint64_t tw = args.trace ? globaltimer() : 0;
            if (!(grp == 0 && wp == args.skip_wait)) {
              for (int s = 0; s < R.n_slices; ++s)
                spin_flag(R.flags + g * R.n_slices + s, R.epoch, args, R.rank, lcta, g);
            }
            trace_event(args, TR_WAIT, R.rank, lcta, g, tw);
            ++wp;
            waited = true;
          }
          wwaited[j] = waited ? 1 : 0;
          mbar_arrive(&wrdy[j]);  // release.cta: the acquired flags -> the producer
          ++q;
        });
      }
    }
    if constexpr (MODE == MODE_A2A) {
      // A2A dispatch: warp 7 of every GEMM CTA pushes (source, expert, chunk) row gathers.
      // Space-sliced: this rank's rows, destinations in the push rotation (own rows first,
      // then e = s+1, s+2, ...).  Time-sliced: every rank's rows, destination-major in the
      // order the experts' tiles run.
      if (warp == Roles<MODE>::kCommWarp0 + 1) {
        const int W = R0.W;
        const int nw = ts ? int(gridDim.x) : args.ctas_per_rank;
        const int w = ts ? int(blockIdx.x) : lcta;
        const int gs0 = ts ? 0 : grp, gs1 = ts ? args.n_group : grp + 1;
        int it = 0;
        uint32_t par = 0;
        for (int ei = 0; ei < W; ++ei) {
          for (int gs = gs0; gs < gs1; ++gs) {
            const RankArgs& S_ = args.rk[gs];
            const int e = ts ? args.rk[ei].rank : (S_.rank + ei) % W;
            const int nj = (a2s.tab[S_.rank][e] + S_.crows - 1) / S_.crows;
            for (int jj = 0; jj < nj; ++jj, ++it) {
              if (it % nw != w) continue;
              if (xp(args, 4096)) {  // timing experiment: 16-byte ld/st row copies
                a2a_push_chunk(a2s, S_, args, e, jj);
              } else {
                if (lane == 0) a2a_push_chunk_tma(a2s, S_, args, e, jj, smem + L.off_comm, commbars, par);
                __syncwarp();
              }
            }
          }
        }
      }
    }
    const RankArgs& R = R0;
    if constexpr (MODE == MODE_RS) {
      if (R.ar && R.n_comm_items > 0) {  // GEMM-AR gather: ld/st pulls of reduced chunks
        const int cw = warp - Roles<MODE>::kCommWarp0;
        // 16 KB of loads in flight per warp (the RS kernel's register budget has room; at 4 KB
        // the gather was latency-bound well below the copy bandwidth)
        if (ts)  // every rank's pulls, owner after owner (the order the owners' reductions finish)
          comm_worker_ts<COMM_LDST, kArPullU>(args, int(blockIdx.x) * kColocCommWarps + cw,
                                              int(gridDim.x) * kColocCommWarps, nullptr, 0, nullptr);
        else
          comm_worker<COMM_LDST, kArPullU>(R, args, lcta * kColocCommWarps + cw, args.ctas_per_rank * kColocCommWarps,
                                           nullptr, 0, nullptr);
      }
    }
    if constexpr (MODE == MODE_AG && COMM != COMM_NONE) {
      if (args.comm_ctas_per_rank == 0) {
        const int cw = warp - Roles<MODE>::kCommWarp0;
        if (ts)
          comm_worker_ts<COMM>(args, int(blockIdx.x) * kColocCommWarps + cw, int(gridDim.x) * kColocCommWarps,
                               smem + L.off_comm + cw * kCommBufs * kColocBufBytes, kColocBufBytes,
                               commbars + cw * kCommBufs);
        else
          comm_worker<COMM>(R, args, lcta * kColocCommWarps + cw, args.ctas_per_rank * kColocCommWarps,
                            smem + L.off_comm + cw * kCommBufs * kColocBufBytes, kColocBufBytes,
                            commbars + cw * kCommBufs);
      }
    }
  }

  tc_fence_before();
  if constexpr (CG >= 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG >= 2)
      tmem_dealloc_cg2(tmem_base, C_::kTmemCols);
    else
      tmem_dealloc(tmem_base, C_::kTmemCols);
  }
}

}  // namespace dev

// ------------------------------------------------------------------------------- launcher
namespace {
template <int BN, int MODE, int COMM, int CG>
cudaError_t launch_one(const KernelArgs& args, cudaStream_t stream) {
  auto kern = dev::fused_kernel<BN, MODE, COMM, CG>;
  constexpr bool tma_comm = (MODE == MODE_AG && COMM == COMM_TMA);
  const size_t smem_gemm =
      dev::gemm_layout<BN, CG, MODE == MODE_A2A ? dev::kA2AOperandBudget
                                                : (MODE == MODE_RS ? dev::kRsOperandBudget : dev::kOperandBudget)>(
          tma_comm, MODE == MODE_RS, MODE == MODE_A2A).total;
  const size_t smem_comm = (MODE == MODE_AG && COMM != COMM_NONE) ? dev::comm_cta_layout().total : 0;
  const size_t smem = smem_gemm > smem_comm ? smem_gemm : smem_comm;
  static bool attr_set = false;
  static bool coop_ok = true;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((args.n_seg > 0 || args.a2a_ts) ? args.ctas_per_rank
                                    : args.n_group * (args.ctas_per_rank + args.comm_ctas_per_rank));
  cfg.blockDim = dim3(dev::Roles<MODE>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CG >= 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (CG == 1 && coop_ok) {
    // all CTAs co-resident (spin-waits, H3).  Cluster launches (CG == 2) rely on
    // grid <= SMs with one CTA per SM instead: ncu cannot replay cooperative cluster
    // launches, and the 2-CTA grid never exceeds the SM count.
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (CG == 4) {  // 4-CTA clusters need whole free GPC slots: not every SM can host one
    static int max_clusters = -1;
    if (max_clusters < 0) {
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
      if (oe != cudaSuccess) return oe;
    }
    if (int(cfg.gridDim.x) / 4 > max_clusters) return cudaErrorCooperativeLaunchTooLarge;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
  return e;
}

template <int BN, int MODE, int CG>
int max_clusters_of() {
  auto kern = dev::fused_kernel<BN, MODE, COMM_NONE, CG>;
  const size_t smem = dev::gemm_layout<BN, CG, MODE == MODE_RS ? dev::kRsOperandBudget : dev::kOperandBudget>(
                          false, MODE == MODE_RS, false).total;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return -1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(4 * 64);
  cfg.blockDim = dim3(dev::Roles<MODE>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = -1;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return -1;
  return n;
}

// Extra CTA-pair tile widths (Q19: wave-quantization-free tiles for the per-GPU
// TP shapes): plain GEMM and AG with copy-engine transfers only.
template <int BN>
cudaError_t launch_bn_pair_extra(const KernelArgs& args, int comm, cudaStream_t stream) {
  if (args.mode == MODE_GEMM) return launch_one<BN, MODE_GEMM, COMM_NONE, 2>(args, stream);
  if (args.mode == MODE_AG && comm == COMM_NONE) return launch_one<BN, MODE_AG, COMM_NONE, 2>(args, stream);
  return cudaErrorInvalidValue;
}

template <int BN, int CG>
cudaError_t launch_bn(const KernelArgs& args, int comm, cudaStream_t stream) {
  switch (args.mode) {
    case MODE_GEMM:
      return launch_one<BN, MODE_GEMM, COMM_NONE, CG>(args, stream);
    case MODE_RS:
      return launch_one<BN, MODE_RS, COMM_NONE, CG>(args, stream);
    case MODE_A2A:
      return launch_one<BN, MODE_A2A, COMM_NONE, CG>(args, stream);
    case MODE_AG:
      if (comm == COMM_TMA) return launch_one<BN, MODE_AG, COMM_TMA, CG>(args, stream);
      if (comm == COMM_LDST) return launch_one<BN, MODE_AG, COMM_LDST, CG>(args, stream);
      return launch_one<BN, MODE_AG, COMM_NONE, CG>(args, stream);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

int max_co_resident_ctas(int cg) {
  // co-resident CTAs (1 per SM) of the fused kernel in clusters of `cg` CTAs
  const int a = cg == 4 ? max_clusters_of<256, MODE_RS, 4>() : max_clusters_of<256, MODE_RS, 2>();
  const int b = cg == 4 ? max_clusters_of<256, MODE_AG, 4>() : max_clusters_of<256, MODE_AG, 2>();
  return (a < 0 || b < 0) ? -1 : cg * (a < b ? a : b);
}

cudaError_t launch_fused(const KernelArgs& args, int bn, int cg, int comm, cudaStream_t stream) {
  if (cg == 2) {
    switch (bn) {
      case 256: return launch_bn<256, 2>(args, comm, stream);
      case 128: return launch_bn<128, 2>(args, comm, stream);
      case 224: return launch_bn_pair_extra<224>(args, comm, stream);
      case 208: return launch_bn_pair_extra<208>(args, comm, stream);
      case 192: return launch_bn_pair_extra<192>(args, comm, stream);
      case 160: return launch_bn_pair_extra<160>(args, comm, stream);
      case 144: return launch_bn_pair_extra<144>(args, comm, stream);
      case 112: return launch_bn_pair_extra<112>(args, comm, stream);
    }
  } else if (cg == 4) {  // two CTA pairs sharing B (multicast): GEMM, AG (copy engine), RS (atomic)
    if (bn == 256) {
      if (args.mode == MODE_GEMM) return launch_one<256, MODE_GEMM, COMM_NONE, 4>(args, stream);
      if (args.mode == MODE_AG && comm == COMM_NONE) return launch_one<256, MODE_AG, COMM_NONE, 4>(args, stream);
      if (args.mode == MODE_RS) return launch_one<256, MODE_RS, COMM_NONE, 4>(args, stream);
    }
  } else {
    if (bn == 256) return launch_bn<256, 1>(args, comm, stream);
    if (bn == 128) return launch_bn<128, 1>(args, comm, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ao
