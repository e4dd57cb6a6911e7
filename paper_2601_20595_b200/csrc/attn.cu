// attn.cu -- sequence-parallel attention with all-gathered KV (
// PAPER.md P:459 "sequence-parallel (SP) schedules, including the overlapped
// RingAttention", Fig.4(c) ring AllGather P:310).
//
// Rank r computes O_r[h] = softmax(Q_r[h] K[h]^T / sqrt(128)) V[h] over the whole sequence.
// The peers' K/V shards arrive chunk by chunk (copy-engine pushes in the ring rotation,
// per-chunk flags); every query tile consumes its KV blocks in ARRIVAL order -- own shard
// first, then ranks r-1, r-2, ... -- which the online softmax makes order-free: the
// RingAttention schedule expressed as the paper's chunk-ordered tile loop.
//
// Persistent kernel, 1 CTA / SM, one work item = (head, 128 query rows), FlashAttention-
// style with tcgen05 (5th-gen tensor cores):
//   warp 0      TMA producer: Q tile once per item, K+V blocks into a 2-stage ring
//   warp 1      MMA issuer: S = Q K^T into TMEM (two S buffers), O += P V into TMEM
//               (P from shared memory, V as an MN-major operand)
//   warps 2..5  softmax: TMEM S -> online max / exp2 / sum -> bf16 P in smem, O row
//               rescale in TMEM, final O / l -> global
//   warp 6      wait warp: per-chunk flag acquires for remote KV blocks, ahead of warp 0
// TMEM: S0 [0,128), S1 [128,256), O [256,384) fp32 columns.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernel_args.h"
#include "ptx.cuh"

namespace ao {
namespace dev {

constexpr int kAThreads = 352;   // 11 warps
constexpr int kSmWarps = 8;      // softmax warps: two per TMEM lane quadrant, 64 columns each
constexpr int kBlk = 128;                  // query rows per item = KV rows per block
constexpr uint32_t kHalf = 16384;          // one 128-row x 64-column bf16 box
constexpr uint32_t kQBytes = 2 * kHalf;    // Q tile (d = 128: two boxes)
constexpr uint32_t kKVBytes = 4 * kHalf;   // K block + V block
#ifndef AO_ATTN_KST
#define AO_ATTN_KST 3
#endif
#ifndef AO_ATTN_VST
#define AO_ATTN_VST 3
#endif
constexpr int kKStages = AO_ATTN_KST;  // K ring (32 KB stages)
constexpr int kVStages = AO_ATTN_VST;  // V ring (32 KB stages)
constexpr int kAttnAhead = 4;
constexpr uint32_t kAttnSmem = kQBytes + (kKStages + kVStages) * (kKVBytes / 2) + 2048 + 1024;  // P lives in TMEM

struct AttnBars {
  uint64_t qfull, qempty, kfull[kKStages], kempty[kKStages], vfull[kVStages], vempty[kVStages];
  uint64_t sfull[2], sfree[2], pfull, pvdone[2], ofree;
  uint64_t wrdy[kAttnAhead], wfre[kAttnAhead];
  uint32_t tmem_slot;
  uint8_t waited[kAttnAhead];
  float xmax[2][128];  // per column half: partial row max of a block (row sums at an item's end)
};

__device__ __noinline__ void attn_spin(const uint32_t* p, uint32_t target, const AttnArgs& A, int rank, int cta, int w) {
  if (ld_relaxed_sys(p) >= target) {  // relaxed polls, one acquire (see fused.cu spin_flag)
    ld_acquire_sys(p);
    return;
  }
  const uint64_t t0 = globaltimer();
  uint32_t ns = 32;
  while (ld_relaxed_sys(p) < target) {
    if (globaltimer() - t0 > A.timeout_ns) {
      if (atomicCAS(&A.err->claim, 0u, 1u) == 0u) {
        A.err->rank = rank;
        A.err->cta = cta;
        A.err->chunk = w;
        A.err->epoch = target;
        A.err->seen = ld_acquire_sys(p);
        __threadfence_system();
        st_release_sys(const_cast<uint32_t*>(&A.err->flag), 1u);
      }
      return;
    }
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
  ld_acquire_sys(p);
}

// Device trace (ao_ctx_trace_enable), compiled in only with -DAO_ATTN_TRACE=1 (the hooks
// cost ~3 % even when off; scripts/attn_trace.py): kind TR_LOAD = the producer's wait for a
// free K stage, TR_MMA = the MMA warp's wait for a tile's P (softmax done), TR_WAIT = a
// softmax warpgroup's wait for S, TR_EPI = its softmax of one block (id = tile x).
#ifndef AO_ATTN_TRACE
#define AO_ATTN_TRACE 0
#endif
__device__ __forceinline__ void attn_trace(const AttnArgs& A, uint32_t kind, int rank, int id, uint64_t t0) {
  if (!AO_ATTN_TRACE || A.trace == nullptr) return;
  const uint32_t i = atomicAdd(A.trace_cursor, 1u);
  if (i < A.trace_cap) {
    TraceEvent e;
    e.t0 = t0;
    e.t1 = globaltimer();
    e.kind = kind | (A.trace_seq << 8);
    e.rank = uint32_t(rank);
    e.cta = blockIdx.x;
    e.id = uint32_t(id);
    A.trace[i] = e;
  }
}

// Work items of this CTA in order: (rank group, item).  Space-sliced: its own group's items
// with the persistent stride; time-sliced: every group's items, rank after rank.
template <class F>
__device__ __forceinline__ void attn_walk(const AttnArgs& a, int n_items, F&& f) {
  if (!a.ts) {
    const int g = blockIdx.x / a.ctas_per_rank, w = blockIdx.x % a.ctas_per_rank;
    for (int i = w; i < n_items; i += a.ctas_per_rank) f(g, i);
  } else {
    for (int i = blockIdx.x; i < a.n_group * n_items; i += gridDim.x) f(i / n_items, i % n_items);
  }
}

__global__ void __launch_bounds__(kAThreads, 1) attn_kernel(const __grid_constant__ AttnArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kQBytes;
  uint8_t* sV = sK + kKStages * (kKVBytes / 2);
  AttnBars& B = *reinterpret_cast<AttnBars*>(sV + kVStages * (kKVBytes / 2));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = args.W, S = args.S_loc, nqb = S / kBlk, nkb = S / kBlk;
  const int n_items = args.H * nqb, nkv = W * nkb;

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(&B.qfull, 1);
      mbar_init(&B.qempty, 1);
      for (int s = 0; s < kKStages; ++s) {
        mbar_init(&B.kfull[s], 1);
        mbar_init(&B.kempty[s], 1);
      }
      for (int s = 0; s < kVStages; ++s) {
        mbar_init(&B.vfull[s], 1);
        mbar_init(&B.vempty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&B.sfull[s], 1);
        mbar_init(&B.sfree[s], kSmWarps);
      }
      mbar_init(&B.pfull, kSmWarps);
      mbar_init(&B.pvdone[0], 1);
      mbar_init(&B.pvdone[1], 1);
      mbar_init(&B.ofree, kSmWarps);
      for (int s = 0; s < kAttnAhead; ++s) {
        mbar_init(&B.wrdy[s], 1);
        mbar_init(&B.wfre[s], 1);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&B.tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_slot;

  if (warp == 0) {
    // ===================================================================== TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      uint32_t t = 0, n = 0, q = 0;
      attn_walk(args, n_items, [&](int g, int item) {
        const AttnRank& R = args.rk[g];
        const int h = item / nqb, qb = item % nqb;
        mbar_wait(&B.qempty, (t & 1u) ^ 1u);
        mbar_arrive_expect_tx(&B.qfull, kQBytes);
        tma_load_2d(sQ, &R.tmQ, &B.qfull, 0, h * S + qb * kBlk, pol);
        tma_load_2d(sQ + kHalf, &R.tmQ, &B.qfull, 64, h * S + qb * kBlk, pol);
        for (int j = 0; j < nkv; ++j, ++n) {
          const int d = j / nkb, kb = j % nkb;
          const int src = (R.rank - d + W) % W;
          const int krow = h * S + kb * kBlk;
          const int slot = int(q % kAttnAhead);
          mbar_wait(&B.wrdy[slot], (q / kAttnAhead) & 1u);
          const bool waited = B.waited[slot] != 0;
          mbar_arrive(&B.wfre[slot]);
          ++q;
          if (waited) fence_proxy_async_global();  // generic-proxy acquire -> TMA reads
          // K and V of a block in separate rings: K is released as soon as S = Q K^T is
          // done, so the next K loads while the softmax and P V of this block run
          const uint32_t kst = n % kKStages, kph = ((n / kKStages) & 1u) ^ 1u;
          const uint32_t vst = n % kVStages, vph = ((n / kVStages) & 1u) ^ 1u;
          uint8_t* kdst = sK + kst * (kKVBytes / 2);
          uint8_t* vdst = sV + vst * (kKVBytes / 2);
          const CUtensorMap* mk = d == 0 ? &R.tmK_loc : &R.tmK;
          const CUtensorMap* mv = d == 0 ? &R.tmV_loc : &R.tmV;
          const int row = d == 0 ? krow : src * args.H * S + krow;
          mbar_wait(&B.kempty[kst], kph);
          mbar_arrive_expect_tx(&B.kfull[kst], kKVBytes / 2);
          tma_load_2d(kdst, mk, &B.kfull[kst], 0, row, pol);
          tma_load_2d(kdst + kHalf, mk, &B.kfull[kst], 64, row, pol);
          mbar_wait(&B.vempty[vst], vph);
          mbar_arrive_expect_tx(&B.vfull[vst], kKVBytes / 2);
          tma_load_2d(vdst, mv, &B.vfull[vst], 0, row, pol);
          tma_load_2d(vdst + kHalf, mv, &B.vfull[vst], 64, row, pol);
        }
        ++t;
      });
    }
  } else if (warp == 1) {
    // ===================================================================== MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16(kBlk, kBlk);      // S = Q . K^T
    constexpr uint32_t idesc_o = make_idesc_bf16_bmn(kBlk, 128);   // O += P . V (V MN-major)
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO = tmem + 256;
    uint32_t t = 0, n = 0;
    auto issue_s = [&](uint32_t nn) {
      const uint32_t st = nn % kKStages, sb = nn & 1u;
      mbar_wait(&B.kfull[st], (nn / kKStages) & 1u);
      mbar_wait(&B.sfree[sb], ((nn >> 1) & 1u) ^ 1u);
      // P of block nn-2 lives in this S buffer's columns: its P.V was issued before this S
      // by this thread (the loop below), and tcgen05.mma ops execute in issue order
      tc_fence_after();
      if (lane == 0) {
        const uint8_t* kb = sK + st * (kKVBytes / 2);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = make_smem_desc_sw128(smem_u32(sQ + (kk >> 2) * kHalf)) + uint64_t((kk & 3) * 2);
          const uint64_t b = make_smem_desc_sw128(smem_u32(kb + (kk >> 2) * kHalf)) + uint64_t((kk & 3) * 2);
          mma_bf16_ss(tS[sb], a, b, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&B.sfull[sb]);
        mma_commit(&B.kempty[st]);  // K block consumed
      }
      __syncwarp();
    };
    attn_walk(args, n_items, [&](int g, int item) {
      (void)g;
      (void)item;
      mbar_wait(&B.qfull, t & 1u);
      tc_fence_after();
      issue_s(n);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) {
          issue_s(n + j + 1);
        } else if (lane == 0) {
          mma_commit(&B.qempty);  // every S of this item issued: Q is free once they complete
        }
        __syncwarp();
        if (j == 0) mbar_wait(&B.ofree, (t & 1u) ^ 1u);  // the previous item's O was read
        mbar_wait(&B.pfull, (n + j) & 1u);
        mbar_wait(&B.vfull[(n + j) % kVStages], ((n + j) / kVStages) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = (n + j) % kVStages;
          const uint8_t* vb = sV + st * (kKVBytes / 2);
          const uint32_t tP = tS[(n + j) & 1u];  // P (bf16 pairs) over the S columns
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t b = make_smem_desc_sw128_mn(smem_u32(vb + kk * 16 * 128), kHalf);
            mma_bf16_ts(tO, tP + kk * 8, b, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&B.vempty[st]);
          mma_commit(&B.pvdone[(n + j) & 1u]);  // P buffer (n+j)&1 free, O updated
        }
        __syncwarp();
      }
      n += nkv;
      ++t;
    });
  } else if (warp < 2 + kSmWarps) {
    // ===================================================================== softmax
    // warps 2..9: two per TMEM lane quadrant (row r), column half hf (64 of the 128 S / P /
    // O columns); the pair combines its partial row maxima through smem every block.
    const int qd = warp & 3;  // TMEM lane quadrant
    const int hf = (warp - 2) >> 2;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t pair_bar = 1 + qd;  // named barrier of the two warps of quadrant qd
    const float sl2 = args.scale_log2;
    uint32_t n = 0;
    uint32_t cons[2] = {0, 0};  // phases of pvdone[b] consumed (PV of blocks b, b+2, ... done)
    // wait until PV of global block nb is done (in order per buffer; never skips a phase)
    auto pv_wait = [&](uint32_t nb) {
      const uint32_t b = nb & 1u;
      while (cons[b] <= (nb >> 1)) {
        mbar_wait(&B.pvdone[b], cons[b] & 1u);
        ++cons[b];
      }
      tc_fence_after();
    };
    attn_walk(args, n_items, [&](int g, int item) {
      const AttnRank& R = args.rk[g];
      const int h = item / nqb, qb = item % nqb;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        const uint32_t nn = n + j, sb = nn & 1u;
        mbar_wait(&B.sfull[sb], (nn >> 1) & 1u);
        // S of block nn exists, so the P.V of block nn-2 has completed (the MMA waited for it
        // before writing this buffer): consume that phase, keeping the per-buffer phase count
        // at most one behind (mbarrier parity waits must never fall two phases behind)
        if (nn >= 2) pv_wait(nn - 2);
        tc_fence_after();
        float s[64];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem + lane_off + sb * 128 + hf * 64 + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.sfree[sb]);
        // row max over the pair's two halves (8 independent partials per half)
        float mp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mp[u] = s[u];
#pragma unroll
        for (int i = 4; i < 32; ++i) mp[i & 7] = max3f(mp[i & 7], s[2 * i], s[2 * i + 1]);
        const float mh = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
        B.xmax[hf][r] = mh;
        named_bar_sync(pair_bar, 64);
        const float mx = fmaxf(mh, B.xmax[hf ^ 1][r]);
        named_bar_sync(pair_bar, 64);  // both read before the next block overwrites
        // lazy rescale: the exponent base m moves only when the row max exceeds it by more
        // than 8 (p <= 2^8 stays exact enough in fp32 / bf16); otherwise alpha = 1 and the
        // O row in TMEM is left alone (the final O / l is consistent for any base)
        const float mxs = mx * sl2;
        const bool grow = mxs > m + 8.f;
        const float m_new = grow ? mxs : m;
        const float alpha = grow ? exp2f(m - m_new) : 1.f;
        // s * scale_log2 - m as FFMA2 pairs, exp2 on the MUFU, row sums as FADD2 pairs
        const uint64_t sc2 = f2_pack(__float_as_uint(sl2), __float_as_uint(sl2));
        const uint64_t nm2 = f2_pack(__float_as_uint(-m_new), __float_as_uint(-m_new));
        uint64_t sp2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float a, b;
          f2_unpack(f2_fma(f2_pack(__float_as_uint(s[2 * i]), __float_as_uint(s[2 * i + 1])), sc2, nm2), a, b);
          s[2 * i] = ex2_ftz(a);
          s[2 * i + 1] = ex2_ftz(b);
          sp2[i & 3] = f2_add(sp2[i & 3], f2_pack(__float_as_uint(s[2 * i]), __float_as_uint(s[2 * i + 1])));
        }
        float sp[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) f2_unpack(sp2[u], sp[2 * u], sp[2 * u + 1]);
        const float sum = ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
        l = l * alpha + sum;
        m = m_new;
        // this half of P row r as bf16 pairs into TMEM over the S columns just read (the
        // A operand of P.V, 32 packed columns per half); the MMA issued the next S into this
        // buffer only after the previous P.V read it
        {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = pack_bf16x2(s[2 * c], s[2 * c + 1]);
          tmem_st_32x32b_x32(tmem + lane_off + sb * 128 + hf * 32, pk);
        }
        const bool rescale = j > 0 && __any_sync(0xffffffffu, alpha < 1.f);
        if (rescale) pv_wait(nn - 1);  // O holds every PV up to block nn-1
        if (rescale) {  // rescale this half of the O row by alpha
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tmem + lane_off + 256 + hf * 64 + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_off + 256 + hf * 64 + c * 32, v);
          }
          tmem_wait_st();
        }
        tmem_wait_st();  // P (and a rescaled O) in TMEM before the MMA reads them
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.pfull);
      }
      // final O half row / l -> bf16 -> global (l = the two halves' partial sums)
      pv_wait(n + nkv - 1);
      B.xmax[hf][r] = l;  // (the exchange slots carry the row sums here)
      named_bar_sync(pair_bar, 64);
      const float inv = 1.f / (l + B.xmax[hf ^ 1][r]);
      named_bar_sync(pair_bar, 64);
      char* orow = R.O + (int64_t(h) * S + qb * kBlk + r) * 256 + hf * 128;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_off + 256 + hf * 64 + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 w = make_uint4(pack_bf16x2(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv));
          *reinterpret_cast<uint4*>(orow + c * 64 + i * 16) = w;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.ofree);
      n += nkv;
    });
  } else if (warp == 2 + kSmWarps) {
    // ===================================================================== wait warp
    if (lane == 0) {
      uint64_t got[AO_MAX_WORLD] = {};
      uint32_t q = 0;
      attn_walk(args, n_items, [&](int g, int item) {
        const AttnRank& R = args.rk[g];
        const int h = item / nqb;
        for (int j = 0; j < nkv; ++j) {
          const int slot = int(q % kAttnAhead);
          mbar_wait(&B.wfre[slot], ((q / kAttnAhead) & 1u) ^ 1u);
          const int d = j / nkb, kb = j % nkb;
          bool waited = false;
          if (d > 0) {
            const int src = (R.rank - d + W) % W;
            const int w = src * args.nch + (h * S + kb * kBlk) / args.crows;
            if (!(w < 64 && ((got[g] >> w) & 1u))) {
              attn_spin(R.flags + w, R.epoch, args, R.rank, int(blockIdx.x), w);
              if (w < 64) got[g] |= 1ull << w;
              waited = true;
            }
          }
          B.waited[slot] = waited ? 1 : 0;
          mbar_arrive(&B.wrdy[slot]);
          ++q;
        }
      });
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// ---- ping-pong variant: two query tiles per item (S_loc % 256 == 0) ------------------------
// Item = (head, 256 queries) = tiles x = 0, 1 sharing every K/V block.  Each tile has its own
// softmax warpgroup (warps 2-5 and 6-9), S buffer and O accumulator in TMEM, so the tensor
// core works on one tile's QK^T / PV while the other tile's softmax runs (the FA4 schedule).
// 10 warps (the producer acquires the chunk flags itself) and at most 152 registers per
// thread, so that 320 x 152 registers leave room on every SM for the copy kernels that
// execute same-device memcpy nodes (the loopback "copy engine" pushes): with 320 x 168 they
// could not be scheduled while this persistent kernel ran and the chunk waits timed out.
constexpr int kPPThreads = 320;
constexpr int kPPK = 2, kPPV = 2;  // K and V ring stages (32 KB each)
constexpr uint32_t kPPSmem = 2 * kQBytes + (kPPK + kPPV) * (kKVBytes / 2) + 2048 + 1024;

struct PPBars {
  uint64_t qfull, qempty, kfull[kPPK], kempty[kPPK], vfull[kPPV], vempty[kPPV];
  uint64_t sfull[2], pfull[2], pvdone[2], ofree[2];  // per tile
  uint64_t wrdy[kAttnAhead], wfre[kAttnAhead];
  uint32_t tmem_slot;
  uint8_t waited[kAttnAhead];
};

// 152 registers x 320 threads = 48.6K of the SM's 64K: the rest stays free for the memcpy
// kernels that carry the loopback K/V pushes (53.7K stalled them; 128 measured 3 % slower
// causal).  CAUSAL is a template parameter so the non-causal kernel carries no mask code.
template <bool CAUSAL>
__global__ void __maxnreg__(152) attn_pp_kernel(const __grid_constant__ AttnArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;  // tile 0 at +0, tile 1 at +kQBytes
  uint8_t* sK = sQ + 2 * kQBytes;
  uint8_t* sV = sK + kPPK * (kKVBytes / 2);
  PPBars& B = *reinterpret_cast<PPBars*>(sV + kPPV * (kKVBytes / 2));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = args.W, S = args.S_loc, nqp = S / (2 * kBlk), nkb = S / kBlk;
  // SP: items (head, query pair) of this rank's queries; HP: items (query source, head of
  // this rank's group, query pair), query sources in arrival order (own rank first, then
  // r-1, r-2, ...).  args.H = heads of the view (SP: all, HP: this rank's H/W).
  const int n_items = (args.hp ? W : 1) * args.H * nqp;
  struct Item {
    int hv, qp, qs;  // head in the view, query pair, source rank of the queries
  };
  auto decode = [&](const AttnRank& R, int item) -> Item {
    if (!args.hp) return Item{item / nqp, item % nqp, R.rank};
    const int per = args.H * nqp, qi = item / per, rem = item - qi * per;
    return Item{rem / nqp, rem % nqp, (R.rank - qi + W) % W};
  };
  // KV blocks of an item, in arrival order: the base shard first (kb = 0, 1, ...), then the
  // sources base-1, base-2, ... (the push rotation); base = this rank (its own shard needs no
  // wait).  Causal: base = the queries' source, only its blocks up to the item's last query
  // (kb <= 2qp+1, the diagonal) and only the sources below it (RingAttention skips the
  // future shards).
  auto nkv_of = [&](const Item& it) -> int { return CAUSAL ? it.qs * nkb + 2 * it.qp + 2 : W * nkb; };
  auto kv_of = [&](const Item& it, int j, int& d, int& kb) {
    const int own = CAUSAL ? 2 * it.qp + 2 : nkb;
    if (j < own) {
      d = 0;
      kb = j;
    } else {
      d = 1 + (j - own) / nkb;
      kb = (j - own) % nkb;
    }
  };
  auto kv_src = [&](const AttnRank& R, const Item& it, int d) -> int { return ((CAUSAL ? it.qs : R.rank) - d + W) % W; };
  const int hv_rows = args.H * S;  // rows of one source's block in the gathered buffers

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(&B.qfull, 1);
      mbar_init(&B.qempty, 1);
      for (int s = 0; s < kPPK; ++s) {
        mbar_init(&B.kfull[s], 1);
        mbar_init(&B.kempty[s], 1);
      }
      for (int s = 0; s < kPPV; ++s) {
        mbar_init(&B.vfull[s], 1);
        mbar_init(&B.vempty[s], 1);
      }
      for (int x = 0; x < 2; ++x) {
        mbar_init(&B.sfull[x], 1);
        mbar_init(&B.pfull[x], 4);
        mbar_init(&B.pvdone[x], 1);
        mbar_init(&B.ofree[x], 4);
      }
      for (int s = 0; s < kAttnAhead; ++s) {
        mbar_init(&B.wrdy[s], 1);
        mbar_init(&B.wfre[s], 1);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&B.tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_slot;  // S_x at x*128, O_x at 256 + x*128

  if (warp == 0) {
    // ===================================================================== TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      uint32_t t = 0, n = 0;
      uint64_t got[AO_MAX_WORLD] = {};  // acquired chunk flags per rank group (w < 64)
      attn_walk(args, n_items, [&](int g, int item) {
        const AttnRank& R = args.rk[g];
        const Item it = decode(R, item);
        const int h = it.hv, qp = it.qp;
        const int hoff = args.hp ? R.rank * args.H : 0;  // HP: this rank's heads in the local tensors
        mbar_wait(&B.qempty, (t & 1u) ^ 1u);
        const CUtensorMap* mq = &R.tmQ;
        int qrow = (hoff + h) * S + qp * 2 * kBlk;
        if (it.qs != R.rank) {  // HP: another source's queries, from the gathered Q
          const int vr = h * S + qp * 2 * kBlk;
          for (int c = vr / args.crows; c <= (vr + 2 * kBlk - 1) / args.crows; ++c) {
            const int w = it.qs * args.nch + c;
            if (!(w < 64 && ((got[g] >> w) & 1u))) {
              attn_spin(R.flags + w, R.epoch, args, R.rank, int(blockIdx.x), w);
              if (w < 64) got[g] |= 1ull << w;
            }
          }
          fence_proxy_async_global();  // generic-proxy acquire -> TMA reads
          mq = &R.tmQg;
          qrow = it.qs * hv_rows + vr;
        }
        mbar_arrive_expect_tx(&B.qfull, 2 * kQBytes);
        tma_load_2d(sQ, mq, &B.qfull, 0, qrow, pol);
        tma_load_2d(sQ + kHalf, mq, &B.qfull, 64, qrow, pol);
        tma_load_2d(sQ + kQBytes, mq, &B.qfull, 0, qrow + kBlk, pol);
        tma_load_2d(sQ + kQBytes + kHalf, mq, &B.qfull, 64, qrow + kBlk, pol);
        const int nkv = nkv_of(it);
        for (int j = 0; j < nkv; ++j, ++n) {
          int d, kb;
          kv_of(it, j, d, kb);
          const int src = kv_src(R, it, d);
          const int krow = h * S + kb * kBlk;  // row in the view of one source's block
          const bool local = src == R.rank;
          if (!local) {  // the chunk (src, h*S + kb*128) must have landed
            const int w = src * args.nch + krow / args.crows;
            if (!(w < 64 && ((got[g] >> w) & 1u))) {
              attn_spin(R.flags + w, R.epoch, args, R.rank, int(blockIdx.x), w);
              if (w < 64) got[g] |= 1ull << w;
              fence_proxy_async_global();  // generic-proxy acquire -> TMA reads
            }
          }
          const uint32_t kst = n % kPPK, vst = n % kPPV;
          const CUtensorMap* mk = local ? &R.tmK_loc : &R.tmK;
          const CUtensorMap* mv = local ? &R.tmV_loc : &R.tmV;
          const int row = local ? hoff * S + krow : src * hv_rows + krow;
          uint8_t* kdst = sK + kst * (kKVBytes / 2);
          uint8_t* vdst = sV + vst * (kKVBytes / 2);
          const uint64_t tk = AO_ATTN_TRACE && args.trace ? globaltimer() : 0;
          mbar_wait(&B.kempty[kst], ((n / kPPK) & 1u) ^ 1u);
          if (AO_ATTN_TRACE && args.trace) attn_trace(args, TR_LOAD, R.rank, int(n), tk);
          mbar_arrive_expect_tx(&B.kfull[kst], kKVBytes / 2);
          tma_load_2d(kdst, mk, &B.kfull[kst], 0, row, pol);
          tma_load_2d(kdst + kHalf, mk, &B.kfull[kst], 64, row, pol);
          mbar_wait(&B.vempty[vst], ((n / kPPV) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&B.vfull[vst], kKVBytes / 2);
          tma_load_2d(vdst, mv, &B.vfull[vst], 0, row, pol);
          tma_load_2d(vdst + kHalf, mv, &B.vfull[vst], 64, row, pol);
        }
        ++t;
      });
    }
  } else if (warp == 1) {
    // ===================================================================== MMA issuer
    constexpr uint32_t idesc_s = make_idesc_bf16(kBlk, kBlk);
    constexpr uint32_t idesc_o = make_idesc_bf16_bmn(kBlk, 128);
    uint32_t t = 0, n = 0;
    auto issue_s = [&](int x, uint32_t nn) {  // S_x = Q_x . K(nn)^T
      const uint32_t st = nn % kPPK;
      mbar_wait(&B.kfull[st], (nn / kPPK) & 1u);
      tc_fence_after();
      if (lane == 0) {
        const uint8_t* kb = sK + st * (kKVBytes / 2);
        const uint8_t* qa = sQ + x * kQBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = make_smem_desc_sw128(smem_u32(qa + (kk >> 2) * kHalf)) + uint64_t((kk & 3) * 2);
          const uint64_t b = make_smem_desc_sw128(smem_u32(kb + (kk >> 2) * kHalf)) + uint64_t((kk & 3) * 2);
          mma_bf16_ss(tmem + x * 128, a, b, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&B.sfull[x]);
        if (x == 1) mma_commit(&B.kempty[st]);  // both tiles have read K(nn)
      }
      __syncwarp();
    };
    attn_walk(args, n_items, [&](int g, int item) {
      const int nkv = nkv_of(decode(args.rk[g], item));
      mbar_wait(&B.qfull, t & 1u);
      for (int x = 0; x < 2; ++x) {
        if (n > 0) mbar_wait(&B.pvdone[x], (n - 1) & 1u);  // P_x of the previous item was read
        issue_s(x, n);
      }
      for (int j = 0; j < nkv; ++j) {
        const uint32_t nn = n + j;
        if (j + 1 == nkv && lane == 0) mma_commit(&B.qempty);  // every S of this item issued
        __syncwarp();
        for (int x = 0; x < 2; ++x) {
          if (j == 0) mbar_wait(&B.ofree[x], (t & 1u) ^ 1u);  // O_x of the previous item read
          const uint64_t tp = AO_ATTN_TRACE && args.trace ? globaltimer() : 0;
          mbar_wait(&B.pfull[x], nn & 1u);
          if (AO_ATTN_TRACE && args.trace && lane == 0) attn_trace(args, TR_MMA, args.rk[g].rank, x, tp);
          if (x == 0) mbar_wait(&B.vfull[nn % kPPV], (nn / kPPV) & 1u);
          tc_fence_after();
          if (lane == 0) {
            const uint8_t* vb = sV + (nn % kPPV) * (kKVBytes / 2);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t b = make_smem_desc_sw128_mn(smem_u32(vb + kk * 16 * 128), kHalf);
              mma_bf16_ts(tmem + 256 + x * 128, tmem + x * 128 + kk * 8, b, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&B.pvdone[x]);
            if (x == 1) mma_commit(&B.vempty[nn % kPPV]);
          }
          __syncwarp();
          // S_x(nn+1) overwrites P_x(nn) in TMEM: tcgen05.mma ops of one thread execute in
          // issue order, so it is issued right behind PV_x(nn) without waiting for its
          // completion (waiting left a commit -> mbarrier round trip as a pipe bubble per block)
          if (j + 1 < nkv) issue_s(x, nn + 1);
        }
      }
      n += nkv;
      ++t;
    });
  } else if (warp < 10) {
    // ===================================================================== softmax (tile x)
    const int x = (warp - 2) >> 2;
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t tS = tmem + lane_off + x * 128, tO = tmem + lane_off + 256 + x * 128;
    const float sl2 = args.scale_log2;
    uint32_t n = 0, cons = 0;
    auto pv_wait = [&](uint32_t nb) {
      while (cons <= nb) {
        mbar_wait(&B.pvdone[x], cons & 1u);
        ++cons;
      }
      tc_fence_after();
    };
    attn_walk(args, n_items, [&](int g, int item) {
      const AttnRank& R = args.rk[g];
      const Item it = decode(R, item);
      const int h = it.hv, qp = it.qp;
      const int nkv = nkv_of(it);
      const int qloc = qp * 2 * kBlk + x * kBlk + r;  // this thread's query (position in its source's shard)
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        const uint32_t nn = n + j;
        int d, kb;
        kv_of(it, j, d, kb);
        // causal: keys kb*128 + c beyond this query are masked (own diagonal blocks only)
        const int kmax = (CAUSAL && d == 0) ? qloc - kb * kBlk : 1 << 30;
        const uint64_t ts0 = AO_ATTN_TRACE && args.trace ? globaltimer() : 0;
        mbar_wait(&B.sfull[x], nn & 1u);
        tc_fence_after();
        if (nn >= 1) pv_wait(nn - 1);  // PV(nn-1) done before O is rescaled / P(nn) written
        const uint64_t ts1 = AO_ATTN_TRACE && args.trace ? globaltimer() : 0;
        if (AO_ATTN_TRACE && args.trace && qd == 0 && lane == 0) attn_trace(args, TR_WAIT, R.rank, x, ts0);
        if (CAUSAL && d == 0 && kb >= 2 * qp) {
          // causal diagonal blocks (two per item): keys past this query become -inf in TMEM,
          // so the passes below stay mask-free (registers are tight)
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tS + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i > kmax) v[i] = 0xff800000u;  // -inf
            tmem_st_32x32b_x32(tS + c * 32, v);
          }
          tmem_wait_st();
        }
        // two passes over the S row in TMEM (max, then exp) keep 64 values live instead of
        // 128: the kernel's registers must leave room for the memcpy kernels (see kPPThreads)
        float mp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mp[u] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tS + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) mp[i & 7] = max3f(mp[i & 7], __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        }
        const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
        const float mxs = mx * sl2;
        const bool grow = mxs > m + 8.f;  // lazy rescale (see attn_kernel)
        const float m_new = grow ? mxs : m;
        const float alpha = grow ? exp2f(m - m_new) : 1.f;
        // s * scale_log2 - m as FFMA2 pairs, exp2 on the MUFU, row sums as FADD2 pairs
        const uint64_t sc2 = f2_pack(__float_as_uint(sl2), __float_as_uint(sl2));
        const uint64_t nm2 = f2_pack(__float_as_uint(-m_new), __float_as_uint(-m_new));
        uint64_t sp2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // exp per 32 columns; P row r as bf16 pairs
          uint32_t v[32];
          tmem_ld_32x32b_x32(tS + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float a, b;
            f2_unpack(f2_fma(f2_pack(v[2 * i], v[2 * i + 1]), sc2, nm2), a, b);
            a = ex2_ftz(a);
            b = ex2_ftz(b);
            sp2[i & 3] = f2_add(sp2[i & 3], f2_pack(__float_as_uint(a), __float_as_uint(b)));
            pk[(c & 1) * 16 + i] = pack_bf16x2(a, b);
          }
          // P columns 32(c/2) .. +31 overwrite S columns this thread has already read
          if (c & 1) tmem_st_32x32b_x32(tS + (c >> 1) * 32, pk);
        }
        float sp[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) f2_unpack(sp2[u], sp[2 * u], sp[2 * u + 1]);
        l = l * alpha + (((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7])));
        m = m_new;
        if (j > 0 && __any_sync(0xffffffffu, alpha < 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, v);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.pfull[x]);
        if (AO_ATTN_TRACE && args.trace && qd == 0 && lane == 0) attn_trace(args, TR_EPI, R.rank, x, ts1);
      }
      pv_wait(n + nkv - 1);
      const float inv = 1.f / l;
      // SP and HP own queries: O rows of this rank; HP other sources: their return buffer,
      // block of this rank's head group
      const int hoff = args.hp ? R.rank * args.H : 0;
      char* orow = it.qs == R.rank ? R.O + (int64_t(hoff + h) * S + qloc) * 256
                                   : R.oret[it.qs] + (int64_t(R.rank) * hv_rows + int64_t(h) * S + qloc) * 256;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tO + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 w = make_uint4(pack_bf16x2(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv),
                                     pack_bf16x2(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv));
          *reinterpret_cast<uint4*>(orow + c * 64 + i * 16) = w;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.ofree[x]);
      if (it.qs != R.rank) {
        // HP: count this tile into its destination block; the last of the block's H*nqp*2
        // tiles releases the destination's return flag (cumulative over the warpgroup's
        // stores, which precede the barrier)
        named_bar_sync(1 + x, 128);
        if (qd == 0 && lane == 0) {
          uint32_t old;
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(R.counters + it.qs) : "memory");
          if (int(old) + 1 == args.H * nqp * 2) {
            R.counters[it.qs] = 0;
            st_release_sys(R.peer_flags[it.qs] + W * args.nch + R.rank, R.epoch);
          }
        }
      }
      n += nkv;
    });
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace dev

cudaError_t launch_attn(const AttnArgs& args, cudaStream_t stream) {
  // two-tile ping-pong kernel when S_loc is a multiple of 256 (AO_ATTN_SINGLE=1 forces the
  // one-tile kernel)
  static const bool single = getenv("AO_ATTN_SINGLE") && getenv("AO_ATTN_SINGLE")[0] == '1';
  const bool pp = args.causal || args.hp || (!single && args.S_loc % (2 * dev::kBlk) == 0);  // causal / HP: pp only
  static bool attr = false, attr_pp = false, attr_ppc = false;
  if (!pp && !attr) {
    cudaError_t e = cudaFuncSetAttribute(dev::attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(dev::kAttnSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (pp && !args.causal && !attr_pp) {
    cudaError_t e = cudaFuncSetAttribute(dev::attn_pp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(dev::kPPSmem));
    if (e != cudaSuccess) return e;
    attr_pp = true;
  }
  if (pp && args.causal && !attr_ppc) {
    cudaError_t e = cudaFuncSetAttribute(dev::attn_pp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(dev::kPPSmem));
    if (e != cudaSuccess) return e;
    attr_ppc = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(args.ts ? args.ctas_per_rank : args.n_group * args.ctas_per_rank);
  cfg.blockDim = dim3(pp ? dev::kPPThreads : dev::kAThreads);
  cfg.dynamicSmemBytes = pp ? dev::kPPSmem : dev::kAttnSmem;
  cfg.stream = stream;
  // Not a cooperative launch: a cooperative kernel was measured to stall the copy-engine
  // chunk pushes on other streams until it exits (the spin-waits then time out).  Co-
  // residency of the spin-waiting CTAs holds by construction instead: grid <= SMs and one
  // CTA per SM (shared memory), as for the cluster-launched GEMM kernels.
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  if (!pp) return cudaLaunchKernelEx(&cfg, dev::attn_kernel, args);
  return args.causal ? cudaLaunchKernelEx(&cfg, dev::attn_pp_kernel<true>, args)
                     : cudaLaunchKernelEx(&cfg, dev::attn_pp_kernel<false>, args);
}

}  // namespace ao
