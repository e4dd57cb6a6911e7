// kernel_args.h -- parameter block of the fused persistent kernel (host <-> device).
//
// One launch carries n_group ranks of the same world that live on the same device
// (loopback) -- or a single rank in the one-process-per-GPU deployment.  Space-sliced
// (n_seg == 0): the block index selects the rank group: CTAs [g*ctas_per_rank,
// (g+1)*ctas_per_rank) are rank g's GEMM workers (plan CTA c = blockIdx % ctas_per_rank);
// dedicated communication CTAs follow.  Time-sliced (n_seg > 0): all ctas_per_rank CTAs
// serve every rank, walking one global list of (rank, position) segments; chunk waits are
// taken per tile from the dependency rule (minimal per worker via an acquired-chunk cache)
// instead of the plan's per-CTA wait table.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "autooverlap.h"

namespace ao {

enum KernelMode : int { MODE_GEMM = 0, MODE_AG = 1, MODE_RS = 2, MODE_A2A = 3 };

// u32 flag words per epoch parity in every rank's symmetric workspace.  The last
// kA2ATailWords hold the A2A count exchange (count flags [W] | count table [W][W]); no op
// uses them as chunk flags (a count could otherwise satisfy another op's epoch wait).
constexpr uint32_t kFlagWordsPerParity = 1u << 18;
constexpr uint32_t kA2ATailWords = 128;
constexpr uint32_t kA2ACountFlags = kFlagWordsPerParity - kA2ATailWords;
enum CommKind : int { COMM_NONE = 0, COMM_TMA = 1, COMM_LDST = 2 };

// ErrorInfo.cta value of an A2A prep record: an invalid routing entry (chunk = token,
// epoch = choice j, seen = the id) rather than a spin timeout.
constexpr int32_t kErrBadRouting = -101;

// Host-mapped record of the first device-side spin timeout.
struct ErrorInfo {
  volatile uint32_t flag;   // published (set after the fields below are written)
  int32_t rank, cta, chunk;
  uint32_t epoch, seen, target;
  uint32_t claim;           // first failing thread wins the CAS on this word
};

// A communication work item of the in-kernel AG backends: copy `bytes` bytes at byte
// offset `off` of chunk `g` from the local shard to rank `peer`'s gathered buffer, then
// release flag word g*n_slices + slice at `peer`.
// AG transfer item of the in-kernel backends.  kind PUSH: local shard -> peer's gathered
// buffer, release the peer's flag.  STAGE (pull plans): local shard -> own gathered buffer
// (the region peers pull from), release the own flag ("ready").  PULL: wait for the source
// peer's ready flag, peer's gathered buffer -> own gathered buffer, release the own flag.
// AR_PULL (GEMM-AR gather): wait for the owner's "reduced" flag of chunk g, copy the
// owner's reduced rows into this rank's output C (no flag released).
enum ItemKind : int32_t { ITEM_PUSH = 0, ITEM_STAGE = 1, ITEM_PULL = 2, ITEM_AR_PULL = 3 };
struct CommItem {
  int32_t peer, g, slice, kind;     // peer: destination (PUSH) or source (PULL) rank
  int64_t src_off, dst_off, bytes;  // byte offsets (src: local shard or peer buffer, dst: buffer)
};

struct alignas(64) RankArgs {
  CUtensorMap tmA;      // AG: gathered buffer (current parity) [M, K]; RS/GEMM: A [M, K]
  CUtensorMap tmA_loc;  // AG: local shard [S, K].  RS: this rank's slots [W*S, N] fp32 (32 x 128 boxes)
  CUtensorMap tmB;      // B [N, K]
  CUtensorMap tmAcc[AO_MAX_WORLD];  // RS ATOMIC: every owner's accumulator [S, N] fp32, 32 x 32 boxes
  const int* order;            // [n_tiles] tile ids in execution order
  const int* wait_off;         // [n_cta + 1] CSR offsets into waits
  const int2* waits;           // (position k, chunk g)
  const int* tiles_per_chunk;  // RS [n_chunks]: 128-row sub-tiles (one per CTA) touching chunk g
  const int* reduce_items;     // RS [n_items] tile ids
  const CommItem* comm_items;  // AG in-kernel comm [n_comm_items]
  const int* comm_by_peer;     // comm item indices grouped by peer (stable), CSR offsets comm_peer_off[W + 1]
  const int* comm_peer_off;
  void* C;                     // AG/GEMM: C [M, N] bf16.  RS: C_shard [S, N] bf16
  const char* A_shard;         // AG: local shard (source of pushes)
  uint32_t* flags;             // this rank's flag words (current parity)
  uint32_t* peer_flags[AO_MAX_WORLD];  // every rank's flag words (current parity)
  char* peer_data[AO_MAX_WORLD];       // every rank's data half (current parity)
  int32_t ar;        // GEMM-AR: RS + pull gather of the reduced chunks
  char* ar_out;      // GEMM-AR: the caller's full output C [M, N] bf16 (gather destination)
  char* ar_red;      // GEMM-AR: this rank's reduced rows [S, N] bf16 in its symmetric buffer
  char* peer_acc[AO_MAX_WORLD];        // RS ATOMIC: every rank's accumulator [S, N] fp32 (current parity)
  uint32_t* counters;                  // RS: local per-chunk completion counters
  int64_t M, N, K, S;
  int32_t rank, W, crows, n_chunks, n_tiles, n_items, n_nb, n_slices, n_comm_items, n_cta;
  uint32_t epoch;
  int32_t rs_atomic;  // RS: 1 = reduce-add into one accumulator (slot 0) instead of per-source slots
  int32_t rs_bf16;    // RS ATOMIC: bf16 wire (bf16 partials reduce-added into a bf16 accumulator; Q14)
  // A2A (NEXT-3): chunk flags [W][maxJ] at word 0, count flags [W] at kA2ACountFlags, count
  // table [W][W] (row s = source s's per-expert counts) after them; receive buffer = peer_data.
  const int32_t* a2a_perm;  // [W][T] this rank's token ids grouped by destination expert
  int32_t T, topk, maxJ, gm;
  // stream-K tail (Q28): positions >= sk_dp are split along K (sk_dp >= n_tiles: off).  Per
  // split position and CTA of the cluster, the tail piece's fp32 partial [ceil(BN/32)][128][32]
  // in sk_ws and a flag word in sk_flags holding the launch sequence number sk_seq.
  float* sk_ws;
  uint32_t* sk_flags;
  uint32_t sk_seq;
  int32_t sk_dp;
};

// A2A prep kernel (routing -> counts, permutation, count exchange, route positions).
struct A2APrepRank {
  const int32_t* topk_idx;  // [T, k]
  int32_t* perm;            // [W][T] out
  int32_t* lpos;            // [T, k] out: position inside the (source, expert) block
  int32_t* route_pos;       // [T, k] out: row in the expert's Y
  int32_t* recv_rows;       // [1] out
  uint32_t* peer_flags[AO_MAX_WORLD];  // every rank's flag words (current parity)
  int32_t rank;
};
struct A2APrepArgs {
  A2APrepRank rk[AO_MAX_WORLD];
  int32_t n_group, W, T, topk, maxJ;
  uint32_t epoch;
  uint64_t timeout_ns;
  ErrorInfo* err;
};

// SP attention (NEXT-4): rank r's queries against the all-gathered K/V, head dim 128.
// Q/K/V/O are [H, S_loc, 128] bf16 viewed as [H*S_loc, 128]; the gathered K and V buffers
// are [W][H*S_loc][128] (source-major) in the symmetric data half (K, then V).
struct AttnRank {
  CUtensorMap tmQ, tmK_loc, tmV_loc, tmK, tmV;  // 2-D maps, boxes of 64 elements x 128 rows
  CUtensorMap tmQg;                             // HP: gathered Q [W][H/W*S_loc][128]
  char* O;                                      // [H*S_loc, 128] bf16
  const uint32_t* flags;                        // this rank's flag words: chunk (src, c) at src*nch + c
  // HP: every rank's O return buffer [W][H/W*S_loc][128] (current parity) and flag words
  // (return flag of source block s at word W*nch + s), tiles done per destination (counters)
  char* oret[AO_MAX_WORLD];
  uint32_t* peer_flags[AO_MAX_WORLD];
  uint32_t* counters;
  int32_t rank;
  uint32_t epoch;
};
struct AttnArgs {
  AttnRank rk[AO_MAX_WORLD];
  int32_t n_group, W, H, S_loc, crows, nch;  // crows: rows of the [H*S_loc] view per chunk
  int32_t ctas_per_rank, ts;                 // ts: time-sliced whole-world group (rank after rank)
  int32_t causal;                            // causal mask over global token positions (ping-pong kernel)
  int32_t hp;                                // head-parallel: items (query source, head of the group, pair)
  float scale_log2;                          // softmax scale * log2(e)
  uint64_t timeout_ns;
  ErrorInfo* err;
  struct TraceEvent* trace;
  uint32_t* trace_cursor;
  uint32_t trace_cap, trace_seq;
};

// In-kernel trace event (AO tracing): 32 bytes, %globaltimer nanoseconds.
// TR_CLK: id = SM clock cycles (clock64) over an MMA span -- the clock the kernel runs at under load.
enum TraceKind : uint32_t { TR_WAIT = 1, TR_LOAD = 2, TR_MMA = 3, TR_EPI = 4, TR_COMM = 5, TR_RED = 6, TR_REDWAIT = 7,
                            TR_CLK = 8 };
struct TraceEvent {
  uint64_t t0, t1;
  uint32_t kind, rank, cta, id;
};

// Time-sliced group (loopback): positions [k0, k1) of rank group g's tile list occupy
// global indices [o, o + k1 - k0) of the launch's single work list; physical worker w
// runs global indices w, w + n_workers, ... (Lst.1's persistent stride over the list).
struct Seg {
  int32_t g, k0, k1, o;
};
constexpr int kMaxSegs = 256;

struct KernelArgs {
  RankArgs rk[AO_MAX_WORLD];
  int32_t n_seg;               // 0: space-sliced (rank group = blockIdx / ctas_per_rank)
  int32_t n_total;             // time-sliced: total positions of the list
  Seg seg[kMaxSegs];           // time-sliced: the global list, in execution order
  int32_t n_group;
  int32_t ctas_per_rank;       // GEMM CTAs per rank (== plan n_cta * cta_group)
  int32_t comm_ctas_per_rank;  // dedicated comm CTAs per rank
  int32_t mode;                // KernelMode
  uint64_t timeout_ns;
  ErrorInfo* err;              // host-mapped
  int32_t skip_wait;           // debug: CSR index of a wait of rank group 0 to skip (-1 none)
  uint32_t delay_ns;           // debug: sleep before each comm signal
  TraceEvent* trace;           // null = tracing off
  uint32_t* trace_cursor;
  uint32_t trace_cap;
  uint32_t trace_seq;          // launch sequence number stamped into events (kind >> 8)
  int32_t exp;                 // timing experiments only (ao_debug_set "exp"); 0 in normal runs
  int32_t l2_hint;             // 0: A evict_first / B evict_last (row order); 1: A evict_last / B evict_first
  int32_t a2a_ts;              // A2A: time-sliced group (all CTAs serve every rank, rank after rank)
};

// Host-side launcher (fused.cu).
// Kernel parameters are passed by value (__grid_constant__); sm_70+ with CUDA >= 12.1 allows 32764 bytes.
static_assert(sizeof(KernelArgs) <= 32764, "KernelArgs exceeds the kernel parameter limit");

// bn: tile N (128/256); cg: 1 (BM = 128) or 2 (CTA pair, BM = 256); comm: CommKind.
cudaError_t launch_fused(const KernelArgs& args, int bn, int cg, int comm, cudaStream_t stream);
cudaError_t launch_a2a_prep(const A2APrepArgs& args, cudaStream_t stream);
// E4 microbenchmark: move `bytes` from src to dst in chunks of `chunk` with the in-kernel
// TMA or LDST backend on n_ctas CTAs of 8 warps (e4.cu).
cudaError_t launch_transfer(int comm, char* dst, const char* src, int64_t bytes, int64_t chunk, int n_ctas,
                            cudaStream_t stream);
// CTAs of the fused kernel that can be co-resident in clusters of cg (2 or 4) CTAs (-1 on error).
int max_co_resident_ctas(int cg);
cudaError_t launch_attn(const AttnArgs& args, cudaStream_t stream);

}  // namespace ao
