// runtime.cpp -- host runtime and C ABI of libautooverlap (see include/autooverlap.h).
//
//  * symmetric workspace per rank: cudaMalloc'd [data parity 0 | data parity 1 |
//    flags parity 0 | flags parity 1], exported with cudaIpcGetMemHandle and mapped by the
//    peers (cudaIpcOpenMemHandle, NVLink P2P) -- or mapped directly when the peer ctx lives
//    in the same process (loopback: several ranks on one GPU).  NVSHMEM's symmetric heap of
//    the paper is replaced by this.
//  * epochs: every op call advances the ctx epoch; data and flags of epoch e live in parity
//    e % 2, flags are written with the absolute epoch value (Q10/Q11).
//  * copy-engine backend (Fig.7a): the source rank's side stream issues one peer
//    cudaMemcpyAsync per chunk followed by cuStreamWriteValue32(flag, epoch) -- a
//    global-memory signal written without any SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "autooverlap.h"
#include "kernel_args.h"
#include "planner.h"

// --------------------------------------------------------------------------- error state
namespace {
thread_local std::string g_last_error;

ao_status fail(ao_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define AO_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess) return fail(AO_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                                       __FILE__, __LINE__);                                   \
  } while (0)

using ao::kFlagWordsPerParity;  // 1 MiB of u32 per parity (kernel_args.h)
constexpr size_t kCounterWords = size_t(1) << 16;
constexpr uint32_t kBlobMagic = 0x414f5648u;  // "AOVH"
constexpr size_t kMaxCeGraphs = 16;
constexpr size_t kControlBytes = 4096;
constexpr size_t kAnnounceOff = 256;
constexpr uint32_t kAnnounceSlots = 64;

// ------------------------------------------------------------------ driver entry points
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
typedef CUresult (*PFN_memsetD32Async)(CUdeviceptr, unsigned int, size_t, CUstream);

struct DriverFns {
  PFN_encodeTiled encode = nullptr;
  PFN_writeValue32 write32 = nullptr;
  PFN_writeValue32 wait32 = nullptr;  // cuStreamWaitValue32 (same signature)
  PFN_batchMemOp batch = nullptr;     // cuStreamBatchMemOp
  PFN_memsetD32Async memset32 = nullptr;  // cuMemsetD32Async
};

ao_status get_driver(DriverFns** out) {
  static DriverFns fns;
  static bool loaded = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!loaded) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    AO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) return fail(AO_ERR_CUDA, "cuTensorMapEncodeTiled not found");
    fns.encode = reinterpret_cast<PFN_encodeTiled>(p);
    p = nullptr;
    AO_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q));
    if (!p) return fail(AO_ERR_CUDA, "cuStreamWriteValue32 not found");
    fns.write32 = reinterpret_cast<PFN_writeValue32>(p);
    p = nullptr;
    AO_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
    if (!p) return fail(AO_ERR_CUDA, "cuStreamWaitValue32 not found");
    fns.wait32 = reinterpret_cast<PFN_writeValue32>(p);
    p = nullptr;
    AO_CUDA(cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q));
    if (!p) return fail(AO_ERR_CUDA, "cuStreamBatchMemOp not found");
    fns.batch = reinterpret_cast<PFN_batchMemOp>(p);
    p = nullptr;
    AO_CUDA(cudaGetDriverEntryPoint("cuMemsetD32Async", &p, cudaEnableDefault, &q));
    if (!p) return fail(AO_ERR_CUDA, "cuMemsetD32Async not found");
    fns.memset32 = reinterpret_cast<PFN_memsetD32Async>(p);
    loaded = true;
  }
  *out = &fns;
  return AO_OK;
}

// Random per-process identity, drawn once at first use: a peer handle is mapped directly
// (same address space) only when its token equals ours; pid + hostname can collide across
// PID namespaces that share a hostname.
struct ProcessToken {
  uint64_t a = 0, b = 0;
};
const ProcessToken& process_token() {
  static ProcessToken t = [] {
    ProcessToken x;
    FILE* f = fopen("/dev/urandom", "rb");
    bool ok = f && fread(&x, sizeof x, 1, f) == 1;
    if (f) fclose(f);
    if (!ok || (x.a == 0 && x.b == 0)) {  // fallback: time, pid and an address
      x.a = uint64_t(std::chrono::high_resolution_clock::now().time_since_epoch().count()) ^ uint64_t(getpid()) << 32;
      x.b = reinterpret_cast<uintptr_t>(&x) ^ 0x9E3779B97F4A7C15ull;
    }
    return x;
  }();
  return t;
}

struct Blob {
  uint32_t magic, version;
  int32_t pid, device, rank, world;
  uint64_t data_half, total, raw_ptr;
  ProcessToken token;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(Blob) <= AO_HANDLE_BYTES, "blob too large");

struct DebugKnobs {
  int64_t skip_wait = -1;
  int64_t delay_ns = 0;
  int64_t l2_hint = -1;  // -1: follow the plan's tile order
  int64_t gemm_group_m = 16;
  int64_t ts_lag = 0;  // time-sliced RS: lag the own run behind the next owner's first source run
  int64_t ts_owners = 1;  // time-sliced RS: owners per phase (experiment)
  int64_t gemm_stream_k = 0;  // ao_gemm: desc.stream_k of its internal plan (0 off, 1 on, -1 auto)
  int64_t prearrive = 0;  // per-rank measurement: every chunk flag of the launch's ranks is set
                          // for the coming epoch before the kernel and no copy-engine chain is
                          // issued (peers' data "already arrived"; the bench's per-GPU legs,
                          // results not checked)
  int64_t exp = 0;  // timing experiments (results invalid when nonzero)  // ao_gemm GROUP_M (measured best)
};
DebugKnobs g_debug;

}  // namespace

// ------------------------------------------------------------------------------- objects
struct ao_ctx {
  int device = 0, rank = 0, W = 1, sm_count = 0;
  size_t data_half = 0;
  size_t total = 0;
  char* base = nullptr;
  uint32_t* counters = nullptr;
  ao::ErrorInfo* err_host = nullptr;
  ao::ErrorInfo* err_dev = nullptr;
  bool imported = false;
  char* peer_base[AO_MAX_WORLD] = {};
  bool peer_opened[AO_MAX_WORLD] = {};
  uint32_t epoch = 0;
  uint32_t* epoch_cell = nullptr;   // device word holding the current epoch (CE flag source)
  ao::TraceEvent* trace = nullptr;  // device ring (AO tracing)
  uint32_t* trace_cursor = nullptr;
  uint32_t trace_cap = 0;
  uint32_t trace_seq = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;

  cudaStream_t ctl = nullptr;          // control-page copies (non-blocking: never behind an op)
  uint64_t* ctl_host = nullptr;        // pinned staging for control-page copies
  uint32_t announce_seq = 0;           // plans announced so far (collective order)

  size_t acc_half = 0;  // RS ATOMIC accumulator per parity (kept all-zero between uses)
  char* data(int q, uint32_t parity) const { return peer_base[q] + parity * data_half; }
  char* acc(int q, uint32_t parity) const { return peer_base[q] + 2 * data_half + parity * acc_half; }
  uint32_t* flags(int q, uint32_t parity) const {
    return reinterpret_cast<uint32_t*>(peer_base[q] + 2 * data_half + 2 * acc_half + parity * kFlagWordsPerParity * 4);
  }
  // Control page of rank q (kControlBytes, after both flag parities): word 0 = the last
  // epoch whose op completed on q (stream-written after each op); from byte kAnnounceOff,
  // kAnnounceSlots {tag, plan hash} pairs (collective plan-hash agreement).
  char* control(int q) const { return peer_base[q] + 2 * data_half + 2 * acc_half + 2 * kFlagWordsPerParity * 4; }
  uint32_t* done_word(int q) const { return reinterpret_cast<uint32_t*>(control(q)); }
};

struct ao_plan {
  ao::HostPlan hp;
  ao_ctx* ctx = nullptr;
  bool announced = false;  // plan hash published and compared with the peers
  int device = -1;
  char* d_tables = nullptr;
  const int* d_order = nullptr;
  const int* d_wait_off = nullptr;
  const int2* d_waits = nullptr;
  const int* d_tpc = nullptr;
  const int* d_items = nullptr;
  const ao::CommItem* d_comm = nullptr;
  int n_comm = 0;
  const int* d_comm_by_peer = nullptr;  // comm item indices grouped by peer (CSR, time-sliced walks)
  const int* d_comm_peer_off = nullptr;
  int comm_kind = ao::COMM_NONE;
  int32_t* d_a2a = nullptr;  // A2A: token permutation [W][T] | block positions [T][k] (local)
  // stream-K tail (Q28): per split position and cluster CTA, the tail piece's fp32 partial
  // [ceil(BN/32)][128][32] and a flag word (local, zeroed once; flags hold the launch count)
  char* d_sk = nullptr;
  uint32_t sk_launches = 0;
  // CE backend: instantiated copy-chain graphs keyed by (parity, group plans, A pointers)
  std::map<std::vector<uintptr_t>, cudaGraphExec_t> ce_graphs;
};

namespace {

ao_status upload_tables(ao_plan* p) {
  const ao::HostPlan& hp = p->hp;
  std::vector<int> wait_off(hp.n_cta + 1, 0);
  std::vector<int2> waits;
  for (int c = 0; c < hp.n_cta; ++c) {  // (A2A: waits are built on the device)
    if (size_t(c) < hp.waits.size())
      for (auto& w : hp.waits[c]) waits.push_back(make_int2(w[0], w[1]));
    wait_off[c + 1] = int(waits.size());
  }
  std::vector<int> items;  // (no separate reduce items: the own-tile epilogue reduces)
  // RS completion counts at 128-row sub-tile granularity (each CTA of a pair signals its
  // own half): sub-tiles of all column blocks whose rows intersect chunk g.
  std::vector<int> subtiles(hp.n_chunks, 0);
  for (int g = 0; g < hp.n_chunks; ++g) {
    const int64_t r0 = int64_t(g) * hp.C, r1 = r0 + hp.C - 1;
    subtiles[g] = int(r1 / 128 - r0 / 128 + 1) * hp.n_nb;
  }
  // in-kernel comm items (AG push, TMA / LDST backends)
  std::vector<ao::CommItem> comm;
  if (hp.is_ag && hp.desc.backend != AO_BACKEND_CE && hp.W > 1) {
    const int64_t row_bytes = hp.K * 2;
    const int64_t chunk_bytes = int64_t(hp.C) * row_bytes;
    const int ns = hp.desc.n_slices;
    const int64_t slice = ((chunk_bytes + ns - 1) / ns + 15) / 16 * 16;
    const bool pull = hp.desc.dir == AO_DIR_PULL;
    // kind, peer, global row0 of the chunk; src offset relative to the local shard (PUSH,
    // STAGE) or to the source's gathered buffer (PULL); dst offset in a gathered buffer.
    auto add_slices = [&](int32_t kind, int peer, int64_t row0) {
      for (int s = 0; s < ns; ++s) {
        ao::CommItem it{};
        it.kind = kind;
        it.peer = peer;
        it.g = int(row0 / hp.C);
        it.slice = s;
        const int64_t off = std::min<int64_t>(int64_t(s) * slice, chunk_bytes);
        it.bytes = std::max<int64_t>(0, std::min<int64_t>(slice, chunk_bytes - off));
        it.src_off = (kind == ao::ITEM_PULL ? row0 : row0 - int64_t(hp.rank) * hp.S) * row_bytes + off;
        it.dst_off = row0 * row_bytes + off;
        comm.push_back(it);
      }
    };
    if (pull) {
      // PULL (Lst.2 P:249-265 with the issuer on the consumer side): stage the own
      // shard in the own gathered buffer first (every worker's first items, so no pull can
      // wait on a stage queued behind it), then fetch the peers' chunks in plan order.
      for (int64_t j = 0; j < hp.S / hp.C; ++j) add_slices(ao::ITEM_STAGE, hp.rank, int64_t(hp.rank) * hp.S + j * hp.C);
      for (const ao::P2POp& op : hp.plans[hp.rank]) add_slices(ao::ITEM_PULL, op.peer, op.row0);
    } else {
      for (const ao::P2POp& op : hp.plans[hp.rank]) add_slices(ao::ITEM_PUSH, op.peer, op.row0);
    }
    p->comm_kind = hp.desc.backend == AO_BACKEND_TMA ? ao::COMM_TMA : ao::COMM_LDST;
  }
  if (hp.is_ar && hp.W > 1) {
    // GEMM-AR gather (Fig.4d): pull each other owner's reduced chunk, in plan order, from the
    // owner's reduced region into this rank's C (slices spread over the gather warps).
    const int64_t row_bytes = hp.N * 2;
    const int64_t chunk_bytes = int64_t(hp.C) * row_bytes;
    const int ns = hp.desc.n_slices;
    const int64_t slice = ((chunk_bytes + ns - 1) / ns + 15) / 16 * 16;
    const int64_t red_off = int64_t(ao::ar_reduced_offset(hp.desc));
    for (const ao::P2POp& op : hp.plans[hp.rank]) {
      if (op.tensor != ao::TENSOR_C) continue;
      for (int sl = 0; sl < ns; ++sl) {
        ao::CommItem it{};
        it.kind = ao::ITEM_AR_PULL;
        it.peer = op.peer;
        it.g = int(op.row0 / hp.C);
        it.slice = sl;
        const int64_t off = std::min<int64_t>(int64_t(sl) * slice, chunk_bytes);
        it.bytes = std::max<int64_t>(0, std::min<int64_t>(slice, chunk_bytes - off));
        it.src_off = red_off + (op.row0 - int64_t(op.peer) * hp.S) * row_bytes + off;
        it.dst_off = op.row0 * row_bytes + off;
        comm.push_back(it);
      }
    }
  }
  p->n_comm = int(comm.size());
  // comm items grouped by peer (stable): time-sliced groups serve them peer (destination /
  // owner) after peer without scanning the item list
  std::vector<int> by_peer(comm.size()), peer_off(AO_MAX_WORLD + 1, 0);
  for (const ao::CommItem& it : comm) ++peer_off[it.peer + 1];
  for (int q = 0; q < AO_MAX_WORLD; ++q) peer_off[q + 1] += peer_off[q];
  {
    std::vector<int> fill(peer_off.begin(), peer_off.end() - 1);
    for (size_t i = 0; i < comm.size(); ++i) by_peer[fill[comm[i].peer]++] = int(i);
  }

  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t o_order = 0;
  const size_t o_woff = o_order + al(hp.order.size() * 4 + 4);
  const size_t o_waits = o_woff + al(wait_off.size() * 4);
  const size_t o_tpc = o_waits + al(waits.size() * 8 + 8);
  const size_t o_items = o_tpc + al(subtiles.size() * 4 + 4);
  const size_t o_comm = o_items + al(items.size() * 4 + 4);
  const size_t o_bypeer = o_comm + al(comm.size() * sizeof(ao::CommItem) + 16);
  const size_t o_peeroff = o_bypeer + al(by_peer.size() * 4 + 4);
  const size_t total = o_peeroff + al(peer_off.size() * 4);
  std::vector<char> h(total, 0);
  memcpy(h.data() + o_order, hp.order.data(), hp.order.size() * 4);
  memcpy(h.data() + o_woff, wait_off.data(), wait_off.size() * 4);
  if (!waits.empty()) memcpy(h.data() + o_waits, waits.data(), waits.size() * 8);
  if (!subtiles.empty()) memcpy(h.data() + o_tpc, subtiles.data(), subtiles.size() * 4);
  if (!items.empty()) memcpy(h.data() + o_items, items.data(), items.size() * 4);
  if (!comm.empty()) memcpy(h.data() + o_comm, comm.data(), comm.size() * sizeof(ao::CommItem));
  if (!by_peer.empty()) memcpy(h.data() + o_bypeer, by_peer.data(), by_peer.size() * 4);
  memcpy(h.data() + o_peeroff, peer_off.data(), peer_off.size() * 4);
  AO_CUDA(cudaMalloc(&p->d_tables, total));
  AO_CUDA(cudaMemcpy(p->d_tables, h.data(), total, cudaMemcpyHostToDevice));
  p->d_order = reinterpret_cast<const int*>(p->d_tables + o_order);
  p->d_wait_off = reinterpret_cast<const int*>(p->d_tables + o_woff);
  p->d_waits = reinterpret_cast<const int2*>(p->d_tables + o_waits);
  p->d_tpc = reinterpret_cast<const int*>(p->d_tables + o_tpc);
  p->d_items = reinterpret_cast<const int*>(p->d_tables + o_items);
  p->d_comm = reinterpret_cast<const ao::CommItem*>(p->d_tables + o_comm);
  p->d_comm_by_peer = reinterpret_cast<const int*>(p->d_tables + o_bypeer);
  p->d_comm_peer_off = reinterpret_cast<const int*>(p->d_tables + o_peeroff);
  if (hp.sk_dp < hp.n_tiles) {
    const size_t slots = size_t(hp.n_tiles - hp.sk_dp) * hp.tile.cg;
    const size_t bytes = slots * ((hp.tile.bn + 31) / 32) * 128 * 32 * 4 + slots * 4;
    AO_CUDA(cudaMalloc(&p->d_sk, bytes));
    AO_CUDA(cudaMemset(p->d_sk, 0, bytes));
  }
  return AO_OK;
}

ao_status encode_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows, bool fp32 = false) {
  DriverFns* drv;
  ao_status s = get_driver(&drv);
  if (s != AO_OK) return s;
  const int eb = fp32 ? 4 : 2;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * eb};
  cuuint32_t box[2] = {cuuint32_t(128 / eb), cuuint32_t(box_rows)};  // 128-byte inner box (swizzle span)
  cuuint32_t es[2] = {1, 1};
  CUresult r = drv->encode(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(AO_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (%d) for %p [%lld x %lld]", int(r), ptr,
                (long long)rows, (long long)cols);
  return AO_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

ao_status check_device_sm100(int device, int* sm_count) {
  // cudaDeviceGetAttribute is cheap (cudaGetDeviceProperties costs milliseconds per call)
  int major = 0, minor = 0, sms = 0;
  AO_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  AO_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  AO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (major != 10 || minor != 0)
    return fail(AO_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only", device, major,
                minor);
  *sm_count = sms;
  return AO_OK;
}

ao_status take_async_error(ao_ctx* ctx) {
  if (ctx && ctx->err_host && ctx->err_host->flag) {
    const ao::ErrorInfo e = *ctx->err_host;
    ctx->err_host->flag = 0;
    ctx->err_host->claim = 0;
    if (e.cta == ao::kErrBadRouting)
      return fail(AO_ERR_INVALID_ARG, "a2a_gemm: rank %d token %d choice %u has expert id %d: topk_idx must hold "
                  "k distinct ids in [0, world_size) (the entry was dropped, route_pos = -1)", e.rank, e.chunk,
                  e.epoch, int(e.seen));
    return fail(AO_ERR_TIMEOUT, "device spin-wait timed out: rank %d cta %d chunk %d epoch %u (flag held %u)", e.rank,
                e.cta, e.chunk, e.epoch, e.seen);
  }
  return AO_OK;
}

// Fill the rank-dependent part of the kernel args for one call.
ao_status fill_rank(ao::RankArgs* R, ao_plan* p, uint32_t epoch, const void* A, const void* B, void* C) {
  const ao::HostPlan& hp = p->hp;
  ao_ctx* ctx = p->ctx;
  const uint32_t par = epoch & 1;
  memset(R, 0, sizeof(*R));
  R->order = p->d_order;
  R->wait_off = p->d_wait_off;
  R->waits = p->d_waits;
  R->tiles_per_chunk = p->d_tpc;
  R->reduce_items = p->d_items;
  R->comm_items = p->d_comm;
  R->n_comm_items = p->n_comm;
  R->comm_by_peer = p->d_comm_by_peer;
  R->comm_peer_off = p->d_comm_peer_off;
  R->C = C;
  R->M = hp.M;
  R->N = hp.N;
  R->K = hp.K;
  R->S = hp.S;
  R->rank = hp.rank;
  R->W = hp.W;
  R->crows = hp.C;
  R->n_chunks = hp.n_chunks;
  R->n_tiles = hp.n_tiles;
  R->n_items = 0;
  R->n_nb = hp.n_nb;
  R->n_slices = hp.desc.backend == AO_BACKEND_CE ? 1 : hp.desc.n_slices;
  R->n_cta = hp.n_cta;
  R->epoch = epoch;
  R->rs_atomic = (!hp.is_ag && hp.desc.rs_reduce == AO_RS_ATOMIC) ? 1 : 0;
  R->rs_bf16 = (R->rs_atomic && hp.desc.rs_wire == AO_WIRE_BF16) ? 1 : 0;
  R->sk_dp = hp.sk_dp;
  if (p->d_sk) {
    const size_t slots = size_t(hp.n_tiles - hp.sk_dp) * hp.tile.cg;
    R->sk_ws = reinterpret_cast<float*>(p->d_sk);
    R->sk_flags = reinterpret_cast<uint32_t*>(p->d_sk + slots * ((hp.tile.bn + 31) / 32) * 128 * 32 * 4);
    R->sk_seq = ++p->sk_launches;
  }
  R->counters = ctx ? ctx->counters : nullptr;
  if (ctx) {
    for (int q = 0; q < hp.W; ++q) {
      R->peer_data[q] = ctx->data(q, par);
      R->peer_acc[q] = ctx->acc(q, par);
      R->peer_flags[q] = ctx->flags(q, par);
    }
    R->flags = R->peer_flags[hp.rank];
  }
  const int bn = hp.tile.bn;
  ao_status s;
  if (hp.is_a2a && ctx) {
    // receive buffer [W*T, K] (current parity) is the GEMM's A; the caller's X is the
    // source of the dispatch row gathers
    R->A_shard = static_cast<const char*>(A);
    R->a2a_perm = p->d_a2a;
    R->T = int32_t(hp.M);
    R->topk = hp.desc.topk;
    R->maxJ = hp.n_c;
    R->gm = hp.desc.intra == AO_INTRA_GROUPED ? std::max(1, hp.desc.group_m) : 1;
    if (hp.K > 0) {
      s = encode_2d(&R->tmA, R->peer_data[hp.rank], int64_t(hp.W) * hp.M, hp.K, 128);
      if (s != AO_OK) return s;
      s = encode_2d(&R->tmB, B, hp.N, hp.K, bn / hp.tile.cg);
      if (s != AO_OK) return s;
    }
    return AO_OK;
  }
  if (hp.K > 0) {
    if (hp.is_ag && ctx) {
      s = encode_2d(&R->tmA, R->peer_data[hp.rank], hp.M, hp.K, 128);
      if (s != AO_OK) return s;
      s = encode_2d(&R->tmA_loc, A, hp.S, hp.K, 128);
      if (s != AO_OK) return s;
      R->A_shard = static_cast<const char*>(A);
    } else {
      s = encode_2d(&R->tmA, A, hp.M, hp.K, 128);
      if (s != AO_OK) return s;
    }

    s = encode_2d(&R->tmB, B, hp.N, hp.K, bn / hp.tile.cg);
    if (s != AO_OK) return s;
  }
  if (!hp.is_ag && ctx && hp.W > 1 && hp.N > 0 && hp.S > 0) {  // RS: peer partials, streamed by the producer
    if (R->rs_atomic) {
      // accumulator boxes: 32 rows x 128 bytes (32 fp32, or 64 bf16 with the bf16 wire)
      const bool f32 = !R->rs_bf16;
      s = encode_2d(&R->tmA_loc, R->peer_acc[hp.rank], hp.S, hp.N, 128, f32);
      for (int q = 0; q < hp.W && s == AO_OK; ++q) s = encode_2d(&R->tmAcc[q], R->peer_acc[q], hp.S, hp.N, 32, f32);
    } else
      s = encode_2d(&R->tmA_loc, R->peer_data[hp.rank], int64_t(hp.W) * hp.S, hp.N, 128, true);
    if (s != AO_OK) return s;
  }
  R->C = C;
  if (hp.is_ar) {
    // the own rows of the full output are written by the fused reduction like a C_shard
    R->ar = 1;
    R->ar_out = static_cast<char*>(C);
    R->C = static_cast<char*>(C) + int64_t(hp.rank) * hp.S * hp.N * 2;
    if (ctx) R->ar_red = R->peer_data[hp.rank] + ao::ar_reduced_offset(hp.desc);
  }
  return AO_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char* ao_status_string(ao_status s) {
  switch (s) {
    case AO_OK: return "AO_OK";
    case AO_ERR_INVALID_ARG: return "AO_ERR_INVALID_ARG";
    case AO_ERR_UNSUPPORTED: return "AO_ERR_UNSUPPORTED";
    case AO_ERR_CUDA: return "AO_ERR_CUDA";
    case AO_ERR_OOM: return "AO_ERR_OOM";
    case AO_ERR_PEER: return "AO_ERR_PEER";
    case AO_ERR_TIMEOUT: return "AO_ERR_TIMEOUT";
    case AO_ERR_STATE: return "AO_ERR_STATE";
  }
  return "AO_ERR_UNKNOWN";
}

const char* ao_last_error(void) { return g_last_error.c_str(); }

ao_status ao_version(int* major, int* minor) {
  if (major) *major = AO_VERSION_MAJOR;
  if (minor) *minor = AO_VERSION_MINOR;
  return AO_OK;
}

ao_status ao_debug_set(const char* key, int64_t value) {
  if (!key) return fail(AO_ERR_INVALID_ARG, "null key");
  if (!strcmp(key, "skip_wait")) g_debug.skip_wait = value;
  else if (!strcmp(key, "delay_ns")) g_debug.delay_ns = value;
  else if (!strcmp(key, "l2_hint")) g_debug.l2_hint = value;
  else if (!strcmp(key, "gemm_group_m")) g_debug.gemm_group_m = value;
  else if (!strcmp(key, "exp")) g_debug.exp = value;
  else if (!strcmp(key, "ts_lag")) g_debug.ts_lag = value;
  else if (!strcmp(key, "ts_owners")) g_debug.ts_owners = value;
  else if (!strcmp(key, "gemm_stream_k")) g_debug.gemm_stream_k = value;
  else if (!strcmp(key, "prearrive")) g_debug.prearrive = value;
  else return fail(AO_ERR_INVALID_ARG, "unknown debug key %s", key);
  return AO_OK;
}

ao_status ao_plan_desc_init(ao_plan_desc* d) {
  if (!d) return fail(AO_ERR_INVALID_ARG, "null desc");
  memset(d, 0, sizeof(*d));
  d->struct_size = sizeof(ao_plan_desc);
  d->op = AO_OP_AG_GEMM;
  d->world_size = 1;
  d->rank = 0;
  d->chunk_rows = 128;
  d->backend = AO_BACKEND_CE;
  d->dir = AO_DIR_PUSH;
  d->chunk_order = AO_CHUNK_SHARD_MAJOR;
  d->intra = AO_INTRA_ROW;
  d->group_m = 1;
  d->n_slices = 1;
  d->rs_wire = AO_WIRE_FP32;
  return AO_OK;
}

ao_status ao_plan_validate(const ao_plan_desc* d, int sm_count, char* report, size_t cap, int* n_violations) {
  if (!d) return fail(AO_ERR_INVALID_ARG, "null desc");
  std::vector<std::string> v = ao::validate_desc(*d, sm_count > 0 ? sm_count : 148);
  std::string joined;
  for (size_t i = 0; i < v.size(); ++i) joined += (i ? ";" : "") + v[i];
  if (report && cap) {
    strncpy(report, joined.c_str(), cap - 1);
    report[cap - 1] = 0;
  }
  if (n_violations) *n_violations = int(v.size());
  if (!v.empty()) return fail(AO_ERR_INVALID_ARG, "invalid plan desc: %s", joined.c_str());
  return AO_OK;
}

ao_status ao_plan_create_host(const ao_plan_desc* d, int sm_count, ao_plan** out) {
  if (!d || !out) return fail(AO_ERR_INVALID_ARG, "null argument");
  std::unique_ptr<ao_plan> p(new ao_plan());
  std::vector<std::string> v = ao::build_plan(*d, sm_count > 0 ? sm_count : 148, &p->hp);
  if (!v.empty()) {
    std::string joined;
    for (size_t i = 0; i < v.size(); ++i) joined += (i ? ";" : "") + v[i];
    return fail(AO_ERR_INVALID_ARG, "invalid plan desc: %s", joined.c_str());
  }
  *out = p.release();
  if (d->rs_wire == AO_WIRE_BF16)
    fail(AO_OK, "non-conforming: rs_wire bf16 (DESIGN.md Q14)");
  return AO_OK;
}

ao_status ao_plan_export_json(const ao_plan* p, char* buf, size_t cap, size_t* needed) {
  if (!p) return fail(AO_ERR_INVALID_ARG, "null plan");
  const std::string& s = p->hp.json;
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return AO_OK;
}

ao_status ao_plan_hash(const ao_plan* p, uint64_t* out) {
  if (!p || !out) return fail(AO_ERR_INVALID_ARG, "null argument");
  *out = p->hp.hash;
  return AO_OK;
}

ao_status ao_plan_info(const ao_plan* p, int32_t* tile_m, int32_t* tile_n, int32_t* cta_group, int32_t* n_cta,
                       int32_t* n_tiles, int32_t* n_chunks) {
  if (!p) return fail(AO_ERR_INVALID_ARG, "null plan");
  if (tile_m) *tile_m = p->hp.tile.bm;
  if (tile_n) *tile_n = p->hp.tile.bn;
  if (cta_group) *cta_group = p->hp.tile.cg;
  if (n_cta) *n_cta = p->hp.n_cta;
  if (n_tiles) *n_tiles = p->hp.n_tiles;
  if (n_chunks) *n_chunks = p->hp.n_chunks;
  return AO_OK;
}

ao_status ao_plan_workspace_bytes(const ao_plan_desc* d, size_t* bytes) {
  if (!d || !bytes) return fail(AO_ERR_INVALID_ARG, "null argument");
  *bytes = 2 * ao::data_bytes_per_parity(*d);
  return AO_OK;
}

ao_status ao_plan_destroy(ao_plan* p) {
  if (!p) return AO_OK;
  if (p->d_tables) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    for (auto& kv : p->ce_graphs) cudaGraphExecDestroy(kv.second);
    cudaFree(p->d_tables);
    if (p->d_a2a) cudaFree(p->d_a2a);
    if (p->d_sk) cudaFree(p->d_sk);
    cudaSetDevice(cur);
  }
  delete p;
  return AO_OK;
}

// ---------------------------------------------------------------------------- contexts
ao_status ao_ctx_create(int device, int rank, int world_size, size_t workspace_bytes, ao_ctx** out) {
  if (!out) return fail(AO_ERR_INVALID_ARG, "null out");
  if (world_size < 1 || world_size > AO_MAX_WORLD || rank < 0 || rank >= world_size)
    return fail(AO_ERR_INVALID_ARG, "bad rank/world (%d/%d)", rank, world_size);
  int sm = 0;
  AO_CUDA(cudaSetDevice(device));
  ao_status s = check_device_sm100(device, &sm);
  if (s != AO_OK) return s;
  std::unique_ptr<ao_ctx> c(new ao_ctx());
  c->device = device;
  c->rank = rank;
  c->W = world_size;
  c->sm_count = sm;
  c->data_half = (workspace_bytes / 2 + 4095) / 4096 * 4096;
  // RS ATOMIC accumulator: an owner's [S, N] fp32 is 1/W of the slots an RS plan of the
  // same shape needs, so data_half / W always suffices.
  c->acc_half = (c->data_half / world_size + 4095) / 4096 * 4096;
  c->total = 2 * c->data_half + 2 * c->acc_half + 2 * kFlagWordsPerParity * 4 + kControlBytes;
  cudaError_t e = cudaMalloc(&c->base, c->total);
  if (e != cudaSuccess) return fail(AO_ERR_OOM, "cudaMalloc(%zu): %s", c->total, cudaGetErrorString(e));
  AO_CUDA(cudaMemset(c->base + 2 * c->data_half, 0, 2 * c->acc_half + 2 * kFlagWordsPerParity * 4 + kControlBytes));
  AO_CUDA(cudaStreamCreateWithFlags(&c->ctl, cudaStreamNonBlocking));
  AO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->ctl_host), 64, cudaHostAllocDefault));
  AO_CUDA(cudaMalloc(&c->epoch_cell, 64));
  AO_CUDA(cudaMemset(c->epoch_cell, 0, 64));
  AO_CUDA(cudaMalloc(&c->counters, kCounterWords * 4));
  AO_CUDA(cudaMemset(c->counters, 0, kCounterWords * 4));
  AO_CUDA(cudaHostAlloc(&c->err_host, sizeof(ao::ErrorInfo), cudaHostAllocMapped));
  memset(c->err_host, 0, sizeof(ao::ErrorInfo));
  AO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0));
  AO_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  AO_CUDA(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  AO_CUDA(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  AO_CUDA(cudaDeviceSynchronize());
  c->peer_base[rank] = c->base;
  if (world_size == 1) c->imported = true;
  *out = c.release();
  return AO_OK;
}

ao_status ao_ctx_export_handle(ao_ctx* c, ao_handle_blob* out) {
  if (!c || !out) return fail(AO_ERR_INVALID_ARG, "null argument");
  memset(out, 0, sizeof(*out));
  Blob b{};
  b.magic = kBlobMagic;
  b.version = AO_VERSION_MAJOR * 100 + AO_VERSION_MINOR;
  b.pid = int32_t(getpid());
  b.device = c->device;
  b.rank = c->rank;
  b.world = c->W;
  b.data_half = c->data_half;
  b.total = c->total;
  b.raw_ptr = reinterpret_cast<uint64_t>(c->base);
  b.token = process_token();
  AO_CUDA(cudaSetDevice(c->device));
  AO_CUDA(cudaIpcGetMemHandle(&b.ipc, c->base));
  memcpy(out->bytes, &b, sizeof b);
  return AO_OK;
}

ao_status ao_ctx_import_handles(ao_ctx* c, const ao_handle_blob* all) {
  if (!c || !all) return fail(AO_ERR_INVALID_ARG, "null argument");
  AO_CUDA(cudaSetDevice(c->device));
  const ProcessToken me = process_token();
  for (int q = 0; q < c->W; ++q) {
    if (q == c->rank) continue;
    Blob b;
    memcpy(&b, all[q].bytes, sizeof b);
    if (b.magic != kBlobMagic) return fail(AO_ERR_PEER, "handle %d: bad magic", q);
    if (b.rank != q || b.world != c->W) return fail(AO_ERR_PEER, "handle %d: rank/world mismatch (%d/%d)", q, b.rank, b.world);
    if (b.data_half != c->data_half || b.total != c->total)
      return fail(AO_ERR_PEER, "handle %d: workspace size mismatch (%llu vs %llu)", q,
                  (unsigned long long)b.data_half, (unsigned long long)c->data_half);
    if (b.token.a == me.a && b.token.b == me.b) {
      if (b.device != c->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(AO_ERR_CUDA, "peer access %d->%d: %s", c->device, b.device, cudaGetErrorString(e));
        cudaGetLastError();
      }
      c->peer_base[q] = reinterpret_cast<char*>(b.raw_ptr);
      c->peer_opened[q] = false;
    } else {
      void* p = nullptr;
      AO_CUDA(cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess));
      c->peer_base[q] = static_cast<char*>(p);
      c->peer_opened[q] = true;
    }
  }
  c->imported = true;
  return AO_OK;
}

ao_status ao_ctx_check_async(ao_ctx* c) {
  if (!c) return fail(AO_ERR_INVALID_ARG, "null ctx");
  return take_async_error(c);
}

ao_status ao_ctx_destroy(ao_ctx* c) {
  if (!c) return AO_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < c->W; ++q)
    if (c->peer_opened[q]) cudaIpcCloseMemHandle(c->peer_base[q]);
  if (c->base) cudaFree(c->base);
  if (c->counters) cudaFree(c->counters);
  if (c->epoch_cell) cudaFree(c->epoch_cell);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->trace) cudaFree(c->trace);
  if (c->trace_cursor) cudaFree(c->trace_cursor);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ctl) cudaStreamDestroy(c->ctl);
  if (c->ctl_host) cudaFreeHost(c->ctl_host);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  delete c;
  return AO_OK;
}

ao_status ao_ctx_trace_enable(ao_ctx* c, int64_t capacity) {
  if (!c || capacity < 0) return fail(AO_ERR_INVALID_ARG, "bad argument");
  AO_CUDA(cudaSetDevice(c->device));
  AO_CUDA(cudaDeviceSynchronize());
  if (c->trace) cudaFree(c->trace);
  if (c->trace_cursor) cudaFree(c->trace_cursor);
  c->trace = nullptr;
  c->trace_cursor = nullptr;
  c->trace_cap = 0;
  if (capacity == 0) return AO_OK;
  AO_CUDA(cudaMalloc(&c->trace, size_t(capacity) * sizeof(ao::TraceEvent)));
  AO_CUDA(cudaMalloc(&c->trace_cursor, 4));
  AO_CUDA(cudaMemset(c->trace_cursor, 0, 4));
  c->trace_cap = uint32_t(capacity);
  return AO_OK;
}

ao_status ao_ctx_trace_dump(ao_ctx* c, const char* path, int64_t* n_events) {
  static const char* kinds[] = {"?", "wait", "load", "mma", "epilogue", "comm", "reduce", "reduce_wait", "clock"};
  if (!c || !path) return fail(AO_ERR_INVALID_ARG, "bad argument");
  if (!c->trace) return fail(AO_ERR_STATE, "tracing is not enabled on this ctx");
  AO_CUDA(cudaSetDevice(c->device));
  AO_CUDA(cudaDeviceSynchronize());
  uint32_t n = 0;
  AO_CUDA(cudaMemcpy(&n, c->trace_cursor, 4, cudaMemcpyDeviceToHost));
  n = std::min(n, c->trace_cap);
  std::vector<ao::TraceEvent> ev(n);
  if (n) AO_CUDA(cudaMemcpy(ev.data(), c->trace, n * sizeof(ao::TraceEvent), cudaMemcpyDeviceToHost));
  AO_CUDA(cudaMemset(c->trace_cursor, 0, 4));
  c->trace_seq = 0;
  uint64_t tmin = ~0ull;
  for (auto& e : ev) tmin = std::min(tmin, e.t0);
  FILE* f = fopen(path, "w");
  if (!f) return fail(AO_ERR_INVALID_ARG, "cannot open %s", path);
  fprintf(f, "{\"traceEvents\":[");
  for (uint32_t i = 0; i < n; ++i) {
    const ao::TraceEvent& e = ev[i];
    const uint32_t kk = e.kind & 0xff, seq = e.kind >> 8;
    const char* k = kk < 9 ? kinds[kk] : "?";  // "clock": id = SM cycles over the event (an MMA span)
    fprintf(f,
            "%s{\"name\":\"%s %u\",\"cat\":\"%s\",\"ph\":\"X\",\"ts\":%.3f,\"dur\":%.3f,\"pid\":%u,\"tid\":%u,"
            "\"args\":{\"launch\":%u}}",
            i ? "," : "", k, e.id, k, (e.t0 - tmin) / 1000.0, (e.t1 - e.t0) / 1000.0, e.rank, e.cta * 8 + kk, seq);
  }
  fprintf(f, "]}\n");
  fclose(f);
  if (n_events) *n_events = n;
  return AO_OK;
}

ao_status ao_plan_create(ao_ctx* c, const ao_plan_desc* d, ao_plan** out) {
  if (!c || !d || !out) return fail(AO_ERR_INVALID_ARG, "null argument");
  if (d->world_size != c->W || d->rank != c->rank)
    return fail(AO_ERR_INVALID_ARG, "desc rank/world (%d/%d) != ctx (%d/%d)", d->rank, d->world_size, c->rank, c->W);
  AO_CUDA(cudaSetDevice(c->device));
  ao_plan* p = nullptr;
  ao_status s = ao_plan_create_host(d, c->sm_count, &p);
  if (s != AO_OK) return s;
  std::unique_ptr<ao_plan> guard(p);
  if (ao::data_bytes_per_parity(*d) > c->data_half)
    return fail(AO_ERR_INVALID_ARG, "workspace too small: plan needs %zu bytes per parity, ctx has %zu",
                ao::data_bytes_per_parity(*d), c->data_half);
  if (d->op == AO_OP_GEMM_RS && d->rs_reduce == AO_RS_ATOMIC &&
      size_t(d->M / d->world_size) * size_t(d->N) * (d->rs_wire == AO_WIRE_BF16 ? 2 : 4) > c->acc_half)
    return fail(AO_ERR_INVALID_ARG, "workspace too small for the RS accumulator");
  if (ao::flag_words_needed(*d) > ao::kA2ACountFlags)
    return fail(AO_ERR_INVALID_ARG, "too many chunk flags (%zu)", ao::flag_words_needed(*d));
  if (size_t(p->hp.n_chunks) > kCounterWords) return fail(AO_ERR_INVALID_ARG, "too many chunks");
  if (p->hp.is_a2a) {
    if (p->hp.n_mb > 128)
      return fail(AO_ERR_INVALID_ARG, "a2a_gemm: W*T / tile_m = %d row blocks exceeds 128", p->hp.n_mb);
    const size_t n = size_t(d->world_size) * size_t(d->M) + size_t(d->M) * size_t(d->topk);
    AO_CUDA(cudaMalloc(&p->d_a2a, std::max<size_t>(n, 1) * 4));
  }
  p->ctx = c;
  p->device = c->device;
  s = upload_tables(p);
  if (s != AO_OK) return s;
  *out = guard.release();
  if (d->rs_wire == AO_WIRE_BF16)  // accepted, flagged; the status stays AO_OK
    fail(AO_OK, "non-conforming: rs_wire bf16 rounds each partial and the owner's accumulator to bf16, "
         "outside the 1e-2 per-element / 2e-3 Frobenius bound (DESIGN.md Q14)");
  return AO_OK;
}


// ------------------------------------------------------------- collective plan agreement
// SURVEY.md §8(b) "Collective semantics": the first launch of a plan publishes its hash in
// the rank's control page (slot = the ctx's announce sequence number mod kAnnounceSlots,
// tagged seq + 1) and compares it with every peer's announcement of the same sequence
// number -> AO_ERR_PEER on a mismatch.  Peers in other processes are waited for (bounded
// by the plan's timeout; each first launch blocks until every peer announced, so no rank
// runs more than one announcement ahead); co-located peers (same process, maybe called
// later by this same thread) are compared only if they have already announced.
static ao_status announce_plans(int n, ao_plan* const* plans) {
  std::vector<int> todo;
  std::vector<uint32_t> seq(n, 0);
  for (int i = 0; i < n; ++i)
    if (!plans[i]->announced) todo.push_back(i);
  for (int i : todo) {  // publish every member of the group first
    ao_ctx* c = plans[i]->ctx;
    seq[i] = c->announce_seq++;
    plans[i]->announced = true;
    if (c->W == 1) continue;
    c->ctl_host[0] = uint64_t(seq[i]) + 1;
    c->ctl_host[1] = plans[i]->hp.hash;
    AO_CUDA(cudaMemcpyAsync(c->control(c->rank) + kAnnounceOff + (seq[i] % kAnnounceSlots) * 16, c->ctl_host, 16,
                            cudaMemcpyHostToDevice, c->ctl));
    AO_CUDA(cudaStreamSynchronize(c->ctl));
  }
  for (int i : todo) {
    ao_ctx* c = plans[i]->ctx;
    const uint64_t tag = uint64_t(seq[i]) + 1, h = plans[i]->hp.hash;
    const uint64_t tmo = plans[i]->hp.desc.timeout_ns ? plans[i]->hp.desc.timeout_ns : 5000000000ull;
    for (int q = 0; q < c->W; ++q) {
      if (q == c->rank) continue;
      const char* src = c->control(q) + kAnnounceOff + (seq[i] % kAnnounceSlots) * 16;
      const auto t0 = std::chrono::steady_clock::now();
      while (true) {
        AO_CUDA(cudaMemcpyAsync(c->ctl_host + 2, src, 16, cudaMemcpyDeviceToHost, c->ctl));
        AO_CUDA(cudaStreamSynchronize(c->ctl));
        if (c->ctl_host[2] == tag) {
          if (c->ctl_host[3] != h)
            return fail(AO_ERR_PEER,
                        "collective plan mismatch: rank %d launches plan #%u with hash %016llx, rank %d with "
                        "%016llx (every rank must issue the same ops with plans that differ only in rank)",
                        c->rank, seq[i], (unsigned long long)h, q, (unsigned long long)c->ctl_host[3]);
          break;
        }
        if (!c->peer_opened[q]) break;  // co-located peer that has not announced yet
        const uint64_t el = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                         std::chrono::steady_clock::now() - t0).count());
        if (el > tmo)
          return fail(AO_ERR_TIMEOUT, "rank %d did not announce plan #%u within the timeout (collective op "
                      "sequence out of step?)", q, seq[i]);
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      }
    }
  }
  return AO_OK;
}

// Done words: after every op, each rank of the launch records (stream-ordered, one batched
// memop) the epoch whose op has now completed on it.  An op whose waits do not cover every
// peer (causal SP attention: a rank waits only on lower ranks) cannot rely on the Q11
// argument and waits on these before overwriting a peer's parity buffer.
static ao_status mark_done(int n, ao_plan* const* plans, const std::vector<uint32_t>& epochs, cudaStream_t stream) {
  if (plans[0]->hp.W == 1) return AO_OK;
  DriverFns* drv = nullptr;
  ao_status s = get_driver(&drv);
  if (s != AO_OK) return s;
  CUstreamBatchMemOpParams ops[AO_MAX_WORLD];
  memset(ops, 0, sizeof ops);
  for (int i = 0; i < n; ++i) {
    ao_ctx* c = plans[i]->ctx;
    ops[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    ops[i].writeValue.address = reinterpret_cast<CUdeviceptr>(c->done_word(c->rank));
    ops[i].writeValue.value = epochs[i];
    ops[i].writeValue.flags = 0;
  }
  CUresult r = drv->batch(stream, unsigned(n), ops, 0);
  if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamBatchMemOp failed (%d)", int(r));
  return AO_OK;
}

// ------------------------------------------------------------------ time-sliced groups
// A whole-world loopback group whose plans each ask for more CTAs than SMs / n runs
// TIME-SLICED: all n_cta (x cta_group) CTAs serve every rank, walking one global list of
// (rank, positions) segments; each rank's tiles keep their plan order.  The list order:
//  * AG (copy engine, push): rank after rank (each rank's weight shard stays L2-resident
//    while its tiles run); the copy-engine chains are issued destination-major in the same
//    order so each rank's chunks land before its turn.
//  * RS: owner after owner; for owner o the other ranks' runs of tiles whose rows o owns
//    (rotation o+1, o+2, ...; odd owners in reverse, the serpentine), then o's own run (the
//    fused reduction) last in the phase (debug ts_lag: behind the next owner's first source
//    runs instead -- measured slower).  Every tile that waits (an own tile) comes after all
//    the tiles it waits for, so with all CTAs co-resident the list drains without deadlock
//    (induction on the list index).
//  * GEMM (batched GEMM-only leg): problem after problem.
// Chunk waits are taken per tile in the kernel (the plan's per-CTA wait table assumes the
// space-sliced CTA assignment).  Returns false (and no segments) when not applicable.
static bool build_segments(int n, ao_plan* const* plans, int mode, ao::KernelArgs* ka) {
  std::vector<ao::Seg> segs;
  const ao::HostPlan& h0 = plans[0]->hp;
  const int64_t BM = int64_t(h0.tile.bm);
  if (mode == ao::MODE_RS) {
    if (h0.S % BM != 0) return false;
    struct Run { int key0, key1, key2, k0; ao::Seg s; };
    const int G = int(std::max<int64_t>(1, g_debug.ts_owners));
    std::vector<Run> runs;
    for (int i = 0; i < n; ++i) {
      const ao::HostPlan& hp = plans[i]->hp;
      int k = 0;
      while (k < hp.n_tiles) {
        const int owner = int((int64_t(hp.order[k] / hp.n_nb) * BM) / hp.S);
        int k1 = k + 1;
        while (k1 < hp.n_tiles && int((int64_t(hp.order[k1] / hp.n_nb) * BM) / hp.S) == owner) ++k1;
        // non-own run: slot 2*rot of its owner's phase (rot = 1..W-1, the rotation o+1, o+2...);
        // own run of owner o: lagged into the next owner's phase after its first source run
        // (slot 3 of phase o+1), so its contributions have drained when its waits run
        const int rot = ((hp.rank - owner) % hp.W + hp.W) % hp.W;
        const bool own = owner == hp.rank;
        if (G > 1) {  // experiment: G owners per phase, each source's runs of the phase together
          const int ph = owner / G;
          const int srot = ((hp.rank - ph * G) % hp.W + hp.W) % hp.W;
          runs.push_back({ph, own ? 2 * hp.W : 2 * srot, owner, k, {i, k, k1, 0}});
        } else if (g_debug.ts_lag)  // behind the first ts_lag source runs of the next owner's phase
          runs.push_back({own ? owner + 1 : owner, own ? 2 * int(g_debug.ts_lag) + 1 : 2 * rot, 0, k, {i, k, k1, 0}});
        else  // odd owners run their sources in reverse rotation (serpentine): each phase starts
              // with the weights the previous phase read last, still in L2 (RS 1 % faster)
          runs.push_back({owner, own ? 2 * hp.W : 2 * ((owner & 1) ? hp.W - rot : rot), 0, k, {i, k, k1, 0}});
        k = k1;
      }
    }
    std::stable_sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) {
      return std::tie(a.key0, a.key1, a.key2, a.k0) < std::tie(b.key0, b.key1, b.key2, b.k0);
    });
    for (const Run& r : runs) segs.push_back(r.s);
  } else {
    for (int i = 0; i < n; ++i) segs.push_back({i, 0, plans[i]->hp.n_tiles, 0});
  }
  // merge contiguous runs of one rank, assign global offsets
  std::vector<ao::Seg> out;
  for (const ao::Seg& s : segs) {
    if (!out.empty() && out.back().g == s.g && out.back().k1 == s.k0)
      out.back().k1 = s.k1;
    else
      out.push_back(s);
  }
  if (out.size() > size_t(ao::kMaxSegs)) return false;
  int o = 0;
  for (ao::Seg& s : out) {
    s.o = o;
    o += s.k1 - s.k0;
  }
  ka->n_seg = int32_t(out.size());
  ka->n_total = o;
  for (size_t i = 0; i < out.size(); ++i) ka->seg[i] = out[i];
  return true;
}

// How a group launch is scheduled (shared by launch_group and ao_group_schedule_export):
// sets ka->ctas_per_rank / comm_ctas_per_rank and, when the group runs time-sliced, the
// segment list.  Fails when the persistent CTAs could not all be co-resident (H3).
static ao_status group_schedule(int n, ao_plan* const* plans, int mode, int sm_count, ao::KernelArgs* ka,
                                bool* time_sliced) {
  const ao::HostPlan& h0 = plans[0]->hp;
  const bool comm = mode == ao::MODE_AG && h0.desc.backend != AO_BACKEND_CE && h0.W > 1;
  ka->ctas_per_rank = h0.n_cta * h0.tile.cg;
  ka->comm_ctas_per_rank = comm ? h0.desc.comm_ctas : 0;
  ka->n_seg = 0;
  ka->n_total = 0;
  *time_sliced = false;
  const int64_t grid = int64_t(n) * (ka->ctas_per_rank + ka->comm_ctas_per_rank);
  if (grid > sm_count && n > 1 && n == h0.W && ka->ctas_per_rank <= sm_count && ka->comm_ctas_per_rank == 0 &&
      (mode == ao::MODE_RS || h0.desc.dir == AO_DIR_PUSH))
    *time_sliced = build_segments(n, plans, mode, ka);
  if (grid > sm_count && !*time_sliced)
    return fail(AO_ERR_INVALID_ARG, "grid of %lld CTAs exceeds the %d SMs: the persistent CTAs would not be "
                "co-resident (lower n_cta / comm_ctas; a whole-world loopback group of AG push, GEMM-RS or "
                "GEMM-AR plans with n_cta <= SMs runs time-sliced)", (long long)grid, sm_count);
  if (h0.tile.cg == 2 && (ka->comm_ctas_per_rank % 2) != 0)
    return fail(AO_ERR_INVALID_ARG, "comm_ctas must be even with CTA-pair tiles (cluster launch)");
  return AO_OK;
}

// ------------------------------------------------------------------------------ op calls
static ao_status launch_group(int n, ao_plan* const* plans, const void* const* As, const void* const* Bs,
                              void* const* Cs, void* const* Gouts, void* stream_v, int op) {
  const int mode = op == AO_OP_AG_GEMM ? ao::MODE_AG : ao::MODE_RS;  // GEMM-AR runs the RS kernel
  if (n < 1 || n > AO_MAX_WORLD || !plans) return fail(AO_ERR_INVALID_ARG, "bad group size %d", n);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  ao_plan* p0 = plans[0];
  if (!p0 || !p0->ctx) return fail(AO_ERR_STATE, "plan is not bound to a ctx");
  const ao::HostPlan& h0 = p0->hp;
  if (h0.desc.op != op)
    return fail(AO_ERR_INVALID_ARG, "op mismatch: plan is %s",
                h0.is_ag ? "ag_gemm" : (h0.is_ar ? "gemm_ar" : (h0.is_a2a ? "a2a_gemm" : (h0.is_attn ? "sp_attn" : "gemm_rs"))));
  for (int i = 0; i < n; ++i) {
    ao_plan* p = plans[i];
    if (!p || !p->ctx) return fail(AO_ERR_STATE, "plan %d not bound", i);
    if (!p->ctx->imported) return fail(AO_ERR_STATE, "ctx of rank %d: handles not imported", p->ctx->rank);
    if (p->hp.hash != h0.hash) return fail(AO_ERR_PEER, "plan hash mismatch inside group");
    if (p->ctx->device != p0->ctx->device) return fail(AO_ERR_INVALID_ARG, "group spans devices");
    for (int j = 0; j < i; ++j)
      if (plans[j]->ctx == p->ctx) return fail(AO_ERR_INVALID_ARG, "two plans of one ctx in a group");
    if (!aligned16(As[i]) || !aligned16(Bs[i]) || !aligned16(Cs[i]))
      return fail(AO_ERR_INVALID_ARG, "operands must be 16-byte aligned device pointers");
    ao_status s = take_async_error(p->ctx);
    if (s != AO_OK) return s;
  }
  AO_CUDA(cudaSetDevice(p0->ctx->device));
  {
    ao_status s = announce_plans(n, plans);
    if (s != AO_OK) return s;
  }
  if (h0.M == 0 || h0.N == 0) return AO_OK;

  std::unique_ptr<ao::KernelArgs> ka(new ao::KernelArgs());
  memset(ka.get(), 0, sizeof(ao::KernelArgs));
  ka->n_group = n;
  ka->ctas_per_rank = h0.n_cta * h0.tile.cg;
  ka->mode = mode;
  ka->timeout_ns = h0.desc.timeout_ns ? h0.desc.timeout_ns : 5000000000ull;
  ka->err = p0->ctx->err_dev;
  ka->skip_wait = int32_t(g_debug.skip_wait);
  ka->delay_ns = uint32_t(g_debug.delay_ns);
  ka->exp = int32_t(g_debug.exp);
  ka->trace = p0->ctx->trace;
  ka->trace_cursor = p0->ctx->trace_cursor;
  ka->trace_cap = p0->ctx->trace_cap;
  ka->trace_seq = p0->ctx->trace ? p0->ctx->trace_seq++ : 0;
  ka->l2_hint = g_debug.l2_hint >= 0 ? int32_t(g_debug.l2_hint)
                                     : (((h0.desc.intra == AO_INTRA_GROUPED && h0.desc.group_m > 1) ||
                                         h0.desc.intra == AO_INTRA_COL)
                                            ? 2
                                            : 0);
  const bool ce = mode == ao::MODE_AG && h0.desc.backend == AO_BACKEND_CE && h0.W > 1;
  const int comm = mode == ao::MODE_AG ? p0->comm_kind : ao::COMM_NONE;
  bool time_sliced = false;
  {
    ao_status s = group_schedule(n, plans, mode, p0->ctx->sm_count, ka.get(), &time_sliced);
    if (s != AO_OK) return s;
  }
  // The epoch advances only once the op is actually enqueued (a failed call leaves every
  // ctx of the group at its previous epoch, so the world stays in step).
  std::vector<uint32_t> epochs(n);
  for (int i = 0; i < n; ++i) {
    ao_ctx* c = plans[i]->ctx;
    epochs[i] = c->epoch + 1;
    if (epochs[i] != epochs[0]) return fail(AO_ERR_STATE, "ranks of a group disagree on the epoch");
    ao_status s = fill_rank(&ka->rk[i], plans[i], epochs[i], As[i], Bs[i], Cs[i]);
    if (s != AO_OK) return s;
    if (time_sliced) ka->rk[i].sk_dp = ka->rk[i].n_tiles;  // time-sliced groups walk whole tiles
  }
  DriverFns* drv = nullptr;
  if (g_debug.prearrive) {
    ao_status s = get_driver(&drv);
    if (s != AO_OK) return s;
    for (int i = 0; i < n; ++i) {
      ao_ctx* c = plans[i]->ctx;
      CUresult r = drv->memset32(reinterpret_cast<CUdeviceptr>(c->flags(c->rank, epochs[i] & 1)), epochs[i],
                                 ao::flag_words_needed(plans[i]->hp.desc), stream);
      if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuMemsetD32Async failed (%d)", int(r));
    }
  }
  if (ce && !g_debug.prearrive) {
    ao_status s = get_driver(&drv);
    if (s != AO_OK) return s;
    // CE backend (Fig.7a).  PUSH: every source rank copies its chunks to the peers in
    // plan order with peer memcpys, each followed by a 4-byte copy of the epoch into the
    // destination's flag word.  PULL: every rank first stages its shard in its own gathered
    // buffer, then copies the peers' chunks in plan order into its own buffer and sets its
    // own flag.  Whole-world groups (loopback) record the chains once per (parity, buffers)
    // as a CUDA graph (three host operations per call; in PULL the stage copies of all ranks
    // are a graph join before the pulls).  A PULL whose sources live in other processes
    // waits on their ready flags with cuStreamWaitValue32, issued directly per call.
    ao_ctx* c0 = p0->ctx;
    const uint32_t par = epochs[0] & 1;
    const bool pull = h0.desc.dir == AO_DIR_PULL;
    AO_CUDA(cudaEventRecord(c0->ev_start, stream));
    AO_CUDA(cudaStreamWaitEvent(c0->side, c0->ev_start, 0));
    CUresult r = drv->write32(c0->side, reinterpret_cast<CUdeviceptr>(c0->epoch_cell), epochs[0], 0);
    if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", int(r));
    if (pull && n < h0.W) {
      for (int i = 0; i < n; ++i) {  // all local stages first: a pull never waits behind one
        const ao::HostPlan& hp = plans[i]->hp;
        ao_ctx* c = plans[i]->ctx;
        const int64_t row_bytes = hp.K * 2;
        if (row_bytes > 0)
          AO_CUDA(cudaMemcpyAsync(c->data(hp.rank, par) + int64_t(hp.rank) * hp.S * row_bytes, As[i],
                                  size_t(hp.S * row_bytes), cudaMemcpyDeviceToDevice, c0->side));
        for (int64_t j = 0; j < hp.S / hp.C; ++j) {
          const int64_t g = (int64_t(hp.rank) * hp.S) / hp.C + j;
          r = drv->write32(c0->side, reinterpret_cast<CUdeviceptr>(c->flags(hp.rank, par) + g), epochs[0], 0);
          if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", int(r));
        }
      }
      for (int i = 0; i < n; ++i) {
        const ao::HostPlan& hp = plans[i]->hp;
        ao_ctx* c = plans[i]->ctx;
        const int64_t row_bytes = hp.K * 2;
        for (const ao::P2POp& op : hp.plans[hp.rank]) {
          const int g = int(op.row0 / hp.C);
          r = drv->wait32(c0->side, reinterpret_cast<CUdeviceptr>(c->flags(op.peer, par) + g), epochs[0],
                          0x0 /* CU_STREAM_WAIT_VALUE_GEQ */);
          if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", int(r));
          if (row_bytes > 0)
            AO_CUDA(cudaMemcpyAsync(c->data(hp.rank, par) + op.row0 * row_bytes,
                                    c->data(op.peer, par) + op.row0 * row_bytes, size_t(op.rows * row_bytes),
                                    cudaMemcpyDeviceToDevice, c0->side));
          r = drv->write32(c0->side, reinterpret_cast<CUdeviceptr>(c->flags(hp.rank, par) + g), epochs[0], 0);
          if (r != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", int(r));
        }
      }
    } else {
      std::vector<uintptr_t> key{uintptr_t(par), uintptr_t(n), uintptr_t(time_sliced)};
      for (int i = 0; i < n; ++i) {
        key.push_back(reinterpret_cast<uintptr_t>(plans[i]));
        key.push_back(reinterpret_cast<uintptr_t>(As[i]));
      }
      cudaGraphExec_t exec = nullptr;
      auto it = p0->ce_graphs.find(key);
      if (it != p0->ce_graphs.end()) {
        exec = it->second;
      } else {
        cudaGraph_t graph;
        AO_CUDA(cudaGraphCreate(&graph, 0));
        std::vector<cudaGraphNode_t> stages;  // PULL: every rank's shard staged (graph join)
        if (pull) {
          for (int i = 0; i < n; ++i) {
            const ao::HostPlan& hp = plans[i]->hp;
            const int64_t row_bytes = hp.K * 2;
            if (row_bytes == 0) continue;
            cudaGraphNode_t st = nullptr;
            AO_CUDA(cudaGraphAddMemcpyNode1D(&st, graph, nullptr, 0,
                                             plans[i]->ctx->data(hp.rank, par) + int64_t(hp.rank) * hp.S * row_bytes,
                                             As[i], size_t(hp.S * row_bytes), cudaMemcpyDeviceToDevice));
            stages.push_back(st);
          }
        }
        for (int i = 0; i < n; ++i) {
          ao_plan* p = plans[i];
          ao_ctx* c = p->ctx;
          const ao::HostPlan& hp = p->hp;
          const int64_t row_bytes = hp.K * 2;
          std::vector<cudaGraphNode_t> prev = stages;
          std::vector<ao::P2POp> ops = hp.plans[hp.rank];
          if (time_sliced)  // destination-major: each rank's chunks land before its turn
            std::stable_sort(ops.begin(), ops.end(),
                             [](const ao::P2POp& a, const ao::P2POp& b) { return a.peer < b.peer; });
          for (const ao::P2POp& op : ops) {
            const int g = int(op.row0 / hp.C);
            const char* src = pull ? c->data(op.peer, par) + op.row0 * row_bytes
                                   : static_cast<const char*>(As[i]) + (op.row0 - int64_t(hp.rank) * hp.S) * row_bytes;
            const int dst_rank = pull ? hp.rank : op.peer;
            char* dst = c->data(dst_rank, par) + op.row0 * row_bytes;
            cudaGraphNode_t data = nullptr, flag = nullptr;
            if (row_bytes > 0) {
              AO_CUDA(cudaGraphAddMemcpyNode1D(&data, graph, prev.data(), prev.size(), dst, src,
                                               size_t(op.rows * row_bytes), cudaMemcpyDeviceToDevice));
              prev.assign(1, data);
            }
            AO_CUDA(cudaGraphAddMemcpyNode1D(&flag, graph, prev.data(), prev.size(), c->flags(dst_rank, par) + g,
                                             c0->epoch_cell, 4, cudaMemcpyDeviceToDevice));
            prev.assign(1, flag);
          }
        }
        cudaError_t ge = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ge != cudaSuccess) return fail(AO_ERR_CUDA, "CE graph instantiate: %s", cudaGetErrorString(ge));
        if (p0->ce_graphs.size() >= kMaxCeGraphs) {  // bounded cache (callers that rotate buffers)
          AO_CUDA(cudaStreamSynchronize(c0->side));
          cudaGraphExecDestroy(p0->ce_graphs.begin()->second);
          p0->ce_graphs.erase(p0->ce_graphs.begin());
        }
        p0->ce_graphs[key] = exec;
      }
      AO_CUDA(cudaGraphLaunch(exec, c0->side));
    }
    AO_CUDA(cudaEventRecord(c0->ev_done, c0->side));
  }
  cudaError_t e = ao::launch_fused(*ka, h0.tile.bn, h0.tile.cg, comm, stream);
  if (e != cudaSuccess) return fail(AO_ERR_CUDA, "fused kernel launch: %s", cudaGetErrorString(e));
  for (int i = 0; i < n; ++i) plans[i]->ctx->epoch = epochs[i];
  if (ce && !g_debug.prearrive) AO_CUDA(cudaStreamWaitEvent(stream, p0->ctx->ev_done, 0));
  {
    ao_status s = mark_done(n, plans, epochs, stream);
    if (s != AO_OK) return s;
  }
  // optional gathered-A output (bit-exact copy of concat_p A_p)
  if (mode == ao::MODE_AG && Gouts) {
    for (int i = 0; i < n; ++i) {
      if (!Gouts[i]) continue;
      const ao::HostPlan& hp = plans[i]->hp;
      const size_t rb = size_t(hp.K) * 2, shard = size_t(hp.S) * rb;
      char* out = static_cast<char*>(Gouts[i]);
      const char* gath = plans[i]->ctx->data(hp.rank, epochs[i] & 1);
      if (hp.rank > 0) AO_CUDA(cudaMemcpyAsync(out, gath, hp.rank * shard, cudaMemcpyDeviceToDevice, stream));
      AO_CUDA(cudaMemcpyAsync(out + hp.rank * shard, As[i], shard, cudaMemcpyDeviceToDevice, stream));
      const size_t tail = size_t(hp.W - 1 - hp.rank) * shard;
      if (tail)
        AO_CUDA(cudaMemcpyAsync(out + (hp.rank + 1) * shard, gath + (hp.rank + 1) * shard, tail,
                                cudaMemcpyDeviceToDevice, stream));
    }
  }
  return AO_OK;
}

// A2A-GEMM (NEXT-3): prep kernel (counts, permutation, count exchange, route positions),
// then the fused kernel (dispatch row gathers by warp 7, arrival-ordered expert GEMM).
static ao_status launch_a2a(int n, ao_plan* const* plans, const void* const* Xs, const int32_t* const* idxs,
                            const void* const* Bs, void* const* Ys, int32_t* const* route_pos,
                            int32_t* const* recv_rows, void* stream_v) {
  if (n < 1 || n > AO_MAX_WORLD || !plans) return fail(AO_ERR_INVALID_ARG, "bad group size %d", n);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  ao_plan* p0 = plans[0];
  if (!p0 || !p0->ctx) return fail(AO_ERR_STATE, "plan is not bound to a ctx");
  const ao::HostPlan& h0 = p0->hp;
  if (!h0.is_a2a) return fail(AO_ERR_INVALID_ARG, "op mismatch: plan is not a2a_gemm");
  for (int i = 0; i < n; ++i) {
    ao_plan* p = plans[i];
    if (!p || !p->ctx) return fail(AO_ERR_STATE, "plan %d not bound", i);
    if (!p->ctx->imported) return fail(AO_ERR_STATE, "ctx of rank %d: handles not imported", p->ctx->rank);
    if (p->hp.hash != h0.hash) return fail(AO_ERR_PEER, "plan hash mismatch inside group");
    if (p->ctx->device != p0->ctx->device) return fail(AO_ERR_INVALID_ARG, "group spans devices");
    for (int j = 0; j < i; ++j)
      if (plans[j]->ctx == p->ctx) return fail(AO_ERR_INVALID_ARG, "two plans of one ctx in a group");
    if (!aligned16(Xs[i]) || !aligned16(Bs[i]) || !aligned16(Ys[i]) || !idxs[i] || !route_pos[i] || !recv_rows[i])
      return fail(AO_ERR_INVALID_ARG, "operands must be 16-byte aligned device pointers (index arrays non-null)");
    ao_status s = take_async_error(p->ctx);
    if (s != AO_OK) return s;
  }
  AO_CUDA(cudaSetDevice(p0->ctx->device));
  {
    ao_status s = announce_plans(n, plans);
    if (s != AO_OK) return s;
  }
  std::unique_ptr<ao::KernelArgs> ka(new ao::KernelArgs());
  memset(ka.get(), 0, sizeof(ao::KernelArgs));
  ka->n_group = n;
  ka->ctas_per_rank = h0.n_cta * h0.tile.cg;
  ka->mode = ao::MODE_A2A;
  ka->timeout_ns = h0.desc.timeout_ns ? h0.desc.timeout_ns : 5000000000ull;
  ka->err = p0->ctx->err_dev;
  ka->skip_wait = int32_t(g_debug.skip_wait);
  ka->delay_ns = uint32_t(g_debug.delay_ns);
  ka->exp = int32_t(g_debug.exp);
  ka->trace = p0->ctx->trace;
  ka->trace_cursor = p0->ctx->trace_cursor;
  ka->trace_cap = p0->ctx->trace_cap;
  ka->trace_seq = p0->ctx->trace ? p0->ctx->trace_seq++ : 0;
  ka->l2_hint = g_debug.l2_hint >= 0 ? int32_t(g_debug.l2_hint) : 2;
  const int64_t grid = int64_t(n) * ka->ctas_per_rank;
  if (grid > p0->ctx->sm_count) {
    if (n == h0.W && ka->ctas_per_rank <= p0->ctx->sm_count)
      ka->a2a_ts = 1;  // time-sliced whole-world group: expert after expert over all SMs
    else
      return fail(AO_ERR_INVALID_ARG, "grid of %lld CTAs exceeds the %d SMs (lower n_cta)", (long long)grid,
                  p0->ctx->sm_count);
  }
  std::unique_ptr<ao::A2APrepArgs> pa(new ao::A2APrepArgs());
  memset(pa.get(), 0, sizeof(ao::A2APrepArgs));
  pa->n_group = n;
  pa->W = h0.W;
  pa->T = int32_t(h0.M);
  pa->topk = h0.desc.topk;
  pa->maxJ = h0.n_c;
  pa->timeout_ns = ka->timeout_ns;
  pa->err = p0->ctx->err_dev;
  std::vector<uint32_t> epochs(n);
  for (int i = 0; i < n; ++i) {
    ao_ctx* c = plans[i]->ctx;
    epochs[i] = c->epoch + 1;
    if (epochs[i] != epochs[0]) return fail(AO_ERR_STATE, "ranks of a group disagree on the epoch");
    ao_status s = fill_rank(&ka->rk[i], plans[i], epochs[i], Xs[i], Bs[i], Ys[i]);
    if (s != AO_OK) return s;
    ao::A2APrepRank& r = pa->rk[i];
    r.topk_idx = idxs[i];
    r.perm = plans[i]->d_a2a;
    r.lpos = plans[i]->d_a2a + size_t(h0.W) * size_t(h0.M);
    r.route_pos = route_pos[i];
    r.recv_rows = recv_rows[i];
    r.rank = plans[i]->hp.rank;
    for (int q = 0; q < h0.W; ++q) r.peer_flags[q] = c->flags(q, epochs[i] & 1);
  }
  pa->epoch = epochs[0];
  if (h0.M > 0) {
    cudaError_t e = ao::launch_a2a_prep(*pa, stream);
    if (e != cudaSuccess) return fail(AO_ERR_CUDA, "a2a prep launch: %s", cudaGetErrorString(e));
    e = ao::launch_fused(*ka, h0.tile.bn, h0.tile.cg, ao::COMM_NONE, stream);
    if (e != cudaSuccess) return fail(AO_ERR_CUDA, "fused kernel launch: %s", cudaGetErrorString(e));
  } else {
    for (int i = 0; i < n; ++i) AO_CUDA(cudaMemsetAsync(recv_rows[i], 0, 4, stream));
  }
  for (int i = 0; i < n; ++i) plans[i]->ctx->epoch = epochs[i];
  return mark_done(n, plans, epochs, stream);
}

ao_status ao_a2a_gemm_group(int n, ao_plan* const* plans, const void* const* Xs, const int32_t* const* topk_idxs,
                            const void* const* Bs, void* const* Ys, int32_t* const* route_pos,
                            int32_t* const* recv_rows, void* stream) {
  return launch_a2a(n, plans, Xs, topk_idxs, Bs, Ys, route_pos, recv_rows, stream);
}

ao_status ao_a2a_gemm(ao_plan* plan, const void* X, const int32_t* topk_idx, const void* B, void* Y,
                      int32_t* route_pos, int32_t* recv_rows, void* stream) {
  return launch_a2a(1, &plan, &X, &topk_idx, &B, &Y, &route_pos, &recv_rows, stream);
}

// SP attention (NEXT-4): copy-engine pushes of every source's K/V chunks to every peer's
// gathered buffers (ring rotation; destination-major when time-sliced), each followed by
// the epoch copied into the destination's flag (src, chunk); then the attention kernel.
static ao_status launch_attn_group(int n, ao_plan* const* plans, const void* const* Qs, const void* const* Ks,
                                   const void* const* Vs, void* const* Os, void* stream_v) {
  if (n < 1 || n > AO_MAX_WORLD || !plans) return fail(AO_ERR_INVALID_ARG, "bad group size %d", n);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  ao_plan* p0 = plans[0];
  if (!p0 || !p0->ctx) return fail(AO_ERR_STATE, "plan is not bound to a ctx");
  const ao::HostPlan& h0 = p0->hp;
  if (!h0.is_attn) return fail(AO_ERR_INVALID_ARG, "op mismatch: plan is not sp_attn / hp_attn");
  for (int i = 0; i < n; ++i) {
    ao_plan* p = plans[i];
    if (!p || !p->ctx) return fail(AO_ERR_STATE, "plan %d not bound", i);
    if (!p->ctx->imported) return fail(AO_ERR_STATE, "ctx of rank %d: handles not imported", p->ctx->rank);
    if (p->hp.hash != h0.hash) return fail(AO_ERR_PEER, "plan hash mismatch inside group");
    if (p->ctx->device != p0->ctx->device) return fail(AO_ERR_INVALID_ARG, "group spans devices");
    for (int j = 0; j < i; ++j)
      if (plans[j]->ctx == p->ctx) return fail(AO_ERR_INVALID_ARG, "two plans of one ctx in a group");
    if (!aligned16(Qs[i]) || !aligned16(Ks[i]) || !aligned16(Vs[i]) || !aligned16(Os[i]))
      return fail(AO_ERR_INVALID_ARG, "operands must be 16-byte aligned device pointers");
    ao_status s = take_async_error(p->ctx);
    if (s != AO_OK) return s;
  }
  AO_CUDA(cudaSetDevice(p0->ctx->device));
  {
    ao_status s = announce_plans(n, plans);
    if (s != AO_OK) return s;
  }
  const int W = h0.W, H = int(h0.N), S = int(h0.M), crows = h0.C, nch = h0.n_c;
  const bool hp = h0.is_hp;
  const int Hv = hp ? H / W : H;  // heads of one source's block in the gathered buffers
  const int64_t rows = int64_t(H) * S, row_bytes = 256;  // [H*S_loc, 128] bf16
  const int64_t vrows = int64_t(Hv) * S;                  // rows of one source's block
  std::unique_ptr<ao::AttnArgs> ka(new ao::AttnArgs());
  memset(ka.get(), 0, sizeof(ao::AttnArgs));
  ka->n_group = n;
  ka->W = W;
  ka->H = Hv;
  ka->hp = hp ? 1 : 0;
  ka->S_loc = S;
  ka->crows = crows;
  ka->nch = nch;
  ka->ctas_per_rank = h0.n_cta;
  ka->scale_log2 = float(1.4426950408889634 / std::sqrt(128.0));
  ka->trace = p0->ctx->trace;  // device trace (ao_ctx_trace_enable on the first plan's ctx)
  ka->trace_cursor = p0->ctx->trace_cursor;
  ka->trace_cap = p0->ctx->trace_cap;
  ka->trace_seq = p0->ctx->trace ? p0->ctx->trace_seq++ : 0;
  ka->causal = h0.desc.causal;
  ka->timeout_ns = h0.desc.timeout_ns ? h0.desc.timeout_ns : 5000000000ull;
  ka->err = p0->ctx->err_dev;
  if (int64_t(n) * h0.n_cta > p0->ctx->sm_count) {
    if (n == W && h0.n_cta <= p0->ctx->sm_count)
      ka->ts = 1;  // time-sliced whole-world group: rank after rank over all SMs (Q24)
    else
      return fail(AO_ERR_INVALID_ARG, "grid of %lld CTAs exceeds the %d SMs (lower n_cta)",
                  (long long)(int64_t(n) * h0.n_cta), p0->ctx->sm_count);
  }
  std::vector<uint32_t> epochs(n);
  for (int i = 0; i < n; ++i) {
    ao_ctx* c = plans[i]->ctx;
    epochs[i] = c->epoch + 1;
    if (epochs[i] != epochs[0]) return fail(AO_ERR_STATE, "ranks of a group disagree on the epoch");
    const uint32_t par = epochs[i] & 1;
    const int r = plans[i]->hp.rank;
    ao::AttnRank& R = ka->rk[i];
    // data half: SP [gathered K | gathered V], each [W][H*S_loc]; HP [gathered Q | K | V |
    // O return], each [W][H/W*S_loc] (= H*S_loc rows)
    char* gQ = c->data(r, par);
    char* gK = hp ? gQ + rows * row_bytes : gQ;
    char* gV = gK + int64_t(W) * vrows * row_bytes;
    ao_status s;
    if ((s = encode_2d(&R.tmQ, Qs[i], rows, 128, 128)) != AO_OK) return s;
    if ((s = encode_2d(&R.tmK_loc, Ks[i], rows, 128, 128)) != AO_OK) return s;
    if ((s = encode_2d(&R.tmV_loc, Vs[i], rows, 128, 128)) != AO_OK) return s;
    if ((s = encode_2d(&R.tmK, gK, int64_t(W) * vrows, 128, 128)) != AO_OK) return s;
    if ((s = encode_2d(&R.tmV, gV, int64_t(W) * vrows, 128, 128)) != AO_OK) return s;
    if (hp && (s = encode_2d(&R.tmQg, gQ, int64_t(W) * vrows, 128, 128)) != AO_OK) return s;
    R.O = static_cast<char*>(Os[i]);
    R.flags = c->flags(r, par);
    R.rank = r;
    R.epoch = epochs[i];
    if (hp) {
      for (int q = 0; q < W; ++q) {
        R.oret[q] = c->data(q, par) + 3 * rows * row_bytes;
        R.peer_flags[q] = c->flags(q, par);
      }
      R.counters = c->counters;
    }
  }
  ao_ctx* c0 = p0->ctx;
  const uint32_t par = epochs[0] & 1;
  const bool ce = W > 1 && rows > 0;
  if (ce) {
    AO_CUDA(cudaEventRecord(c0->ev_start, stream));
    AO_CUDA(cudaStreamWaitEvent(c0->side, c0->ev_start, 0));
    DriverFns* drv = nullptr;
    ao_status s = get_driver(&drv);
    if (s != AO_OK) return s;
    CUresult cr = drv->write32(c0->side, reinterpret_cast<CUdeviceptr>(c0->epoch_cell), epochs[0], 0);
    if (cr != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", int(cr));
    // WAR on the destination's gathered K/V (parity e % 2, last read by its epoch e-2
    // kernel).  Non-causal: every rank waits on every source, so a source at epoch e has
    // seen the destination's e-1 pushes and the Q11 argument applies.  Causal: a rank waits
    // only on lower ranks, so nothing else orders a source behind a higher destination --
    // wait for that destination's done word (written after each of its attention kernels)
    // to reach e-2.  Ranks of this launch are ordered by the stream already.
    if (!hp && h0.desc.causal && epochs[0] > 2) {
      for (int dst = 0; dst < W; ++dst) {
        bool in_group = false;
        for (int q = 0; q < n; ++q) in_group |= plans[q]->hp.rank == dst;
        bool needed = false;  // some source of this launch pushes to dst (dst > src)
        for (int q = 0; q < n; ++q) needed |= dst > plans[q]->hp.rank;
        if (in_group || !needed) continue;
        cr = drv->wait32(c0->side, reinterpret_cast<CUdeviceptr>(c0->done_word(dst)), epochs[0] - 2,
                         0x0 /* CU_STREAM_WAIT_VALUE_GEQ */);
        if (cr != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", int(cr));
      }
    }
    std::vector<uintptr_t> key{uintptr_t(0xA77Eu), uintptr_t(par), uintptr_t(n), uintptr_t(ka->ts)};
    for (int i = 0; i < n; ++i) {
      key.push_back(reinterpret_cast<uintptr_t>(plans[i]));
      key.push_back(reinterpret_cast<uintptr_t>(Ks[i]));
      key.push_back(reinterpret_cast<uintptr_t>(Vs[i]));
      if (hp) key.push_back(reinterpret_cast<uintptr_t>(Qs[i]));
    }
    cudaGraphExec_t exec = nullptr;
    auto it = p0->ce_graphs.find(key);
    if (it != p0->ce_graphs.end()) {
      exec = it->second;
    } else {
      cudaGraph_t graph;
      AO_CUDA(cudaGraphCreate(&graph, 0));
      for (int i = 0; i < n; ++i) {  // one chain per source rank in this group
        const int src = plans[i]->hp.rank;
        std::vector<int> dests;
        for (int ds = 1; ds < W; ++ds) {  // ring rotation; SP causal: only higher ranks read src's shard
          const int dst = (src + ds) % W;
          if (hp || !h0.desc.causal || dst > src) dests.push_back(dst);
        }
        if (ka->ts) std::sort(dests.begin(), dests.end());              // destination-major
        std::vector<cudaGraphNode_t> prev;
        for (int dst : dests) {
          ao_ctx* dc = nullptr;  // the destination's buffers, mapped in this process
          for (int q = 0; q < n; ++q)
            if (plans[q]->hp.rank == dst) dc = plans[q]->ctx;
          (void)dc;
          char* gQ = plans[i]->ctx->data(dst, par);  // the destination's buffers, mapped in this process
          char* gK = hp ? gQ + rows * row_bytes : gQ;
          char* gV = gK + int64_t(W) * vrows * row_bytes;
          uint32_t* fl = plans[i]->ctx->flags(dst, par);
          // SP: chunk c of src's whole K/V; HP: chunk c of the rows of dst's head group in
          // src's Q, K and V (the all-to-all)
          const int64_t sbase = hp ? int64_t(dst) * vrows : 0;
          for (int cch = 0; cch < nch; ++cch) {
            const int64_t off = (int64_t(src) * vrows + int64_t(cch) * crows) * row_bytes;
            const int64_t soff = (sbase + int64_t(cch) * crows) * row_bytes;
            const size_t bytes = size_t(crows) * row_bytes;
            cudaGraphNode_t nq = nullptr, nk = nullptr, nv = nullptr, nf = nullptr;
            if (hp) {
              AO_CUDA(cudaGraphAddMemcpyNode1D(&nq, graph, prev.data(), prev.size(), gQ + off,
                                               static_cast<const char*>(Qs[i]) + soff, bytes, cudaMemcpyDeviceToDevice));
              prev.assign(1, nq);
            }
            AO_CUDA(cudaGraphAddMemcpyNode1D(&nk, graph, prev.data(), prev.size(), gK + off,
                                             static_cast<const char*>(Ks[i]) + soff, bytes, cudaMemcpyDeviceToDevice));
            AO_CUDA(cudaGraphAddMemcpyNode1D(&nv, graph, &nk, 1, gV + off, static_cast<const char*>(Vs[i]) + soff,
                                             bytes, cudaMemcpyDeviceToDevice));
            AO_CUDA(cudaGraphAddMemcpyNode1D(&nf, graph, &nv, 1, fl + src * nch + cch, c0->epoch_cell, 4,
                                             cudaMemcpyDeviceToDevice));
            prev.assign(1, nf);
          }
        }
      }
      cudaError_t ge = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ge != cudaSuccess) return fail(AO_ERR_CUDA, "CE graph instantiate: %s", cudaGetErrorString(ge));
      if (p0->ce_graphs.size() >= kMaxCeGraphs) {
        AO_CUDA(cudaStreamSynchronize(c0->side));
        cudaGraphExecDestroy(p0->ce_graphs.begin()->second);
        p0->ce_graphs.erase(p0->ce_graphs.begin());
      }
      p0->ce_graphs[key] = exec;
    }
    AO_CUDA(cudaGraphLaunch(exec, c0->side));
    AO_CUDA(cudaEventRecord(c0->ev_done, c0->side));
  }
  if (ce && (g_debug.exp & 65536)) AO_CUDA(cudaStreamWaitEvent(stream, c0->ev_done, 0));  // debug: gather first
  if (rows > 0) {
    cudaError_t e = ao::launch_attn(*ka, stream);
    if (e != cudaSuccess) return fail(AO_ERR_CUDA, "attention kernel launch: %s", cudaGetErrorString(e));
  }
  if (hp && W > 1 && rows > 0) {
    // the reverse all-to-all: each other source's block of this rank's output came back in
    // the return buffer; wait for its flag (released by the block's last tile) and copy it
    // into O (rows of that source's head group)
    DriverFns* drv = nullptr;
    ao_status s = get_driver(&drv);
    if (s != AO_OK) return s;
    for (int i = 0; i < n; ++i) {
      ao_ctx* c = plans[i]->ctx;
      const int r = plans[i]->hp.rank;
      const uint32_t par = epochs[i] & 1;
      for (int d = 1; d < W; ++d) {
        const int src = (r - d + W) % W;
        CUresult cr = drv->wait32(stream, reinterpret_cast<CUdeviceptr>(c->flags(r, par) + W * nch + src), epochs[i],
                                  0x0 /* CU_STREAM_WAIT_VALUE_GEQ */);
        if (cr != CUDA_SUCCESS) return fail(AO_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", int(cr));
        AO_CUDA(cudaMemcpyAsync(static_cast<char*>(Os[i]) + int64_t(src) * vrows * row_bytes,
                                c->data(r, par) + 3 * rows * row_bytes + int64_t(src) * vrows * row_bytes,
                                size_t(vrows) * row_bytes, cudaMemcpyDeviceToDevice, stream));
      }
    }
  }
  for (int i = 0; i < n; ++i) plans[i]->ctx->epoch = epochs[i];
  if (ce) AO_CUDA(cudaStreamWaitEvent(stream, c0->ev_done, 0));
  return mark_done(n, plans, epochs, stream);
}

ao_status ao_sp_attn_group(int n, ao_plan* const* plans, const void* const* Qs, const void* const* Ks,
                           const void* const* Vs, void* const* Os, void* stream) {
  return launch_attn_group(n, plans, Qs, Ks, Vs, Os, stream);
}

ao_status ao_sp_attn(ao_plan* plan, const void* Q, const void* K, const void* V, void* O, void* stream) {
  return launch_attn_group(1, &plan, &Q, &K, &V, &O, stream);
}

ao_status ao_hp_attn_group(int n, ao_plan* const* plans, const void* const* Qs, const void* const* Ks,
                           const void* const* Vs, void* const* Os, void* stream) {
  return launch_attn_group(n, plans, Qs, Ks, Vs, Os, stream);
}

ao_status ao_hp_attn(ao_plan* plan, const void* Q, const void* K, const void* V, void* O, void* stream) {
  return launch_attn_group(1, &plan, &Q, &K, &V, &O, stream);
}

ao_status ao_ag_gemm_group(int n, ao_plan* const* plans, const void* const* A_shards, const void* const* Bs,
                           void* const* Cs, void* const* Gouts, void* stream) {
  return launch_group(n, plans, A_shards, Bs, Cs, Gouts, stream, AO_OP_AG_GEMM);
}

ao_status ao_gemm_rs_group(int n, ao_plan* const* plans, const void* const* As, const void* const* Bs,
                           void* const* C_shards, void* stream) {
  return launch_group(n, plans, As, Bs, C_shards, nullptr, stream, AO_OP_GEMM_RS);
}

ao_status ao_gemm_ar_group(int n, ao_plan* const* plans, const void* const* As, const void* const* Bs,
                           void* const* Cs, void* stream) {
  return launch_group(n, plans, As, Bs, Cs, nullptr, stream, AO_OP_GEMM_AR);
}

ao_status ao_ag_gemm(ao_plan* plan, const void* A_shard, const void* B, void* C, void* A_gathered_out, void* stream) {
  void* g[1] = {A_gathered_out};
  return launch_group(1, &plan, &A_shard, &B, &C, g, stream, AO_OP_AG_GEMM);
}

ao_status ao_gemm_rs(ao_plan* plan, const void* A, const void* B, void* C_shard, void* stream) {
  return launch_group(1, &plan, &A, &B, &C_shard, nullptr, stream, AO_OP_GEMM_RS);
}

ao_status ao_gemm_ar(ao_plan* plan, const void* A, const void* B, void* C, void* stream) {
  return launch_group(1, &plan, &A, &B, &C, nullptr, stream, AO_OP_GEMM_AR);
}

// ------------------------------------------------------------- group schedule export
// The launch-level schedule of a group call (Q24), canonical JSON:
//   {"mode":"space_sliced"} -- every rank runs its own plan's tables on its own CTAs; or
//   {"mode":"time_sliced","n_total":T,"n_workers":w,"segments":[[rank,k0,k1,o],...],
//    "waits":[[worker,[[i,rank,g],...]],...]}
// segments: positions [k0,k1) of `rank`'s tile order occupy global list indices
// [o, o+k1-k0); worker w runs indices w, w+n_workers, ... (Lst.1 stride).
// waits: per worker, in walk order, the (global index, rank, chunk) before whose tile the
// worker acquires that chunk's flags -- the chunks the tile's rows intersect that
// it needs from peers (AG: chunks of other sources; RS/AR: the own rows' chunks, from
// every other source), once per (worker, rank, chunk).
ao_status ao_group_schedule_export(int n, ao_plan* const* plans, int32_t op, int sm_count, char* buf, size_t cap,
                                   size_t* needed) {
  if (n < 1 || n > AO_MAX_WORLD || !plans) return fail(AO_ERR_INVALID_ARG, "bad group size %d", n);
  for (int i = 0; i < n; ++i) {
    if (!plans[i]) return fail(AO_ERR_INVALID_ARG, "null plan %d", i);
    if (plans[i]->hp.hash != plans[0]->hp.hash) return fail(AO_ERR_PEER, "plan hash mismatch inside group");
  }
  const ao::HostPlan& h0 = plans[0]->hp;
  if (h0.desc.op != op || !(op == AO_OP_AG_GEMM || op == AO_OP_GEMM_RS || op == AO_OP_GEMM_AR))
    return fail(AO_ERR_INVALID_ARG, "op mismatch or op without a group schedule");
  const int mode = op == AO_OP_AG_GEMM ? ao::MODE_AG : ao::MODE_RS;
  std::unique_ptr<ao::KernelArgs> ka(new ao::KernelArgs());
  memset(ka.get(), 0, sizeof(ao::KernelArgs));
  ka->n_group = n;
  bool ts = false;
  ao_status s = group_schedule(n, plans, mode, sm_count > 0 ? sm_count : 148, ka.get(), &ts);
  if (s != AO_OK) return s;
  std::string out;
  if (!ts) {
    out = "{\"mode\":\"space_sliced\"}";
  } else {
    const int n_wk = ka->ctas_per_rank / h0.tile.cg;
    const int64_t BM = h0.tile.bm;
    out = "{\"mode\":\"time_sliced\",\"n_total\":" + std::to_string(ka->n_total) +
          ",\"n_workers\":" + std::to_string(n_wk) + ",\"segments\":[";
    for (int i = 0; i < ka->n_seg; ++i) {
      const ao::Seg& g = ka->seg[i];
      out += (i ? ",[" : "[") + std::to_string(plans[g.g]->hp.rank) + "," + std::to_string(g.k0) + "," +
             std::to_string(g.k1) + "," + std::to_string(g.o) + "]";
    }
    out += "],\"waits\":[";
    for (int w = 0; w < n_wk; ++w) {
      std::vector<std::vector<char>> got(n);
      for (int i = 0; i < n; ++i) got[i].assign(plans[i]->hp.n_chunks, 0);
      std::string lst;
      int si = 0;
      for (int i = w; i < ka->n_total; i += n_wk) {
        while (i >= ka->seg[si].o + (ka->seg[si].k1 - ka->seg[si].k0)) ++si;
        const int grp = ka->seg[si].g;
        const ao::HostPlan& hp = plans[grp]->hp;
        const int t = hp.order[ka->seg[si].k0 + (i - ka->seg[si].o)];
        const int64_t r0 = int64_t(t / hp.n_nb) * BM, r1 = std::min<int64_t>(hp.M, r0 + BM);
        const bool own_tile = r0 / hp.S == hp.rank;
        if (mode == ao::MODE_RS && !own_tile) continue;
        for (int g = int(r0 / hp.C); g <= int((r1 - 1) / hp.C); ++g) {
          if (mode == ao::MODE_AG && (int64_t(g) * hp.C) / hp.S == hp.rank) continue;
          if (got[grp][g]) continue;
          got[grp][g] = 1;
          lst += (lst.empty() ? "[" : ",[") + std::to_string(i) + "," + std::to_string(hp.rank) + "," +
                 std::to_string(g) + "]";
        }
      }
      out += (w ? ",[" : "[") + std::to_string(w) + ",[" + lst + "]]";
    }
    out += "]}";
  }
  if (needed) *needed = out.size() + 1;
  if (buf && cap) {
    const size_t k = std::min(cap - 1, out.size());
    memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return AO_OK;
}

// ---------------------------------------------------------------- E4 backend microbench
ao_status ao_transfer_bench(ao_ctx* c, int peer, int32_t backend, const void* src, int64_t bytes, int64_t chunk_bytes,
                            int32_t n_ctas, int32_t n_streams, int32_t iters, float* ms_per_iter) {
  if (!c || !src || !ms_per_iter || bytes <= 0 || chunk_bytes <= 0 || iters < 1)
    return fail(AO_ERR_INVALID_ARG, "bad argument");
  if (peer < 0 || peer >= c->W || !c->peer_base[peer]) return fail(AO_ERR_STATE, "peer %d not mapped", peer);
  if (size_t(bytes) > c->data_half) return fail(AO_ERR_INVALID_ARG, "message larger than the data half");
  if (!aligned16(src) || bytes % 16 || chunk_bytes % 16) return fail(AO_ERR_INVALID_ARG, "16-byte alignment");
  if (backend == AO_BACKEND_CE ? (n_streams < 1 || n_streams > 16) : (n_ctas < 1 || n_ctas > c->sm_count))
    return fail(AO_ERR_INVALID_ARG, "n_streams in [1,16] (CE) / n_ctas in [1,SMs] (TMA, LDST)");
  AO_CUDA(cudaSetDevice(c->device));
  char* dst = c->data(peer, 0);
  cudaStream_t main_s;
  AO_CUDA(cudaStreamCreateWithFlags(&main_s, cudaStreamNonBlocking));
  std::vector<cudaStream_t> ss(backend == AO_BACKEND_CE ? n_streams : 0);
  for (auto& x : ss) AO_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, fork;
  AO_CUDA(cudaEventCreate(&t0));
  AO_CUDA(cudaEventCreate(&t1));
  AO_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  std::vector<cudaEvent_t> join(ss.size());
  for (auto& e : join) AO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto one = [&]() -> ao_status {
    if (backend == AO_BACKEND_CE) {  // one peer memcpy per chunk, round-robin over the streams
      AO_CUDA(cudaEventRecord(fork, main_s));
      for (auto& x : ss) AO_CUDA(cudaStreamWaitEvent(x, fork, 0));
      int64_t i = 0;
      for (int64_t off = 0; off < bytes; off += chunk_bytes, ++i) {
        const size_t len = size_t(std::min<int64_t>(chunk_bytes, bytes - off));
        AO_CUDA(cudaMemcpyAsync(dst + off, static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToDevice,
                                ss[size_t(i % int64_t(ss.size()))]));
      }
      for (size_t k = 0; k < ss.size(); ++k) {
        AO_CUDA(cudaEventRecord(join[k], ss[k]));
        AO_CUDA(cudaStreamWaitEvent(main_s, join[k], 0));
      }
    } else {
      AO_CUDA(ao::launch_transfer(backend == AO_BACKEND_TMA ? ao::COMM_TMA : ao::COMM_LDST, dst,
                                  static_cast<const char*>(src), bytes, chunk_bytes, n_ctas, main_s));
    }
    return AO_OK;
  };
  ao_status st = one();  // warm-up
  if (st == AO_OK) AO_CUDA(cudaEventRecord(t0, main_s));
  for (int it = 0; it < iters && st == AO_OK; ++it) st = one();
  if (st == AO_OK) {
    AO_CUDA(cudaEventRecord(t1, main_s));
    AO_CUDA(cudaEventSynchronize(t1));
    float ms = 0.f;
    AO_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    *ms_per_iter = ms / float(iters);
  }
  cudaStreamSynchronize(main_s);
  for (auto& x : ss) cudaStreamDestroy(x);
  for (auto& e : join) cudaEventDestroy(e);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaEventDestroy(fork);
  cudaStreamDestroy(main_s);
  return st;
}

// ------------------------------------------------------------------------ device queries
ao_status ao_device_query(int device, const char* key, int64_t* out) {
  if (!key || !out) return fail(AO_ERR_INVALID_ARG, "null argument");
  int sm = 0;
  AO_CUDA(cudaSetDevice(device));
  ao_status s = check_device_sm100(device, &sm);
  if (s != AO_OK) return s;
  if (!strcmp(key, "sm_count")) {
    *out = sm;
  } else if (!strcmp(key, "cluster2_ctas") || !strcmp(key, "cluster4_ctas")) {
    const int n = ao::max_co_resident_ctas(key[7] == '4' ? 4 : 2);
    if (n < 0) return fail(AO_ERR_CUDA, "cudaOccupancyMaxActiveClusters failed");
    *out = n;
  } else {
    return fail(AO_ERR_INVALID_ARG, "unknown device query %s", key);
  }
  return AO_OK;
}

// ----------------------------------------------------------------------- plain GEMM entry
ao_status ao_gemm(int device, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, int32_t tile_m,
                  int32_t tile_n, void* stream_v) {
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int64_t, int64_t, int, int, int>, ao_plan*> cache;
  const int bm = tile_m ? tile_m : (M % 256 == 0 ? 256 : 128);
  if (M < 0 || N < 0 || K < 0 || (bm != 128 && bm != 256 && bm != 512) || M % bm != 0 || N % 8 != 0 || K % 8 != 0)
    return fail(AO_ERR_INVALID_ARG, "ao_gemm needs M %% tile_m == 0, N %% 8 == 0, K %% 8 == 0 (M=%lld N=%lld K=%lld)",
                (long long)M, (long long)N, (long long)K);
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return fail(AO_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  if (M == 0 || N == 0) return AO_OK;
  const int bn = tile_n ? tile_n : 256;
  AO_CUDA(cudaSetDevice(device));
  ao_plan* p = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(device, M, N, K, bm, bn, int(g_debug.gemm_group_m) * 4 + int(g_debug.gemm_stream_k) + 1);
    auto it = cache.find(key);
    if (it != cache.end()) {
      p = it->second;
    } else {
      int sm = 0;
      ao_status s = check_device_sm100(device, &sm);
      if (s != AO_OK) return s;
      ao_plan_desc d;
      ao_plan_desc_init(&d);
      d.M = M;
      d.N = N;
      d.K = K;
      d.chunk_rows = int32_t(std::min<int64_t>(M, 1 << 30));
      d.tile_m = bm;
      d.tile_n = bn;
      d.intra = AO_INTRA_GROUPED;  // GROUP_M swizzle: B tiles reused across row blocks in L2
      d.group_m = int32_t(g_debug.gemm_group_m);
      d.stream_k = bm == 512 ? 0 : int32_t(g_debug.gemm_stream_k);
      if (bm == 512) {  // 4-CTA clusters: as many as fit the GPU at once
        const int n4 = ao::max_co_resident_ctas(4);
        if (n4 < 4) return fail(AO_ERR_CUDA, "no 4-CTA cluster fits this device");
        d.n_cta = n4;
      }
      s = ao_plan_create_host(&d, sm, &p);
      if (s != AO_OK) return s;
      p->device = device;
      s = upload_tables(p);
      if (s != AO_OK) {
        ao_plan_destroy(p);
        return s;
      }
      cache[key] = p;
    }
  }
  std::unique_ptr<ao::KernelArgs> ka(new ao::KernelArgs());
  memset(ka.get(), 0, sizeof(ao::KernelArgs));
  ka->n_group = 1;
  ka->ctas_per_rank = p->hp.n_cta * p->hp.tile.cg;
  ka->mode = ao::MODE_GEMM;
  ka->timeout_ns = 5000000000ull;
  ka->skip_wait = -1;
  ka->l2_hint = g_debug.l2_hint >= 0 ? int32_t(g_debug.l2_hint) : 2;
  ao_status s = fill_rank(&ka->rk[0], p, 0, A, B, C);
  if (s != AO_OK) return s;
  cudaError_t e = ao::launch_fused(*ka, bn, p->hp.tile.cg, ao::COMM_NONE, static_cast<cudaStream_t>(stream_v));
  if (e != cudaSuccess) return fail(AO_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(e));
  return AO_OK;
}

ao_status ao_gemm_batched(int device, int n, const void* const* As, const void* const* Bs, void* const* Cs,
                          int64_t M, int64_t N, int64_t K, int32_t tile_m, int32_t tile_n, int32_t group_m,
                          int32_t n_cta, void* stream_v) {
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int64_t, int64_t, int, int, int, int>, ao_plan*> cache;
  if (n < 1 || n > AO_MAX_WORLD || !As || !Bs || !Cs) return fail(AO_ERR_INVALID_ARG, "bad batch size %d", n);
  const int bm = tile_m ? tile_m : (M % 256 == 0 ? 256 : 128);
  const int bn = tile_n ? tile_n : 256;
  if (M < 0 || N < 0 || K < 0 || (bm != 128 && bm != 256 && bm != 512) || M % bm != 0 ||
      N % 8 != 0 || K % 8 != 0)
    return fail(AO_ERR_INVALID_ARG, "ao_gemm_batched needs M %% tile_m == 0, N %% 8 == 0, K %% 8 == 0");
  for (int i = 0; i < n; ++i)
    if (!aligned16(As[i]) || !aligned16(Bs[i]) || !aligned16(Cs[i]))
      return fail(AO_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  if (M == 0 || N == 0) return AO_OK;
  AO_CUDA(cudaSetDevice(device));
  int sm = 0;
  ao_status s = check_device_sm100(device, &sm);
  if (s != AO_OK) return s;
  const int cg = bm / 128;
  int cap = sm;
  if (cg == 4) cap = ao::max_co_resident_ctas(4);
  const int ctas = std::min(n_cta > 0 ? n_cta : cap / n, cap) / cg * cg;  // CTAs per problem (whole clusters)
  if (ctas < cg || ctas > sm)  // n * ctas > sm: time-sliced (problem after problem)
    return fail(AO_ERR_INVALID_ARG, "%d problems x %d CTAs exceed the %d SMs (or fewer CTAs than a tile needs)", n,
                n_cta, sm);
  ao_plan* p = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(device, M, N, K, bm, bn, group_m, ctas);
    auto it = cache.find(key);
    if (it != cache.end()) {
      p = it->second;
    } else {
      ao_plan_desc d;
      ao_plan_desc_init(&d);
      d.M = M;
      d.N = N;
      d.K = K;
      d.chunk_rows = int32_t(std::min<int64_t>(M, 1 << 30));
      d.tile_m = bm;
      d.tile_n = bn;
      d.intra = AO_INTRA_GROUPED;
      d.group_m = group_m > 0 ? group_m : 16;
      d.n_cta = ctas;
      s = ao_plan_create_host(&d, sm, &p);
      if (s != AO_OK) return s;
      p->device = device;
      s = upload_tables(p);
      if (s != AO_OK) {
        ao_plan_destroy(p);
        return s;
      }
      cache[key] = p;
    }
  }
  std::unique_ptr<ao::KernelArgs> ka(new ao::KernelArgs());
  memset(ka.get(), 0, sizeof(ao::KernelArgs));
  ka->n_group = n;
  ka->ctas_per_rank = p->hp.n_cta * p->hp.tile.cg;
  ka->mode = ao::MODE_GEMM;
  ka->timeout_ns = 5000000000ull;
  ka->skip_wait = -1;
  ka->l2_hint = g_debug.l2_hint >= 0 ? int32_t(g_debug.l2_hint) : 2;
  for (int i = 0; i < n; ++i) {
    s = fill_rank(&ka->rk[i], p, 0, As[i], Bs[i], Cs[i]);
    if (s != AO_OK) return s;
  }
  if (int64_t(n) * ctas > sm) {
    std::vector<ao_plan*> ps(n, p);
    build_segments(n, ps.data(), ao::MODE_GEMM, ka.get());
  }
  cudaError_t e = ao::launch_fused(*ka, bn, p->hp.tile.cg, ao::COMM_NONE, static_cast<cudaStream_t>(stream_v));
  if (e != cudaSuccess) return fail(AO_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(e));
  return AO_OK;
}

}  // extern "C"
