/*
 * autooverlap.h -- C ABI of the B200-native AutoOverlap hot path (arXiv 2601.20595).
 *
 * The library runs ONE persistent fused kernel per op that overlaps a tensor-parallel
 * collective with the GEMM that consumes or produces it, at communication-chunk
 * granularity (§5):
 *
 *   ao_ag_gemm : AllGather -> GEMM.   C_r[M, N] = concat_p(A_p)[M, K] . B_r[N, K]^T
 *                Each chunk of every rank's row shard A_p is pushed to the peers (Lst.2,
 *                P:249-265); tiles spin on per-chunk ready flags and the tile order
 *                follows chunk arrival.
 *   ao_gemm_rs : GEMM -> ReduceScatter.  C_shard_r[S, N] = (sum_s A_s . B_s^T)[rS:(r+1)S, :]
 *                Finished fp32 partial tiles are pushed into the owner's slots per chunk;
 *                the owner's epilogue fuses the peer reduction.
 *
 * The calls follow the paper's statement of the user API: register symmetric
 * buffers (ao_ctx_*), build a chunk schedule (ao_plan_*: chunk size, chunk->tile mapping,
 * transfer backend), run the op with the local kernel's signature plus
 * rank / world size.
 *
 * Conventions
 *  - Every call returns ao_status; no C++ exception crosses the ABI.  On failure
 *    ao_last_error() returns a thread-local human-readable detail.
 *  - All matrices are bf16, row-major, contiguous, 16-byte aligned DEVICE pointers on the
 *    ctx's device, owned by the caller.  Layouts follow Lst.1: A [rows, K],
 *    B [N, K] (nn.Linear weight), C [rows, N].
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All op
 *    calls are asynchronous; device-side spin timeouts surface through
 *    ao_ctx_check_async() (or the next op call).
 *  - Collective semantics: every rank of a world must issue the same sequence of ops,
 *    with plans built from descs that differ only in `rank` (equal ao_plan_hash).
 *  - There is no CPU fallback: on a device that is not sm_100 the ctx/plan calls return
 *    AO_ERR_UNSUPPORTED.
 */
#ifndef AUTOOVERLAP_H
#define AUTOOVERLAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AO_VERSION_MAJOR 0
#define AO_VERSION_MINOR 1
#define AO_MAX_WORLD 8
#define AO_HANDLE_BYTES 256

typedef enum {
  AO_OK = 0,
  AO_ERR_INVALID_ARG = 1, /* desc/pointer validation failed; ao_last_error lists violations */
  AO_ERR_UNSUPPORTED = 2, /* not an sm_100 device, or a feature not built (e.g. PULL execution) */
  AO_ERR_CUDA = 3,        /* a CUDA runtime/driver call failed */
  AO_ERR_OOM = 4,
  AO_ERR_PEER = 5,        /* handle / plan mismatch across ranks */
  AO_ERR_TIMEOUT = 6,     /* a device spin-wait on a chunk flag expired */
  AO_ERR_STATE = 7        /* call order violated (e.g. op before ao_ctx_import_handles) */
} ao_status;

typedef enum { AO_OP_AG_GEMM = 0, AO_OP_GEMM_RS = 1, AO_OP_GEMM_AR = 2 /* NEXT-1 */,
               AO_OP_A2A_GEMM = 3 /* NEXT-3: MoE All-to-All dispatch + expert GEMM */,
               AO_OP_SP_ATTN = 4 /* NEXT-4: sequence-parallel attention over all-gathered KV */,
               AO_OP_HP_ATTN = 5 /* NEXT-4: head-parallel (all-to-all) attention */ } ao_op;
/* Transfer backends of P:397 / Fig.7.  CE = copy-engine peer memcpy on a side
 * stream with stream-memop flags; TMA = cp.async.bulk peer copies issued from
 * communication warps; LDST = 16-byte vector ld/st over NVSwitch from CUDA cores. */
typedef enum { AO_BACKEND_CE = 0, AO_BACKEND_TMA = 1, AO_BACKEND_LDST = 2 } ao_backend;
/* a P2P op recorded on the source side is a push, on the destination side a pull. */
typedef enum { AO_DIR_PUSH = 0, AO_DIR_PULL = 1 } ao_dir;
/* Order of a rank's ops: all chunks for peer r+1, then r+2, ... (shard-major, the Lst.2
 * rotation) or chunk j for every peer before chunk j+1 (chunk-major).  DESIGN.md Q3. */
typedef enum { AO_CHUNK_SHARD_MAJOR = 0, AO_CHUNK_CHUNK_MAJOR = 1 } ao_chunk_order;
/* Intra-chunk tile swizzle (Fig.6): row-major, column-major, Triton GROUP_M. */
typedef enum { AO_INTRA_ROW = 0, AO_INTRA_COL = 1, AO_INTRA_GROUPED = 2 } ao_intra;
/* GEMM-RS wire format of the partials.  FP32 is the conforming default (Q14). */
typedef enum { AO_WIRE_FP32 = 0, AO_WIRE_BF16 = 1 } ao_wire;
/* GEMM-RS reduction: SLOTS = each source writes its own fp32 slot and the owner's epilogue
 * sums them in ascending source rank (bitwise deterministic, default); ATOMIC = sources
 * reduce-add (red.global.add.f32, in the owner's L2 / over NVLink) into one accumulator that
 * the owner's epilogue adds to its own tile -- 1/(W-1) of the owner-side reads, summation
 * order not fixed (Q23). */
typedef enum { AO_RS_SLOTS = 0, AO_RS_ATOMIC = 1 } ao_rs_reduce;

typedef struct ao_ctx ao_ctx;
typedef struct ao_plan ao_plan;

/* Opaque per-rank handle for the symmetric workspace (IPC handle + metadata).  The caller
 * moves these between processes (e.g. torch.distributed.all_gather_object). */
typedef struct {
  unsigned char bytes[AO_HANDLE_BYTES];
} ao_handle_blob;

/* The chunk schedule description (the plan's whole config surface).
 * Integer fields hold the enums above.  0 in tile_m/tile_n/n_cta/timeout_ns = default. */
typedef struct {
  uint32_t struct_size; /* = sizeof(ao_plan_desc); ABI versioning */
  int32_t op;           /* ao_op */
  int32_t world_size;   /* W, 1..AO_MAX_WORLD */
  int32_t rank;         /* r, 0..W-1 */
  int64_t M;            /* AG: gathered rows (S = M/W per rank).  RS: rows of A and of the partial */
  int64_t N;            /* AG: this rank's columns of B/C.  RS: columns of C */
  int64_t K;            /* AG: reduction dim.  RS: this rank's K shard */
  int32_t chunk_rows;   /* C: rows per chunk; must divide S and be a multiple of 8 */
  int32_t backend;      /* ao_backend */
  int32_t dir;          /* ao_dir (PULL: AG only) */
  int32_t chunk_order;  /* ao_chunk_order */
  int32_t intra;        /* ao_intra */
  int32_t group_m;      /* GROUP_M for AO_INTRA_GROUPED */
  int32_t tile_m;       /* BM (0 = planner picks by wave-quantization utilization).  Shapes:
                           128x{128,256} (1 CTA), 256x{256,128} (CTA pair), 256x{224,208,192,160,
                           144,112} (CTA pair; AG + CE only), 512x256 (two pairs sharing B by
                           multicast; AG + CE, RS / AR atomic; needs n_cta) */
  int32_t tile_n;       /* BN (0 together with tile_m) */
  int32_t n_cta;        /* persistent GEMM CTAs (0 = SMs - comm_ctas) */
  int32_t comm_ctas;    /* TMA/LDST: 0 = co-located comm warps, >0 = dedicated comm CTAs */
  int32_t n_slices;     /* TMA/LDST: slices (flag words) per chunk; CE uses 1 */
  int32_t rs_wire;      /* ao_wire (RS only) */
  uint64_t timeout_ns;  /* device spin bound (0 = 5 s) */
  int32_t rs_reduce;    /* ao_rs_reduce (RS only) */
  int32_t topk;         /* A2A: experts per token (k); other ops: 0 */
  int32_t causal;       /* SP attention: 1 = causal mask over global token positions; other ops: 0 */
  int32_t stream_k;     /* AG (copy engine) / plain GEMM, tiles of <= 2 CTAs: split the last two
                           waves' tiles along K over all workers (data-parallel + stream-K tail,
                           DESIGN.md Q28) so a tile count that is not a multiple of the workers
                           leaves no idle tail wave.  0 = off, 1 = on, -1 = auto (on when the
                           wave utilization T / (ceil(T/n) n) < 0.9) */
} ao_plan_desc;

/* ---- status / version ---------------------------------------------------------------- */
const char* ao_status_string(ao_status s);
const char* ao_last_error(void); /* thread-local detail of the last failing call ("" if none) */
ao_status ao_version(int* major, int* minor);

/* ---- plans (host-only part: no GPU needed) ---------------------------------------------
 * ao_plan_desc_init: fills defaults (AG, W=1, CE, PUSH, SHARD_MAJOR, ROW, ...).
 * ao_plan_validate: checks a desc against the rules in DESIGN.md "Validation"
 *   (M % W, S % chunk_rows, K % 8, N % 8, tile shape, PULL only with AG, ...); returns
 *   AO_OK with *n_violations = 0 when valid, AO_ERR_INVALID_ARG otherwise; a ';'-separated
 *   list of violations is written to report (truncated to cap, NUL-terminated).
 * ao_plan_create_host: builds the chunk table, chunk->tile dependency table, tile order,
 *   per-CTA minimal wait lists and signal counts for a device with `sm_count`
 *   SMs, without binding to a ctx.  The result can be exported / hashed, not launched.
 * ao_plan_export_json: canonical JSON (sorted keys, no whitespace, integers only; the
 *   bit-exact contract checked against the oracle).  Writes min(cap, needed) bytes incl.
 *   the NUL; *needed = bytes required incl. NUL.
 * ao_plan_hash: FNV-1a 64 of the rank-independent part of the schedule.
 * ao_plan_workspace_bytes: symmetric workspace a ctx needs to run this desc (both epoch
 *   parities, data + flags). */
ao_status ao_plan_desc_init(ao_plan_desc* desc);
ao_status ao_plan_validate(const ao_plan_desc* desc, int sm_count, char* report, size_t cap,
                           int* n_violations);
ao_status ao_plan_create_host(const ao_plan_desc* desc, int sm_count, ao_plan** out);
ao_status ao_plan_export_json(const ao_plan* plan, char* buf, size_t cap, size_t* needed);
ao_status ao_plan_hash(const ao_plan* plan, uint64_t* out);
ao_status ao_plan_info(const ao_plan* plan, int32_t* tile_m, int32_t* tile_n, int32_t* cta_group,
                       int32_t* n_cta, int32_t* n_tiles, int32_t* n_chunks);
ao_status ao_plan_workspace_bytes(const ao_plan_desc* desc, size_t* bytes);
ao_status ao_plan_destroy(ao_plan* plan);

/* ---- symmetric memory (one ctx per rank) ------------------------------------------------
 * ao_ctx_create: selects `device`, checks it is sm_100, cudaMallocs the symmetric workspace
 *   (`workspace_bytes` of data, split in two epoch parities, plus flag words) and a
 *   host-mapped error word.  The workspace is owned by the library.
 * ao_ctx_export_handle: this rank's handle (cudaIpc memory handle + pid/device/size).
 * ao_ctx_import_handles: `all` has world_size entries indexed by rank (own entry ignored).
 *   Handles from the same process (loopback: several ranks on one GPU) are mapped
 *   directly; others through cudaIpcOpenMemHandle (NVLink P2P).  Fails with AO_ERR_PEER
 *   on a world/size mismatch.
 * ao_ctx_check_async: AO_ERR_TIMEOUT if a device spin-wait expired since the last check
 *   (detail in ao_last_error), else AO_OK.  Does not synchronize. */
ao_status ao_ctx_create(int device, int rank, int world_size, size_t workspace_bytes, ao_ctx** out);
ao_status ao_ctx_export_handle(ao_ctx* ctx, ao_handle_blob* out);
ao_status ao_ctx_import_handles(ao_ctx* ctx, const ao_handle_blob* all);
ao_status ao_ctx_check_async(ao_ctx* ctx);
ao_status ao_ctx_destroy(ao_ctx* ctx);

/* ---- plans bound to a ctx, and the ops -------------------------------------------------
 * ao_plan_create: ao_plan_create_host with the ctx's SM count, plus device copies of the
 *   tables.  The ctx must outlive the plan.
 * ao_ag_gemm: A_shard [M/W, K] (this rank's rows), B [N, K], C [M, N];
 *   A_gathered_out (nullable) [M, K] receives concat_p A_p (bit-exact copy).
 * ao_gemm_rs: A [M, K], B [N, K] (this rank's K shard), C_shard [M/W, N].
 * ao_*_group: ONE fused launch for n ranks of a world that live in this process on the
 *   same device (loopback).  plans[i] must belong to distinct ctxs of one world; the
 *   pointer arrays are indexed like plans.  The n=1 case equals the single-rank call.
 *   Space-sliced when n * (plan CTAs) <= SMs (each rank on its own CTAs, concurrently);
 *   TIME-SLICED when n == world_size and each plan asks for more than SMs / n CTAs (up to
 *   all SMs): every CTA serves every rank, walking one global list of the ranks' tile runs
 *   (AG rank after rank with destination-major pushes; RS / GEMM-AR owner after owner, the
 *   owner's own tiles after their contributions), with per-tile chunk waits (DESIGN.md
 *   Q24).  Otherwise AO_ERR_INVALID_ARG (the spin-waiting CTAs must be co-resident). */
ao_status ao_plan_create(ao_ctx* ctx, const ao_plan_desc* desc, ao_plan** out);
ao_status ao_ag_gemm(ao_plan* plan, const void* A_shard, const void* B, void* C, void* A_gathered_out,
                     void* stream);
ao_status ao_gemm_rs(ao_plan* plan, const void* A, const void* B, void* C_shard, void* stream);
ao_status ao_ag_gemm_group(int n, ao_plan* const* plans, const void* const* A_shards,
                           const void* const* Bs, void* const* Cs, void* const* A_gathered_outs,
                           void* stream);
ao_status ao_gemm_rs_group(int n, ao_plan* const* plans, const void* const* As, const void* const* Bs,
                           void* const* C_shards, void* stream);

/* ---- GEMM-AllReduce (NEXT-1; "GEMM--AllReduce", Fig.4d) -------------------
 * C[M, N] = sum_s A_s[M, K] . B_s[N, K]^T on EVERY rank (A, B as in ao_gemm_rs; C is the
 * caller's full [M, N] bf16 output, 16-byte aligned).  Partition-based AllReduce: the
 * GEMM-RS schedule (peers' fp32 partials pushed / reduce-added to the row owner, fused
 * owner reduction in the own tiles' epilogue), whose owner also writes its reduced bf16
 * rows to its symmetric buffer and releases a per-chunk flag; every rank's gather warps
 * pull the other owners' reduced chunks straight into C.  The plan's op must be
 * AO_OP_GEMM_AR with backend AO_BACKEND_LDST (gather transport) and comm_ctas == 0;
 * n_slices splits each gathered chunk.  Same collective rules and errors as ao_gemm_rs. */
ao_status ao_gemm_ar(ao_plan* plan, const void* A, const void* B, void* C, void* stream);
ao_status ao_gemm_ar_group(int n, ao_plan* const* plans, const void* const* As, const void* const* Bs,
                           void* const* Cs, void* stream);

/* ---- launch-level schedule of a group call (host-only; Q24) -------------------
 * What ao_{ag_gemm,gemm_rs,gemm_ar}_group(n, plans, ...) would run on a device with
 * `sm_count` SMs, as canonical JSON (sorted keys, no whitespace, integers only), written
 * like ao_plan_export_json (min(cap, needed) bytes incl. NUL; *needed = size incl. NUL).
 * plans: n plans (host-only ones suffice) in group order, equal hash; op: their ao_op
 * (AG_GEMM, GEMM_RS or GEMM_AR).
 *   {"mode":"space_sliced"}: each rank runs its own plan tables on its own CTAs;
 *   {"mode":"time_sliced","n_total":T,"n_workers":w,"segments":[[rank,k0,k1,o],...],
 *    "waits":[[worker,[[i,rank,g],...]],...]}: one global list of T tile positions --
 *   positions [k0,k1) of rank's plan order at global indices [o, o+k1-k0); worker w runs
 *   indices w, w+w_n, ... (Lst.1 persistent stride) and, before the tile at
 *   global index i, acquires the flags of chunk g of `rank` (AG: a chunk from another
 *   source that the tile's rows read; RS/AR: a chunk of the rank's own rows, from every
 *   other source), once per (worker, rank, chunk) (minimal waits).
 * Errors: AO_ERR_INVALID_ARG (bad n / op, or a group that cannot be co-resident: the
 * same condition under which the launch fails), AO_ERR_PEER (plan hashes differ). */
ao_status ao_group_schedule_export(int n, ao_plan* const* plans, int32_t op, int sm_count, char* buf, size_t cap,
                                   size_t* needed);

/* ---- A2A-GEMM (NEXT-3; P:437 / P:529 "A2A-GEMM"; BASELINE configs[3]) -------------------
 * Expert-parallel MoE dispatch fused with the expert GEMM: expert e lives on rank e
 * (W experts).  Rank s holds T = desc.M tokens X [T, K] bf16 and routing topk_idx [T, k]
 * int32 (device; k = desc.topk distinct expert ids per token).  The op forms, on every
 * rank e, A_e = concat_{s=0..W-1} X_s[tokens of s routed to e, ascending] (the
 * all_to_all_single layout, Q25) and computes Y = A_e . B^T with B [N, K] this
 * rank's expert weight.  Outputs (device, caller-owned):
 *   Y [W*T, N] bf16: rows [0, *recv_rows) valid, rows beyond are left untouched;
 *   route_pos [T, k] int32: row of (token t, choice j) in the Y of expert topk_idx[t, j];
 *   recv_rows [1] int32: number of received rows R_e.
 * Chunks are C = chunk_rows consecutive rows of one source's block; the count matrix is
 * exchanged first (every rank publishes its per-expert counts to every rank), then
 * in-kernel ld/st warps push each chunk (a row gather of the routed tokens) to its expert
 * and release a per-(source, chunk) flag that the tiles covering those rows wait on; the
 * tile order follows the arrival order (own rows, then sources e-1, e-2, ...).  Plan:
 * op AO_OP_A2A_GEMM, backend AO_BACKEND_LDST, dir PUSH, comm_ctas 0, 1 <= topk <= W,
 * (W*T) % tile_m == 0.  Same collective rules and errors as ao_ag_gemm.  The ranks' prep
 * kernels wait for each other (count exchange): ranks sharing one device must use
 * ao_a2a_gemm_group (per-rank calls on separate streams of one process can be serialised
 * by the driver's stream-to-hardware-queue mapping and time out). */
ao_status ao_a2a_gemm(ao_plan* plan, const void* X, const int32_t* topk_idx, const void* B, void* Y,
                      int32_t* route_pos, int32_t* recv_rows, void* stream);
ao_status ao_a2a_gemm_group(int n, ao_plan* const* plans, const void* const* Xs, const int32_t* const* topk_idxs,
                            const void* const* Bs, void* const* Ys, int32_t* const* route_pos,
                            int32_t* const* recv_rows, void* stream);

/* ---- SP attention (NEXT-4; "sequence-parallel (SP) schedules, including the
 * overlapped RingAttention", Fig.4c ring AllGather P:310) ----------------------------------
 * Rank r holds Q, K, V [H, S_loc, 128] bf16 (heads x its S_loc tokens x head dim 128) and
 * gets O [H, S_loc, 128] bf16 = softmax(Q K_all^T / sqrt(128)) V_all per head, non-causal,
 * over the keys/values of all ranks (concatenated in rank order).  The peers' K/V shards
 * are pushed by the copy engine in chunks of chunk_rows rows of the [H*S_loc, 128] view
 * (ring rotation), each released by a per-chunk flag; every (head, 128-query) tile
 * consumes its KV blocks in arrival order (own shard first, then r-1, r-2, ...) with an
 * online softmax, so the result does not depend on the order (Q27).  Plan: op
 * AO_OP_SP_ATTN, M = S_loc (multiple of 128), N = H, K = 128, chunk_rows a multiple of 128
 * dividing H*S_loc, backend AO_BACKEND_CE, dir PUSH, comm_ctas 0.  causal = 1: query
 * i of rank r (global position r*S_loc + i) sees keys at positions <= its own (RingAttention
 * with the causal mask: ranks s > r are skipped, rank r's own shard is masked on the
 * diagonal blocks); requires S_loc % 256 == 0.  Collective rules and errors as ao_ag_gemm. */
ao_status ao_sp_attn(ao_plan* plan, const void* Q, const void* K, const void* V, void* O, void* stream);
ao_status ao_sp_attn_group(int n, ao_plan* const* plans, const void* const* Qs, const void* const* Ks,
                           const void* const* Vs, void* const* Os, void* stream);

/* ---- HP attention (NEXT-4; "head-parallel (HP)" attention, DeepSpeed-Ulysses) -------
 * Same operands and result as ao_sp_attn (rank r holds Q, K, V [H, S_loc, 128] of its
 * tokens and gets O [H, S_loc, 128] = attention over the keys of all ranks), computed
 * head-parallel: rank r owns the head group G_r = [r*H/W, (r+1)*H/W).  The copy engine
 * pushes every source's Q, K, V rows of G_p to rank p (an all-to-all) in chunks of
 * chunk_rows rows of the [H/W * S_loc, 128] view of a source block, each released by a
 * per-chunk flag; rank r computes, for its heads, every source's queries against every
 * source's keys (items (source, head, 256 queries); keys in arrival order, causal: the
 * sources up to the query's), and writes each output tile straight to its owner: its own
 * rows into O, the other sources' rows into that source's symmetric return buffer, the last
 * tile of a (source, head group) block releasing a flag there; after the kernel the stream
 * waits for the W-1 return flags and copies the returned blocks into O (the reverse
 * all-to-all).  Plan: op AO_OP_HP_ATTN, M = S_loc (multiple of 256), N = H (multiple of W),
 * K = 128, chunk_rows a multiple of 128 dividing H/W * S_loc, backend CE, dir PUSH.
 * ao_hp_attn / ao_hp_attn_group are ao_sp_attn / ao_sp_attn_group on an HP plan. */
ao_status ao_hp_attn(ao_plan* plan, const void* Q, const void* K, const void* V, void* O, void* stream);
ao_status ao_hp_attn_group(int n, ao_plan* const* plans, const void* const* Qs, const void* const* Ks,
                           const void* const* Vs, void* const* Os, void* stream);

/* ---- plain local GEMM through the same tcgen05 mainloop (no communication) -------------
 * C[M, N] = A[M, K] . B[N, K]^T, bf16 in / fp32 accumulate / bf16 out (Lst.1's local
 * kernel).  Used for W = 1 and as the GEMM-only reference of the fused ops.
 * tile_m: 128 (1 CTA) or 256 (CTA pair, cta_group::2); 0 = 256 when M % 256 == 0.
 * tile_n: 128 or 256; 0 = 256.  Requires M % tile_m == 0, N % 8 == 0, K % 8 == 0. */
ao_status ao_gemm(int device, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                  int32_t tile_m, int32_t tile_n, void* stream);

/* ---- GEMM-only leg of the fused ops (SURVEY.md §8(d) baseline (iii)) -------------------
 * n independent problems C_i = A_i . B_i^T of one shape in ONE persistent launch of the
 * same kernel, each problem on its own n_cta workers (CTAs, or CTA pairs when tile_m =
 * 256), exactly as a loopback group of n ranks runs the fused ops, but with no transfers,
 * flags or reductions.  "Exposed communication" = T_fused - T_gemm_batched.
 * n in [1, AO_MAX_WORLD]; A_i [M, K], B_i [N, K], C_i [M, N] bf16 device pointers on
 * `device`, 16-byte aligned; tile_m/tile_n as ao_gemm (must be given, no 0 default
 * for tile_m unless M % 256 == 0); group_m: GROUP_M tile swizzle (0 = 16); n_cta: CTAs per
 * problem as in ao_plan_desc.n_cta (rounded down to whole CTA pairs when tile_m = 256;
 * 0 = SMs / n).  n * n_cta must not exceed the SM count (co-residency), else
 * AO_ERR_INVALID_ARG. */
ao_status ao_gemm_batched(int device, int n, const void* const* As, const void* const* Bs, void* const* Cs,
                          int64_t M, int64_t N, int64_t K, int32_t tile_m, int32_t tile_n, int32_t group_m,
                          int32_t n_cta, void* stream);

/* ---- E4: transfer-backend microbenchmark (Fig.2c,d) ------------
 * ao_transfer_bench: copy `bytes` from `src` (device, this ctx's GPU) to rank `peer`'s
 * symmetric data half (an IPC-mapped peer buffer, or this rank's own) in chunks of
 * chunk_bytes, `iters` times back to back, and return the mean ms per copy (CUDA events).
 *   AO_BACKEND_CE  : one cudaMemcpyAsync per chunk, round-robin over n_streams streams;
 *   AO_BACKEND_TMA : n_ctas CTAs x 8 warps, chunk c by warp c mod 8 n_ctas, cp.async.bulk
 *                    global -> smem -> global (the fused kernel's comm-warp code);
 *   AO_BACKEND_LDST: the same with 16-byte vector ld/st.
 * Requires bytes <= the ctx data half, 16-byte alignment.  Blocks until done. */
ao_status ao_transfer_bench(ao_ctx* ctx, int peer, int32_t backend, const void* src, int64_t bytes,
                            int64_t chunk_bytes, int32_t n_ctas, int32_t n_streams, int32_t iters,
                            float* ms_per_iter);

/* ---- device queries ---------------------------------------------------------------------
 * ao_device_query(device, key, out): "sm_count"; "cluster2_ctas" / "cluster4_ctas" = how
 * many CTAs of the fused kernel can be co-resident (one per SM) when launched in clusters
 * of 2 / 4 CTAs -- a 4-CTA cluster needs a free slot of 4 SMs inside one GPC, so not every
 * SM can host one.  The 512-row cluster tiles (tile_m 512, two CTA pairs sharing B by TMA
 * multicast) take their worker count from this: desc.n_cta = cluster4_ctas at most.
 * AO_ERR_UNSUPPORTED off sm_100, AO_ERR_INVALID_ARG for an unknown key. */
ao_status ao_device_query(int device, const char* key, int64_t* out);

/* ---- tracing -------------------------------------------------------------
 * ao_ctx_trace_enable: allocate a device event buffer of `capacity` events (0 = off).  Op
 *   launches whose first plan belongs to this ctx record %globaltimer-stamped events:
 *   chunk waits, tile loads, MMA, epilogue, transfers, reductions.
 * ao_ctx_trace_dump: synchronize, write the recorded events as Chrome-trace JSON to `path`
 *   (pid = rank, tid = CTA*8 + role), reset the buffer; *n_events = events written. */
ao_status ao_ctx_trace_enable(ao_ctx* ctx, int64_t capacity);
ao_status ao_ctx_trace_dump(ao_ctx* ctx, const char* path, int64_t* n_events);

/* ---- test hooks (deterministic fault injection; see tests/) ----------------------------
 * ao_debug_set: key "skip_wait" = index of a wait (global over CTAs) the kernel must skip
 * (-1 = none); "delay_ns" = nanosleep before each transfer/signal (fuzzes arrival order);
 * "prearrive" = 1: every chunk flag of a launch's ranks is set before it and no copy-engine
 * chain is issued (per-rank measurement with peers simulated as arrived); "gemm_stream_k"
 * = desc.stream_k of ao_gemm's internal plan (0 / 1 / -1). */
ao_status ao_debug_set(const char* key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* AUTOOVERLAP_H */
