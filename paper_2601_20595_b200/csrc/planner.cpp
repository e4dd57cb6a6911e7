// planner.cpp -- host chunk-schedule planner (closed forms; see planner.h).
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Qn = DESIGN.md reading n.
#include "planner.h"

#include <algorithm>
#include <map>
#include <sstream>
#include <tuple>

namespace ao {

// The first four shapes run every op; the narrower CTA-pair widths after them (wave-
// quantization-free tiles for the per-GPU TP shapes) are built for AG with copy-engine
// transfers (and the plain GEMM, which plans as a one-rank AG) only.
const TileShape kTileCandidates[] = {{256, 256, 2}, {256, 128, 2}, {128, 256, 1}, {128, 128, 1},
                                     {256, 224, 2}, {256, 208, 2}, {256, 192, 2}, {256, 160, 2},
                                     {256, 144, 2}, {256, 112, 2}, {512, 256, 4}};
constexpr int kNumAllOpTiles = 4;
constexpr int kClusterTile = 10;  // two CTA pairs sharing B by multicast (BM = 512)
// Relative mainloop efficiency (percent) per candidate: profiles/r02_tile_eff.json
// "eff_pct", written by scripts/measure_tile_eff.py on a B200 (plain GEMM, ~55 waves, no
// ragged edge, vs the 2-CTA 256x256 tile; Q19).  0 = explicit tile only.
static const int kTileEff[] = {100, 61, 87, 59, 94, 82, 85, 74, 68, 56, 0};
const int kNumTileCandidates = sizeof(kTileCandidates) / sizeof(kTileCandidates[0]);

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static const char* op_name(int op) {
  return op == AO_OP_AG_GEMM   ? "ag_gemm"
         : op == AO_OP_GEMM_RS ? "gemm_rs"
         : op == AO_OP_GEMM_AR ? "gemm_ar"
         : op == AO_OP_A2A_GEMM ? "a2a_gemm"
         : op == AO_OP_HP_ATTN  ? "hp_attn"
                                : "sp_attn";
}
static const char* tensor_name(int t) { return t == TENSOR_A ? "A" : (t == TENSOR_P ? "P" : "C"); }
static const char* backend_name(int b) { return b == AO_BACKEND_CE ? "ce" : (b == AO_BACKEND_TMA ? "tma" : "ldst"); }
static const char* dir_name(int d) { return d == AO_DIR_PUSH ? "push" : "pull"; }
static const char* chunk_order_name(int o) { return o == AO_CHUNK_SHARD_MAJOR ? "shard_major" : "chunk_major"; }
static const char* intra_name(int i) { return i == AO_INTRA_ROW ? "row" : (i == AO_INTRA_COL ? "col" : "grouped"); }

static int workers(const ao_plan_desc& d, int sm_count) { return d.n_cta > 0 ? d.n_cta : sm_count - d.comm_ctas; }

// Candidate i exists for this desc's op / backend (the narrow pair widths: AG + CE only).
// The 512-row cluster tile: AG + CE, and RS / AR with the atomic reduction (the slots
// reduction streams peer partials through the operand ring, which the two pairs share).
static bool tile_allowed(const ao_plan_desc& d, int i) {
  if (i < kNumAllOpTiles) return true;
  if (i == kClusterTile)
    return (d.op == AO_OP_AG_GEMM && d.backend == AO_BACKEND_CE) ||
           ((d.op == AO_OP_GEMM_RS || d.op == AO_OP_GEMM_AR) && d.rs_reduce == AO_RS_ATOMIC);
  return d.op == AO_OP_AG_GEMM && d.backend == AO_BACKEND_CE;
}

std::vector<std::string> validate_desc(const ao_plan_desc& d, int sm_count) {
  std::vector<std::string> v;
  if (d.struct_size != sizeof(ao_plan_desc)) v.push_back("struct_size");
  if (d.op != AO_OP_AG_GEMM && d.op != AO_OP_GEMM_RS && d.op != AO_OP_GEMM_AR && d.op != AO_OP_A2A_GEMM &&
      d.op != AO_OP_SP_ATTN && d.op != AO_OP_HP_ATTN)
    v.push_back("op");
  if (d.op == AO_OP_HP_ATTN) {
    // M = S_loc tokens per rank, N = heads (split over the ranks), K = head dim 128
    const int W = d.world_size;
    if (W < 1 || W > AO_MAX_WORLD) v.push_back("world_size");
    if (!(d.rank >= 0 && d.rank < std::max(W, 1))) v.push_back("rank");
    if (d.K != 128) v.push_back("head dim (K) must be 128");
    if (d.M <= 0 || d.M % 256 != 0) v.push_back("S_loc (M) % 256");
    if (d.N < 1 || (W >= 1 && d.N % W != 0)) v.push_back("heads (N) % world_size");
    const int64_t view = W >= 1 ? d.M * (d.N / std::max(W, 1)) : 0;  // rows of a source block
    if (d.chunk_rows <= 0 || d.chunk_rows % 128 != 0 || (view > 0 && view % d.chunk_rows != 0))
      v.push_back("chunk_rows");
    if (d.backend != AO_BACKEND_CE) v.push_back("backend for hp_attn");
    if (d.dir != AO_DIR_PUSH) v.push_back("dir for hp_attn");
    if (d.comm_ctas != 0) v.push_back("comm_ctas with hp_attn");
    if (d.topk != 0) v.push_back("topk");
    if (d.causal != 0 && d.causal != 1) v.push_back("causal");
    if (d.n_cta < 0) v.push_back("n_cta");
    return v;
  }
  if (d.op == AO_OP_SP_ATTN) {
    // M = S_loc tokens per rank, N = heads, K = head dim (the kernel is built for 128)
    const int W = d.world_size;
    if (W < 1 || W > AO_MAX_WORLD) v.push_back("world_size");
    if (!(d.rank >= 0 && d.rank < std::max(W, 1))) v.push_back("rank");
    if (d.K != 128) v.push_back("head dim (K) must be 128");
    if (d.M <= 0 || d.M % 128 != 0) v.push_back("S_loc (M) % 128");
    if (d.N < 1) v.push_back("heads (N)");
    if (d.chunk_rows <= 0 || d.chunk_rows % 128 != 0 || (d.M > 0 && d.N > 0 && (d.M * d.N) % d.chunk_rows != 0))
      v.push_back("chunk_rows");
    if (d.backend != AO_BACKEND_CE) v.push_back("backend for sp_attn");
    if (d.dir != AO_DIR_PUSH) v.push_back("dir for sp_attn");
    if (d.comm_ctas != 0) v.push_back("comm_ctas with sp_attn");
    if (d.topk != 0) v.push_back("topk");
    if (d.causal != 0 && d.causal != 1) v.push_back("causal");
    if (d.causal == 1 && d.M % 256 != 0) v.push_back("causal needs S_loc (M) % 256");
    if (d.n_cta < 0) v.push_back("n_cta");
    return v;
  }
  const int W = d.world_size;
  if (W < 1 || W > AO_MAX_WORLD) v.push_back("world_size");
  if (!(d.rank >= 0 && d.rank < std::max(W, 1))) v.push_back("rank");
  if (d.M < 0 || d.N < 0 || d.K < 0) v.push_back("shape");
  if (d.causal != 0) v.push_back("causal");
  const bool a2a = d.op == AO_OP_A2A_GEMM;
  if (a2a) {
    // M = tokens per rank T; the received rows R_e <= W*T are routing-dependent (Q25)
    if (d.topk < 1 || d.topk > W) v.push_back("topk");
    if (d.chunk_rows <= 0 || d.chunk_rows % 8 != 0) v.push_back("chunk_rows");
    if (d.backend != AO_BACKEND_LDST) v.push_back("backend for a2a_gemm");
    if (d.dir != AO_DIR_PUSH) v.push_back("dir for a2a_gemm");
    if (d.comm_ctas != 0) v.push_back("comm_ctas with a2a_gemm");
  } else {
    if (d.topk != 0) v.push_back("topk");
    if (W >= 1 && d.M % W != 0) v.push_back("M % world_size");
  }
  const int64_t S = W >= 1 ? d.M / W : 0;
  if (!a2a && (d.chunk_rows <= 0 || d.chunk_rows % 8 != 0 || (S > 0 && S % d.chunk_rows != 0)))
    v.push_back("chunk_rows");
  if (d.K % 8 != 0) v.push_back("K % 8");
  if (d.N % 8 != 0) v.push_back("N % 8");
  if (d.backend < AO_BACKEND_CE || d.backend > AO_BACKEND_LDST) v.push_back("backend");
  if (d.dir != AO_DIR_PUSH && d.dir != AO_DIR_PULL) v.push_back("dir");
  if (d.dir == AO_DIR_PULL && d.op == AO_OP_GEMM_RS) v.push_back("pull with gemm_rs");
  if (d.dir == AO_DIR_PULL && d.op == AO_OP_GEMM_AR) v.push_back("pull with gemm_ar");
  // GEMM-AR's gather phase is pulled by in-kernel ld/st warps (the RS kernel's smem is full)
  if (d.op == AO_OP_GEMM_AR && d.backend != AO_BACKEND_LDST) v.push_back("backend for gemm_ar");
  if (d.op == AO_OP_GEMM_AR && d.comm_ctas != 0) v.push_back("comm_ctas with gemm_ar");
  if (d.chunk_order != AO_CHUNK_SHARD_MAJOR && d.chunk_order != AO_CHUNK_CHUNK_MAJOR) v.push_back("chunk_order");
  if (d.intra < AO_INTRA_ROW || d.intra > AO_INTRA_GROUPED) v.push_back("intra");
  if (d.intra == AO_INTRA_GROUPED && d.group_m < 1) v.push_back("group_m");
  if (d.comm_ctas < 0 || d.comm_ctas >= sm_count) v.push_back("comm_ctas");
  if (d.n_cta < 0) v.push_back("n_cta");
  if (d.n_slices < 1 || d.n_slices > 64) v.push_back("n_slices");
  if (d.rs_wire != AO_WIRE_FP32 && d.rs_wire != AO_WIRE_BF16) v.push_back("rs_wire");
  // the bf16 partial wire breaks the per-element bound (Q14): built for GEMM-RS
  // with the atomic reduction only (bf16 TMA reduce-adds into a bf16 accumulator), accepted
  // and flagged non-conforming by ao_plan_create / ao_plan_create_host (ao_last_error)
  if (d.rs_wire == AO_WIRE_BF16 && (d.op == AO_OP_GEMM_AR || (d.op == AO_OP_GEMM_RS && d.rs_reduce != AO_RS_ATOMIC)))
    v.push_back("rs_wire bf16 (GEMM-RS with rs_reduce atomic only)");
  if (d.rs_reduce != AO_RS_SLOTS && d.rs_reduce != AO_RS_ATOMIC) v.push_back("rs_reduce");
  if (d.stream_k < -1 || d.stream_k > 1) v.push_back("stream_k");
  if (d.stream_k == 1 && (d.op != AO_OP_AG_GEMM || d.backend != AO_BACKEND_CE || d.tile_m == 512))
    v.push_back("stream_k (AG with the copy engine, tiles of <= 2 CTAs)");
  if ((d.tile_m == 0) != (d.tile_n == 0)) v.push_back("tile");
  if (d.tile_m != 0) {
    bool ok = false;
    for (int i = 0; i < kNumTileCandidates; ++i)
      if (kTileCandidates[i].bm == d.tile_m && kTileCandidates[i].bn == d.tile_n && tile_allowed(d, i)) ok = true;
    if (!ok) v.push_back("tile");
    // clusters of 4 CTAs do not fit every SM (whole GPC slots): the worker count is the
    // caller's (ao_device_query "cluster4_ctas"), never derived here
    if (ok && d.tile_m == 512 && d.n_cta <= 0) v.push_back("n_cta (512-row cluster tile)");
  }
  if (v.empty()) {
    TileShape t;
    if (!pick_tile(d, sm_count, &t)) v.push_back("no tile shape fits");
  }
  return v;
}

// Q19: explicit tile, else the least estimated time waves * (per-SM area) / efficiency,
// waves = ceil(T / n); exact comparison by cross-multiplication; ties ->
// larger BM*BN, then larger BN.
bool pick_tile(const ao_plan_desc& d, int sm_count, TileShape* out) {
  if (d.op == AO_OP_A2A_GEMM) {
    // the tile grid is routing-dependent: explicit tile, else the largest candidate that
    // divides the receive capacity W*T (row blocks never straddle its end)
    const int64_t cap = int64_t(d.world_size) * d.M;
    for (int i = 0; i < kNumAllOpTiles; ++i) {
      const TileShape c = kTileCandidates[i];
      if (d.tile_m != 0 && !(c.bm == d.tile_m && c.bn == d.tile_n)) continue;
      if (cap % c.bm != 0) continue;
      *out = c;
      return true;
    }
    return false;
  }
  const int64_t S = d.M / d.world_size;
  bool have = false;
  int64_t best_num = 0, best_eff = 1, best_den = 1, best_area = -1, best_bn = -1;
  for (int i = 0; i < kNumTileCandidates; ++i) {
    const TileShape c = kTileCandidates[i];
    if (!tile_allowed(d, i)) continue;
    if (d.tile_m != 0 && !(c.bm == d.tile_m && c.bn == d.tile_n)) continue;
    if (d.tile_m == 0 && kTileEff[i] == 0) continue;
    if (S % c.bm != 0) continue;
    const int64_t n = std::max(1, workers(d, sm_count) / c.cg);
    const int64_t T = (d.M / c.bm) * ceil_div(d.N, c.bn);
    // cost = waves * per-SM tile area / eff, waves = ceil(T / n); with a stream-K tail (Q28)
    // the waves are T / n (the last partial wave is spread over all workers): cost = num / (den * eff)
    const bool sk = d.op == AO_OP_AG_GEMM && d.backend == AO_BACKEND_CE && c.cg <= 2 && d.K > 0 && T > n &&
                    T % n != 0 && (d.stream_k == 1 || (d.stream_k == -1 && T * 10 < ceil_div(T, n) * n * 9));
    const int64_t num = (sk ? T : ceil_div(T, n)) * (int64_t(c.bm) * c.bn / c.cg);
    const int64_t den = sk ? n : 1;
    const int64_t eff = kTileEff[i] > 0 ? kTileEff[i] : 1;
    const int64_t area = int64_t(c.bm) * c.bn;
    bool better;
    if (!have) {
      better = true;
    } else {
      const __int128 lhs = __int128(num) * best_eff * best_den, rhs = __int128(best_num) * eff * den;  // cost < best
      better = lhs < rhs || (lhs == rhs && std::make_tuple(area, int64_t(c.bn)) > std::make_tuple(best_area, best_bn));
    }
    if (better) {
      have = true;
      best_num = num;
      best_eff = eff;
      best_den = den;
      best_area = area;
      best_bn = c.bn;
      *out = c;
    }
  }
  return have;
}

size_t ar_reduced_offset(const ao_plan_desc& d) {
  // after the W slots [W*S, N] fp32 (slots mode); atomic mode keeps the same size so that
  // the ctx's accumulator region (data half / W) holds [S, N] fp32
  return size_t(d.M) * size_t(d.N) * 4;
}

size_t data_bytes_per_parity(const ao_plan_desc& d) {
  if (d.op == AO_OP_AG_GEMM) return size_t(d.M) * size_t(d.K) * 2;  // gathered A
  if (d.op == AO_OP_A2A_GEMM) return size_t(d.world_size) * size_t(d.M) * size_t(d.K) * 2;  // receive buffer
  if (d.op == AO_OP_SP_ATTN)  // gathered K then V, [W][H*S_loc][128] bf16 each
    return 2 * size_t(d.world_size) * size_t(d.N) * size_t(d.M) * size_t(d.K) * 2;
  if (d.op == AO_OP_HP_ATTN)  // gathered Q, K, V and the O return buffer, [W][H/W*S_loc][128] bf16 each
    return 4 * size_t(d.N) * size_t(d.M) * size_t(d.K) * 2;
  if (d.op == AO_OP_GEMM_AR)  // (slots) + the owner's reduced rows [S, N] bf16
    return ar_reduced_offset(d) + size_t(d.world_size > 0 ? d.M / d.world_size : 0) * size_t(d.N) * 2;
  const size_t eb = d.rs_wire == AO_WIRE_BF16 ? 2 : 4;
  return size_t(d.M) * size_t(d.N) * eb;  // W slots of [S, N]
}

size_t a2a_max_chunks(const ao_plan_desc& d) { return d.chunk_rows > 0 ? size_t(ceil_div(d.M, d.chunk_rows)) : 0; }

size_t flag_words_needed(const ao_plan_desc& d) {
  if (d.op == AO_OP_SP_ATTN)  // chunk flags [W sources][H*S_loc / chunk_rows]
    return d.chunk_rows > 0 ? size_t(d.world_size) * size_t(d.M * d.N / d.chunk_rows) : 0;
  if (d.op == AO_OP_HP_ATTN)  // chunk flags [W sources][H/W*S_loc / chunk_rows], then O return flags [W]
    return d.chunk_rows > 0 && d.world_size > 0
               ? size_t(d.world_size) * size_t(d.M * (d.N / d.world_size) / d.chunk_rows) + size_t(d.world_size)
               : 0;
  if (d.op == AO_OP_A2A_GEMM)  // chunk flags [W][maxJ] (the count exchange uses the reserved tail)
    return size_t(d.world_size) * a2a_max_chunks(d);
  const size_t nch = d.chunk_rows > 0 ? size_t(d.M / d.chunk_rows) : 0;
  if (d.op == AO_OP_AG_GEMM) return nch * size_t(d.backend == AO_BACKEND_CE ? 1 : d.n_slices);
  if (d.op == AO_OP_GEMM_AR) return nch * size_t(d.world_size) + nch;  // + per-chunk "reduced" flags
  return nch * size_t(d.world_size);
}

uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// ---------------------------------------------------------------------------------------
// canonical JSON writer: keys sorted bytewise (== Python json.dumps(sort_keys=True) for
// ASCII keys), separators (',', ':'), integers only.
namespace {
struct Obj {
  std::map<std::string, std::string> kv;
  void put(const std::string& k, const std::string& raw) { kv[k] = raw; }
  void put(const std::string& k, int64_t v) { kv[k] = std::to_string(v); }
  void put_str(const std::string& k, const std::string& s) { kv[k] = "\"" + s + "\""; }
  std::string str() const {
    std::string o = "{";
    bool first = true;
    for (auto& e : kv) {
      if (!first) o += ",";
      first = false;
      o += "\"" + e.first + "\":" + e.second;
    }
    return o + "}";
  }
};
template <class T>
std::string int_list(const T& v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ",";
    o += std::to_string(v[i]);
  }
  return o + "]";
}
template <class T>
std::string list_of(const std::vector<T>& v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ",";
    o += int_list(v[i]);
  }
  return o + "]";
}
}  // namespace

static std::string rank_independent_key(const HostPlan& p) {
  const ao_plan_desc& d = p.desc;
  Obj o;
  o.put_str("op", op_name(d.op));
  o.put("world_size", p.W);
  o.put("M", p.M);
  o.put("N", p.N);
  o.put("K", p.K);
  o.put("chunk_rows", p.C);
  o.put("tile", int_list(std::vector<int>{p.tile.bm, p.tile.bn, p.tile.cg}));
  o.put_str("backend", backend_name(d.backend));
  o.put_str("dir", dir_name(d.dir));
  o.put_str("chunk_order", chunk_order_name(d.chunk_order));
  o.put_str("intra", intra_name(d.intra));
  o.put("group_m", d.group_m);
  o.put("n_cta", p.n_cta);
  o.put("comm_ctas", d.comm_ctas);
  o.put("n_slices", d.backend == AO_BACKEND_CE ? 1 : d.n_slices);
  o.put("rs_wire", d.rs_wire);
  o.put("rs_reduce", d.rs_reduce);
  if (d.op == AO_OP_A2A_GEMM) o.put("topk", d.topk);
  if (d.op == AO_OP_SP_ATTN || d.op == AO_OP_HP_ATTN) o.put("causal", d.causal);
  if (p.sk_dp < p.n_tiles) o.put("sk_dp", p.sk_dp);
  return o.str();
}

std::vector<SkPiece> worker_pieces(const HostPlan& p, int c) {
  std::vector<SkPiece> out;
  const int n = p.n_cta, nkb = p.nkb;
  for (int k = c; k < p.sk_dp; k += n) out.push_back({k, 0, nkb, 0});
  if (p.sk_dp < p.n_tiles) {
    const int64_t U = int64_t(p.n_tiles - p.sk_dp) * nkb;
    int64_t u = U * c / n;
    const int64_t u1 = U * (c + 1) / n;
    while (u < u1) {
      const int t = int(u / nkb), kb0 = int(u % nkb);
      const int kb1 = int(std::min<int64_t>(nkb, kb0 + (u1 - u)));
      out.push_back({p.sk_dp + t, kb0, kb1, (kb0 == 0 && kb1 == nkb) ? 0 : (kb0 != 0 ? 1 : 2)});
      u += kb1 - kb0;
    }
  }
  return out;
}

std::vector<std::string> build_plan(const ao_plan_desc& d, int sm_count, HostPlan* p) {
  std::vector<std::string> viol = validate_desc(d, sm_count);
  if (!viol.empty()) return viol;
  HostPlan& P = *p;
  P = HostPlan{};
  P.desc = d;
  P.sm_count = sm_count;
  P.W = d.world_size;
  P.rank = d.rank;
  P.M = d.M;
  P.N = d.N;
  P.K = d.K;
  P.S = d.M / d.world_size;
  P.C = d.chunk_rows;
  P.is_ag = d.op == AO_OP_AG_GEMM;
  P.is_ar = d.op == AO_OP_GEMM_AR;
  P.is_a2a = d.op == AO_OP_A2A_GEMM;
  P.is_attn = d.op == AO_OP_SP_ATTN || d.op == AO_OP_HP_ATTN;
  P.is_hp = d.op == AO_OP_HP_ATTN;
  if (P.is_hp) {
    // HP attention (NEXT-4): items (query source, head of the group, 256 queries); one chunk =
    // chunk_rows rows of a source's [H/W * S_loc, 128] Q, K and V blocks
    P.tile = TileShape{256, 128, 1};
    P.n_cta = std::max(1, workers(d, sm_count));
    P.S = d.M;
    P.n_c = int(d.M * (d.N / P.W) / d.chunk_rows);
    P.n_chunks = P.W * P.n_c;
    P.n_mb = int(P.W * (d.N / P.W) * (d.M / 256));
    P.n_nb = 1;
    P.n_tiles = P.n_mb;
    Obj o;
    o.put_str("op", op_name(d.op));
    o.put("world_size", P.W);
    o.put("rank", P.rank);
    o.put("S_loc", P.M);
    o.put("heads", P.N);
    o.put("heads_per_rank", P.N / P.W);
    o.put("head_dim", P.K);
    o.put("chunk_rows", P.C);
    o.put("chunks_per_source", P.n_c);
    o.put_str("backend", backend_name(d.backend));
    o.put_str("dir", dir_name(d.dir));
    o.put("n_cta", P.n_cta);
    o.put("items", P.n_tiles);
    o.put_str("kv_order", d.causal ? "query_source_down" : "ring");
    o.put("causal", d.causal);
    P.json = o.str();
    P.hash = fnv1a64(rank_independent_key(P));
    return {};
  }
  if (P.is_attn) {
    // SP attention (NEXT-4): items (head, 128 queries), KV blocks of 128 in arrival order;
    // one chunk = chunk_rows rows of a source's [H*S_loc, 128] K and V
    P.tile = TileShape{128, 128, 1};
    P.n_cta = std::max(1, workers(d, sm_count));
    P.S = d.M;
    P.n_c = int(d.M * d.N / d.chunk_rows);
    P.n_chunks = P.W * P.n_c;
    P.n_mb = int(d.N * (d.M / 128));
    P.n_nb = 1;
    P.n_tiles = P.n_mb;
    Obj o;
    o.put_str("op", op_name(d.op));
    o.put("world_size", P.W);
    o.put("rank", P.rank);
    o.put("S_loc", P.M);
    o.put("heads", P.N);
    o.put("head_dim", P.K);
    o.put("chunk_rows", P.C);
    o.put("chunks_per_source", P.n_c);
    o.put_str("backend", backend_name(d.backend));
    o.put_str("dir", dir_name(d.dir));
    o.put("n_cta", P.n_cta);
    o.put("items", P.n_tiles);
    o.put_str("kv_order", "ring");
    o.put("causal", d.causal);
    P.json = o.str();
    P.hash = fnv1a64(rank_independent_key(P));
    return {};
  }
  pick_tile(d, sm_count, &P.tile);
  P.n_cta = std::max(1, workers(d, sm_count) / P.tile.cg);
  if (P.is_a2a) {
    // A2A (NEXT-3): the chunk table, dependency table and tile order are functions of the
    // routing counts, built on the device after the count exchange (Q25); the
    // host plan fixes the rest of the schedule: chunk rows, tile, workers, intra order.
    P.S = d.M;
    P.n_c = int(a2a_max_chunks(d));
    P.n_chunks = P.W * P.n_c;
    P.n_nb = int(ceil_div(P.N, P.tile.bn));
    P.n_mb = int(int64_t(P.W) * P.M / P.tile.bm);
    P.n_tiles = P.n_mb * P.n_nb;  // capacity; the launched count is routing-dependent
    Obj o;
    o.put_str("op", op_name(d.op));
    o.put("world_size", P.W);
    o.put("rank", P.rank);
    o.put("M", P.M);
    o.put("N", P.N);
    o.put("K", P.K);
    o.put("topk", d.topk);
    o.put("chunk_rows", P.C);
    o.put("tile", int_list(std::vector<int>{P.tile.bm, P.tile.bn, P.tile.cg}));
    o.put_str("backend", backend_name(d.backend));
    o.put_str("dir", dir_name(d.dir));
    o.put_str("intra", intra_name(d.intra));
    o.put("group_m", d.group_m);
    o.put("n_cta", P.n_cta);
    o.put("max_chunks_per_source", P.n_c);
    o.put("dynamic", 1);
    P.json = o.str();
    P.hash = fnv1a64(rank_independent_key(P));
    return {};
  }
  P.n_chunks = int(P.M / P.C);
  P.n_c = int(P.S / P.C);
  P.n_mb = int(P.M / P.tile.bm);
  P.n_nb = int(ceil_div(P.N, P.tile.bn));
  P.n_tiles = P.n_mb * P.n_nb;
  const int W = P.W, r = P.rank, n_c = P.n_c;

  // Rule 1: chunk g covers rows [gC, (g+1)C); src/owner = floor(gC / S); j = index in shard.
  auto owner_of = [&](int g) { return int((int64_t(g) * P.C) / P.S); };
  auto j_of = [&](int g) { return int((int64_t(g) * P.C - int64_t(owner_of(g)) * P.S) / P.C); };

  // Rule 2/3: per-rank op lists and arrival positions (closed forms).
  P.plans.assign(W, {});
  for (int q = 0; q < W; ++q) {
    std::vector<P2POp>& ops = P.plans[q];
    if (P.is_ag) {
      // Lst.2: peer = (i + rank) mod W for i = 1..W-1 (Q1); push sends own shard, pull
      // fetches the peer's shard.
      auto emit = [&](int dstep, int j) {
        const int peer = (q + dstep) % W;
        const int src = d.dir == AO_DIR_PUSH ? q : peer;
        const int g = src * n_c + j;
        ops.push_back(P2POp{peer, int64_t(g) * P.C, P.C, d.dir, 0, TENSOR_A});
      };
      if (d.chunk_order == AO_CHUNK_SHARD_MAJOR) {
        for (int ds = 1; ds < W; ++ds)
          for (int j = 0; j < n_c; ++j) emit(ds, j);
      } else {
        for (int j = 0; j < n_c; ++j)
          for (int ds = 1; ds < W; ++ds) emit(ds, j);
      }
    } else {
      // owners q+1, ..., q+W-1, then q (own rows last)
      auto emit = [&](int e, int j) {
        const int o = (q + e + 1) % W;
        const int g = o * n_c + j;
        ops.push_back(P2POp{o, int64_t(g) * P.C, P.C, AO_DIR_PUSH, 1, TENSOR_P});
      };
      if (d.chunk_order == AO_CHUNK_SHARD_MAJOR) {
        for (int e = 0; e < W; ++e)
          for (int j = 0; j < n_c; ++j) emit(e, j);
      } else {
        // chunk-major with the own chunk lagged by one round (Q21)
        for (int j = 0; j < n_c; ++j) {
          for (int e = 0; e < W - 1; ++e) emit(e, j);
          if (j >= 1) emit(W - 1, j - 1);
        }
        if (n_c > 0) emit(W - 1, n_c - 1);
      }
      if (P.is_ar) {
        // GEMM-AR = partition-based AllReduce (Fig.4d): after the ReduceScatter part,
        // q pulls every other owner's reduced chunk j (owners reduce their chunks in
        // ascending j), owners in the 1-D rotation q+1, ..., q+W-1 (Lst.2).
        for (int j = 0; j < n_c; ++j)
          for (int ds = 1; ds < W; ++ds) {
            const int o = (q + ds) % W;
            ops.push_back(P2POp{o, int64_t(o * n_c + j) * P.C, P.C, AO_DIR_PULL, 0, TENSOR_C});
          }
      }
    }
  }
  P.chunks.resize(P.n_chunks);
  for (int g = 0; g < P.n_chunks; ++g) {
    const int src = owner_of(g), j = j_of(g);
    int pos;
    if (P.is_ag) {
      if (src == r) {
        pos = 0;
      } else {
        const int dstep = d.dir == AO_DIR_PUSH ? (r - src + W) % W : (src - r + W) % W;
        const int idx = d.chunk_order == AO_CHUNK_SHARD_MAJOR ? (dstep - 1) * n_c + j : j * (W - 1) + (dstep - 1);
        pos = 1 + idx;
      }
    } else {
      const int dd = (src - r + W) % W;
      const int e = dd == 0 ? W - 1 : dd - 1;
      if (d.chunk_order == AO_CHUNK_SHARD_MAJOR) {
        pos = e * n_c + j;
      } else if (e < W - 1) {
        pos = j == 0 ? e : j * W - 1 + e;  // round 0 has W-1 ops, later rounds W
      } else {
        pos = j < n_c - 1 ? (j + 2) * W - 2 : n_c * W - 1;  // own chunk j lagged into round j+1
      }
    }
    P.chunks[g] = {g, int(int64_t(g) * P.C), P.C, src, pos};
  }

  // Rule 4/5: deps and groups.
  const int BM = P.tile.bm;
  P.deps.resize(P.n_tiles);
  std::vector<int> glo_of(P.n_tiles), ghi_of(P.n_tiles);
  for (int t = 0; t < P.n_tiles; ++t) {
    const int mb = t / P.n_nb;
    const int64_t r0 = int64_t(mb) * BM, r1 = std::min<int64_t>(P.M, int64_t(mb + 1) * BM);
    const int glo = int(r0 / P.C), ghi = int(ceil_div(r1, P.C) - 1);
    int grp = 0;
    for (int g = glo; g <= ghi; ++g) grp = std::max(grp, P.chunks[g][4]);
    P.deps[t] = {t, glo, ghi, grp};
    glo_of[t] = glo;
    ghi_of[t] = ghi;
  }

  // Rule 6: stable sort by (group, intra key).
  auto intra_key = [&](int t) {
    const int mb = t / P.n_nb, nb = t % P.n_nb;
    if (d.intra == AO_INTRA_ROW) return std::make_tuple(mb, nb, 0);
    if (d.intra == AO_INTRA_COL) return std::make_tuple(nb, mb, 0);
    return std::make_tuple(mb / d.group_m, nb, mb);
  };
  P.order.resize(P.n_tiles);
  for (int t = 0; t < P.n_tiles; ++t) P.order[t] = t;
  std::stable_sort(P.order.begin(), P.order.end(), [&](int a, int b) {
    return std::make_tuple(P.deps[a][3], intra_key(a)) < std::make_tuple(P.deps[b][3], intra_key(b));
  });

  // RS: tiles_per_chunk (tiles contributing to chunk g at a source rank).
  if (!P.is_ag) {
    P.tiles_per_chunk.assign(P.n_chunks, 0);
    for (int g = 0; g < P.n_chunks; ++g) {
      const int64_t r0 = int64_t(g) * P.C, r1 = r0 + P.C - 1;
      const int mb_lo = int(r0 / BM), mb_hi = int(r1 / BM);
      P.tiles_per_chunk[g] = (mb_hi - mb_lo + 1) * P.n_nb;
    }
  }

  // Rules 7/8: CTA k mod n_cta; one wait per (CTA, chunk) first use.  AG tiles wait for
  // remote chunks; RS own-row tiles (fused peer reduction in their epilogue) wait for the
  // other sources' contributions.
  // Stream-K tail (Q28): AG with the copy engine (and plain GEMM), <= 2-CTA tiles.
  P.nkb = int(ceil_div(P.K, kBK));
  P.sk_dp = P.n_tiles;
  {
    const int T = P.n_tiles, n = P.n_cta;
    const bool able = P.is_ag && d.backend == AO_BACKEND_CE && P.tile.cg <= 2 && P.nkb > 0 && T > n && T % n != 0;
    const bool want = d.stream_k == 1 || (d.stream_k == -1 && int64_t(T) * 10 < int64_t(ceil_div(T, n)) * n * 9);
    if (able && want) P.sk_dp = (T / n - 1) * n;
  }
  P.waits.assign(P.n_cta, {});
  std::vector<int> seen(P.n_chunks, -1);
  for (int c = 0; c < P.n_cta; ++c) {
    for (const SkPiece& pc : worker_pieces(P, c)) {
      const int k = pc.k;
      const int t = P.order[k];
      for (int g = glo_of[t]; g <= ghi_of[t]; ++g) {
        const bool own = P.chunks[g][3] == r;
        if (P.is_ag ? own : (!own || W == 1)) continue;
        if (seen[g] == c) continue;
        seen[g] = c;
        P.waits[c].push_back({k, g});
      }
    }
  }

  // Rule 9: signal words per chunk at this rank.
  P.contrib.resize(P.n_chunks);
  const int ns = d.backend == AO_BACKEND_CE ? 1 : d.n_slices;
  for (int g = 0; g < P.n_chunks; ++g) {
    const bool own = P.chunks[g][3] == r;
    P.contrib[g] = P.is_ag ? (own ? 0 : ns) : (own ? W - 1 : 0);
  }

  // ---- canonical export ---------------------------------------------------------------
  Obj o;
  o.put_str("op", op_name(d.op));
  o.put("world_size", W);
  o.put("rank", r);
  o.put("M", P.M);
  o.put("N", P.N);
  o.put("K", P.K);
  o.put("chunk_rows", P.C);
  o.put("tile", int_list(std::vector<int>{P.tile.bm, P.tile.bn, P.tile.cg}));
  o.put_str("backend", backend_name(d.backend));
  o.put_str("dir", dir_name(d.dir));
  o.put_str("chunk_order", chunk_order_name(d.chunk_order));
  o.put_str("intra", intra_name(d.intra));
  o.put("group_m", d.group_m);
  o.put("n_cta", P.n_cta);
  o.put("comm_ctas", d.comm_ctas);
  o.put("n_slices", ns);
  {
    Obj tens;
    if (P.is_ag) {
      Obj a, c;
      a.put("elem_bytes", 2);
      a.put("shape", int_list(std::vector<int64_t>{P.M, P.K}));
      c.put("elem_bytes", 2);
      c.put("shape", int_list(std::vector<int64_t>{P.M, P.N}));
      tens.put("A", a.str());
      tens.put("C", c.str());
    } else {  // RS and AR: output C, fp32 partials P
      Obj c, pp;
      c.put("elem_bytes", 2);
      c.put("shape", int_list(std::vector<int64_t>{P.M, P.N}));
      pp.put("elem_bytes", 4);
      pp.put("shape", int_list(std::vector<int64_t>{P.M, P.N}));
      tens.put("C", c.str());
      tens.put("P", pp.str());
    }
    o.put("tensors", tens.str());
  }
  {
    std::string s = "[";
    for (int q = 0; q < W; ++q) {
      if (q) s += ",";
      Obj reg;
      if (P.is_ag) {
        reg.put("A", "[" + int_list(std::vector<int64_t>{int64_t(q) * P.S, P.S}) + "]");
      } else {
        if (P.is_ar) reg.put("C", "[" + int_list(std::vector<int64_t>{int64_t(q) * P.S, P.S}) + "]");
        reg.put("P", "[" + int_list(std::vector<int64_t>{0, P.M}) + "]");
      }
      s += reg.str();
    }
    o.put("owner_regions", s + "]");
  }
  {
    std::string s = "[";
    for (int q = 0; q < W; ++q) {
      if (q) s += ",";
      s += "[";
      for (size_t i = 0; i < P.plans[q].size(); ++i) {
        const P2POp& op = P.plans[q][i];
        if (i) s += ",";
        Obj e;
        e.put("accumulate", op.accumulate);
        e.put("deps", "[]");
        e.put_str("direction", dir_name(op.direction));
        e.put("dst_chunk", int_list(std::vector<int64_t>{op.row0, op.rows}));
        e.put("peer", op.peer);
        e.put("src_chunk", int_list(std::vector<int64_t>{op.row0, op.rows}));
        e.put_str("tensor", tensor_name(op.tensor));
        e.put_str("variant", "p2p");
        s += e.str();
      }
      s += "]";
    }
    o.put("plans", s + "]");
  }
  o.put("chunks", list_of(P.chunks));
  o.put("deps", list_of(P.deps));
  o.put("order", int_list(P.order));
  {
    std::string s = "[";
    for (int c = 0; c < P.n_cta; ++c) {
      if (c) s += ",";
      s += "[" + std::to_string(c) + "," + list_of(P.waits[c]) + "]";
    }
    o.put("waits", s + "]");
  }
  o.put("contrib", int_list(P.contrib));
  if (P.sk_dp < P.n_tiles) o.put("sk_dp", P.sk_dp);
  if (!P.is_ag) {
    o.put("tiles_per_chunk", int_list(P.tiles_per_chunk));
    o.put_str("rs_reduce", d.rs_reduce == AO_RS_ATOMIC ? "atomic" : "slots");
    if (d.rs_wire == AO_WIRE_BF16) o.put_str("rs_wire", "bf16");
  }
  P.json = o.str();
  P.hash = fnv1a64(rank_independent_key(P));
  return {};
}

}  // namespace ao
