// planner.h -- host chunk-schedule planner (no CUDA dependency).
//
// Builds, for one rank, the tables the fused kernels execute (§5.2):
//   chunk table          "a chunk is a logical block of data communicated as a unit"
//   per-rank op lists    the communication schedule `schedule := [rank, List[CommOp]]`
//                        -- 1-D swizzle AllGather (Lst.2) / owner-rotation RS
//   chunk->tile deps     "for each tile, we determine which chunks it reads and writes"
//   tile order           "reorder the sequence of waves so that each chunk is consumed as soon
//                        as it arrives ... intra-chunk swizzle"
//   per-CTA wait lists   "the minimal set of synchronization points"
// using closed forms (the oracle re-derives the same tables by enumeration; the two
// canonical JSON exports must match byte for byte).
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "autooverlap.h"

namespace ao {

struct TileShape {
  int bm, bn, cg;
};
// Tile shapes the kernels implement, in candidate order (Q19).
extern const TileShape kTileCandidates[];
extern const int kNumTileCandidates;
constexpr int kBK = 64;

enum OpTensor { TENSOR_A = 0, TENSOR_P = 1, TENSOR_C = 2 };
struct P2POp {
  int peer;
  int64_t row0, rows;
  int direction;  // ao_dir
  int accumulate;
  int tensor;     // OpTensor: gathered A (AG), fp32 partial P (RS), reduced C (AR gather)
};

struct HostPlan {
  ao_plan_desc desc{};
  int sm_count = 0;
  // derived
  int W = 1, rank = 0;
  int64_t M = 0, N = 0, K = 0, S = 0;
  int C = 0, n_chunks = 0, n_c = 0;
  TileShape tile{128, 256, 1};
  int n_cta = 1;  // workers (CTAs, or CTA pairs when cg == 2)
  int n_mb = 0, n_nb = 0, n_tiles = 0;
  bool is_ag = true;
  bool is_a2a = false;
  bool is_attn = false;  // SP or HP attention (NEXT-4)
  bool is_hp = false;    // HP (head-parallel, all-to-all) attention
  bool is_ar = false;  // GEMM-AR: the RS schedule + a pull AllGather of the reduced chunks
  // tables
  std::vector<std::array<int, 5>> chunks;  // g, row0, rows, src_or_owner, pos
  std::vector<std::vector<P2POp>> plans;   // all ranks
  std::vector<std::array<int, 4>> deps;    // t, g_lo, g_hi, group
  std::vector<int> order;
  std::vector<std::vector<std::array<int, 2>>> waits;  // per CTA: (k, g)
  std::vector<int> contrib;
  std::vector<int> tiles_per_chunk;                // RS
  // stream-K tail (Q28): positions [0, sk_dp) run data-parallel (worker c: c, c + n_cta, ...);
  // positions [sk_dp, n_tiles) are split along K into n_cta contiguous ranges of k-blocks
  // (sk_dp == n_tiles: off)
  int sk_dp = 1 << 30;
  int nkb = 0;
  std::string json;
  uint64_t hash = 0;
};

// Returns the list of violations (empty = valid).
std::vector<std::string> validate_desc(const ao_plan_desc& d, int sm_count);
// Picks the tile shape (explicit or utilization argmax).  false if none fits.
bool pick_tile(const ao_plan_desc& d, int sm_count, TileShape* out);
// Builds every table + the canonical JSON + hash.  Returns violations (empty = ok).
std::vector<std::string> build_plan(const ao_plan_desc& d, int sm_count, HostPlan* p);
// Workspace bytes per epoch parity for the data region of this desc.
size_t data_bytes_per_parity(const ao_plan_desc& d);
// GEMM-AR: byte offset of the owner's reduced bf16 rows [S, N] inside a data parity half.
size_t ar_reduced_offset(const ao_plan_desc& d);
// Flag words per parity this desc needs.
size_t a2a_max_chunks(const ao_plan_desc& d);
size_t flag_words_needed(const ao_plan_desc& d);

uint64_t fnv1a64(const std::string& s);

// Stream-K piece of a worker's walk: tile position k, k-blocks [kb0, kb1), role 0 = whole
// tile, 1 = tail piece (stores its fp32 partial), 2 = head piece (adds the tail's partial).
struct SkPiece {
  int k, kb0, kb1, role;
};
// The positions/pieces worker c runs, in order (shared by the wait tables and tests).
std::vector<SkPiece> worker_pieces(const HostPlan& p, int c);

}  // namespace ao
