"""Brute-force CPU oracle for the chunk schedule of the AutoOverlap hot path.

TEST INFRASTRUCTURE ONLY (see oracle/numeric.py header for who may import it).  This
module shares no code with the C++ planner (paper_2601_20595_b200/csrc/planner.cpp);
tests compare the two canonical JSON exports byte for byte.

It follows, step by step, the paper's chunk-scheduling pipeline (§5.1-§5.2)
as made concrete by SURVEY.md §8(c) rules 1-9 and the readings Q1-Q20 listed in
DESIGN.md, deliberately by enumeration rather than closed forms:

  1. Chunks    -- "a chunk is a logical block of data that is communicated as a unit"
                  (P:288); row membership is enumerated row by row.
  2. Plans     -- the communication schedule `schedule := [rank, List[CommOp]]`
                  built as explicit per-rank op lists: the 1-D swizzle AllGather of
                  Lst.2 (peer = (i + rank) mod W, reading Q1) and the owner-
                  rotation ReduceScatter swizzle.
  3. Arrival   -- a chunk's position = 1 + index of the op that delivers it, found by
                  scanning the issuer's op list (P:295 push/pull: the op is recorded on
                  exactly one side).
  4. Deps      -- "for each tile, we determine which chunks it reads and writes based on
                  its tile index and the tensor layout": tile rows are enumerated.
  5. Group     -- a tile joins the latest chunk it needs.
  6. Order     -- "reorder the sequence of waves so that each chunk is consumed as soon
                  as it arrives, and apply an intra-chunk swizzle".
  7. CTAs      -- static persistent stride `tile_id += NUM_SMS` of Lst.1.
  8. Waits     -- "the minimal set of synchronization points ... a tile that consumes a
                  given chunk cannot start until the corresponding communication operator
                  has completed": one wait per (CTA, chunk) first use.
  9. Signals   -- "global-memory signals": per-chunk flag words.  In GEMM-RS the
                  owner's own-row tiles come last and their epilogue fuses the peer reduction
                  (north star: "the epilogue of gemm_rs fusing the peer reduction"), so those
                  tiles wait for the W-1 other sources of their chunks.

GEMM-AR is the partition-based AllReduce of Fig.4d: the
GEMM-RS schedule followed by a pull AllGather of the owners' reduced chunks.

Canonical export: JSON, sorted keys, no whitespace, integers only, strings only for
enum names.  Parity: not applicable (exact).
"""
from __future__ import annotations

import json
import math

# Tile shapes the kernel library implements, in the planner's candidate order
# (BM, BN, cta_group).  Shared *specification* with the C++ planner (Q19);
# each side types it independently.
TILE_CANDIDATES = [(256, 256, 2), (256, 128, 2), (128, 256, 1), (128, 128, 1)]
# Narrower CTA-pair widths (wave-quantization-free tiles for the per-GPU TP shapes, Q19),
# built for AG with the copy-engine backend only.
PAIR_TILES_AG_CE = [(256, 224, 2), (256, 208, 2), (256, 192, 2), (256, 160, 2), (256, 144, 2), (256, 112, 2)]
# Two CTA pairs stacked along M sharing B by multicast (a 4-CTA cluster, BM = 512): AG with
# the copy engine, and RS / AR with the atomic reduction; the worker count (clusters that
# fit the GPU) is always given explicitly (n_cta).
CLUSTER_TILES = [(512, 256, 4)]
# Relative mainloop efficiency (percent) of each candidate: the measurement record
# profiles/r02_tile_eff.json "eff_pct" (scripts/measure_tile_eff.py on a B200: plain GEMM
# with ~55 waves of the shape's own tiles, no ragged edge, relative to 256x256).  Planner
# spec constant shared with the C++ planner (Q19); tests pin it to the record.
TILE_EFF = {(256, 256, 2): 100, (256, 128, 2): 61, (128, 256, 1): 87, (128, 128, 1): 59,
            (256, 224, 2): 94, (256, 208, 2): 82, (256, 192, 2): 85, (256, 160, 2): 74, (256, 144, 2): 68,
            (256, 112, 2): 56, (512, 256, 4): 0}  # 0: explicit tile only (never picked automatically)


def tile_candidates(desc):
    """The shapes a desc may use (in planner order)."""
    if desc["op"] == "ag_gemm" and desc["backend"] == "ce":
        return TILE_CANDIDATES + PAIR_TILES_AG_CE + CLUSTER_TILES
    if desc["op"] in ("gemm_rs", "gemm_ar") and desc.get("rs_reduce", "slots") == "atomic":
        return TILE_CANDIDATES + CLUSTER_TILES
    return list(TILE_CANDIDATES)

BK = 64  # K-block of the mainloop (TMA 128-B swizzle => 64 bf16), DESIGN.md


def _ceil_div(a, b):
    return -(-a // b)


def default_desc(**kw):
    d = dict(op="ag_gemm", world_size=2, rank=0, M=512, N=512, K=512, chunk_rows=64,
             backend="ce", dir="push", chunk_order="shard_major", intra="row", group_m=1,
             tile_m=0, tile_n=0, n_cta=0, comm_ctas=0, n_slices=1, rs_reduce="slots")
    d.update(kw)
    return d


def validate(desc, sm_count=148):
    """Violations as data.  Returns a list of strings, empty = valid."""
    v = []
    W, r = desc["world_size"], desc["rank"]
    M, N, K, C = desc["M"], desc["N"], desc["K"], desc["chunk_rows"]
    if desc["op"] not in ("ag_gemm", "gemm_rs", "gemm_ar"):
        v.append("op")
    if W < 1 or W > 8:
        v.append("world_size")
    if not (0 <= r < max(W, 1)):
        v.append("rank")
    if M < 0 or N < 0 or K < 0:
        v.append("shape")
    if W >= 1 and M % W != 0:
        v.append("M % world_size")
    S = M // W if W >= 1 else 0
    if C <= 0 or C % 8 != 0 or (S > 0 and S % C != 0):
        v.append("chunk_rows")
    if K % 8 != 0:
        v.append("K % 8")
    if N % 8 != 0:
        v.append("N % 8")
    if desc["backend"] not in ("ce", "tma", "ldst"):
        v.append("backend")
    if desc["dir"] not in ("push", "pull"):
        v.append("dir")
    if desc["dir"] == "pull" and desc["op"] == "gemm_rs":
        v.append("pull with gemm_rs")
    if desc["dir"] == "pull" and desc["op"] == "gemm_ar":
        v.append("pull with gemm_ar")
    if desc["op"] == "gemm_ar" and desc["backend"] != "ldst":
        v.append("backend for gemm_ar")
    if desc["op"] == "gemm_ar" and desc["comm_ctas"] != 0:
        v.append("comm_ctas with gemm_ar")
    if desc["chunk_order"] not in ("shard_major", "chunk_major"):
        v.append("chunk_order")
    if desc["intra"] not in ("row", "col", "grouped"):
        v.append("intra")
    if desc["intra"] == "grouped" and desc["group_m"] < 1:
        v.append("group_m")
    if desc["comm_ctas"] < 0 or desc["comm_ctas"] >= sm_count:
        v.append("comm_ctas")
    if desc["n_cta"] < 0:
        v.append("n_cta")
    if desc["n_slices"] < 1 or desc["n_slices"] > 64:
        v.append("n_slices")
    # DESIGN.md Q14: bf16 partials break the per-element bound; built (non-conforming) for
    # GEMM-RS with the atomic reduction only
    if desc.get("rs_wire", "fp32") == "bf16" and (desc["op"] == "gemm_ar" or (
            desc["op"] == "gemm_rs" and desc.get("rs_reduce", "slots") != "atomic")):
        v.append("rs_wire bf16")
    if desc.get("rs_reduce", "slots") not in ("slots", "atomic"):
        v.append("rs_reduce")
    sk = desc.get("stream_k", 0)
    if sk not in (-1, 0, 1):
        v.append("stream_k")
    if sk == 1 and (desc["op"] != "ag_gemm" or desc["backend"] != "ce" or desc["tile_m"] == 512):
        v.append("stream_k (AG with the copy engine, tiles of <= 2 CTAs)")
    if (desc["tile_m"] == 0) != (desc["tile_n"] == 0):
        v.append("tile")
    if desc["tile_m"] and (desc["tile_m"], desc["tile_n"]) not in [(a, b) for a, b, _ in tile_candidates(desc)]:
        v.append("tile")
    elif desc["tile_m"] == 512 and desc["n_cta"] <= 0:
        v.append("n_cta (512-row cluster tile)")
    if not v and pick_tile(desc, sm_count) is None:
        v.append("no tile shape fits")
    return v


def n_workers(desc, sm_count):
    return desc["n_cta"] if desc["n_cta"] > 0 else sm_count - desc["comm_ctas"]


def pick_tile(desc, sm_count):
    """Tile shape: explicit, else the candidate with the least estimated time
    waves * (per-SM tile area) / efficiency, waves = ceil(T / n) -- wave quantization
    (Fig.2a) weighted by the measured per-shape efficiency (Q19).  Exact
    rational comparison; ties -> larger BM*BN, then larger BN.  Enumerates every candidate."""
    from fractions import Fraction
    W, M, N = desc["world_size"], desc["M"], desc["N"]
    S = M // W
    cands = tile_candidates(desc)
    if desc["tile_m"]:
        cands = [c for c in cands if (c[0], c[1]) == (desc["tile_m"], desc["tile_n"])]
    else:
        cands = [c for c in cands if TILE_EFF[c] > 0]
    best = None
    for bm, bn, cg in cands:
        if S % bm != 0:
            continue
        n = max(1, n_workers(desc, sm_count) // cg)
        T = (M // bm) * _ceil_div(N, bn)
        # with a stream-K tail (Q28) the last partial wave is spread over all workers: T / n waves
        waves = Fraction(T, n) if stream_k_dp(desc, T, n, cg) < T else _ceil_div(T, n)
        cost = Fraction(waves * (bm * bn // cg), max(1, TILE_EFF[(bm, bn, cg)]))
        key = (-cost, bm * bn, bn)
        if best is None or key > best[0]:
            best = (key, (bm, bn, cg))
    return None if best is None else best[1]


def _chunks(desc):
    """Rule 1 by enumeration: row -> chunk membership, chunk -> (row0, rows, src/owner)."""
    W, M, C = desc["world_size"], desc["M"], desc["chunk_rows"]
    S = M // W
    n_chunks = M // C if C > 0 else 0
    row_chunk = [None] * M
    rows_of = [[] for _ in range(n_chunks)]
    for i in range(M):
        g = i // C
        row_chunk[i] = g
        rows_of[g].append(i)
    chunks = []
    for g in range(n_chunks):
        rows = rows_of[g]
        row0 = rows[0]
        owner = row0 // S  # the shard holding row0 (AG source / RS owner)
        assert all(x // S == owner for x in rows), "chunk spans shards"
        chunks.append((row0, len(rows), owner))
    return chunks, row_chunk


def _shard_chunks(chunks, p):
    """Chunks of shard p in row order (their index j inside the shard)."""
    return [g for g, (_, _, o) in enumerate(chunks) if o == p]


def _build_plans(desc, chunks):
    """Per-rank op lists -- 1-D swizzle AllGather (Lst.2) for AG, owner-rotation
    ReduceScatter for RS.  Op dicts use SPEC's P2P fields."""
    W = desc["world_size"]
    plans = []
    for q in range(W):
        ops = []
        if desc["op"] == "ag_gemm":
            # Lst.2: for i in range(mesh): peer = (i + rank) % mesh; skip self (Q1).
            peers = [(i + q) % W for i in range(W) if (i + q) % W != q]
            if desc["dir"] == "push":
                # push: q sends its own shard's chunks to each peer
                per_peer = [(p, _shard_chunks(chunks, q)) for p in peers]
            else:
                # pull: q fetches each peer's shard chunks (Lst.2 TransferOp.PULL)
                per_peer = [(p, _shard_chunks(chunks, p)) for p in peers]
            seq = []
            if desc["chunk_order"] == "shard_major":
                for p, gs in per_peer:
                    for g in gs:
                        seq.append((p, g))
            else:
                n_c = len(per_peer[0][1]) if per_peer else 0
                for j in range(n_c):
                    for p, gs in per_peer:
                        seq.append((p, gs[j]))
            for p, g in seq:
                row0, rows, _ = chunks[g]
                ops.append({"accumulate": 0, "deps": [], "direction": desc["dir"], "dst_chunk": [row0, rows],
                            "peer": p, "src_chunk": [row0, rows], "tensor": "A", "variant": "p2p"})
        else:
            # RS: owners q+1, ..., q+W-1, then q itself (own rows last, SURVEY rule 3)
            owners = [(q + e + 1) % W for e in range(W)]
            seq = []
            if desc["chunk_order"] == "shard_major":
                for o in owners:
                    for g in _shard_chunks(chunks, o):
                        seq.append((o, g))
            else:
                # chunk-major: round j = chunk j of every peer owner; the own (local
                # accumulate) op of chunk j is lagged into round j+1, so the owner's fused
                # reduction of chunk j never waits on the peer tile issued just before it
                # (reading Q21); the last own chunk closes the list.
                n_c = len(_shard_chunks(chunks, 0)) if W > 0 else 0
                for j in range(n_c):
                    for o in owners[:-1]:
                        seq.append((o, _shard_chunks(chunks, o)[j]))
                    if j >= 1:
                        seq.append((q, _shard_chunks(chunks, q)[j - 1]))
                if n_c:
                    seq.append((q, _shard_chunks(chunks, q)[n_c - 1]))
            for o, g in seq:
                row0, rows, _ = chunks[g]
                ops.append({"accumulate": 1, "deps": [], "direction": "push", "dst_chunk": [row0, rows],
                            "peer": o, "src_chunk": [row0, rows], "tensor": "P", "variant": "p2p"})
            if desc["op"] == "gemm_ar":
                # Partition-based AllReduce (Fig.4d): the ReduceScatter above, then q
                # fetches every other owner's reduced chunk (owners finish their chunks in
                # ascending j), owners visited in the Lst.2 rotation q+1, ..., q+W-1.
                n_c = len(_shard_chunks(chunks, 0)) if W > 0 else 0
                for j in range(n_c):
                    for i in range(1, W):
                        o = (q + i) % W
                        row0, rows, _ = chunks[_shard_chunks(chunks, o)[j]]
                        ops.append({"accumulate": 0, "deps": [], "direction": "pull", "dst_chunk": [row0, rows],
                                    "peer": o, "src_chunk": [row0, rows], "tensor": "C", "variant": "p2p"})
        plans.append(ops)
    return plans


def _arrival_pos(desc, chunks, plans):
    """Rule 2/3: arrival position of every chunk at this rank, by scanning op lists."""
    W, r = desc["world_size"], desc["rank"]
    pos = []
    for g, (row0, rows, owner) in enumerate(chunks):
        if desc["op"] == "ag_gemm":
            if owner == r:
                pos.append(0)
                continue
            found = None
            if desc["dir"] == "push":
                for idx, op in enumerate(plans[owner]):
                    if op["peer"] == r and op["src_chunk"] == [row0, rows]:
                        found = idx
                        break
            else:
                for idx, op in enumerate(plans[r]):
                    if op["peer"] == owner and op["src_chunk"] == [row0, rows]:
                        found = idx
                        break
            assert found is not None
            pos.append(1 + found)
        else:
            found = None
            for idx, op in enumerate(plans[r]):
                if op["tensor"] == "P" and op["src_chunk"] == [row0, rows]:
                    found = idx
                    break
            assert found is not None
            pos.append(found)
    return pos


def _intra_key(desc, mb, nb):
    if desc["intra"] == "row":
        return (mb, nb)
    if desc["intra"] == "col":
        return (nb, mb)
    gm = desc["group_m"]
    return (mb // gm, nb, mb)


def plan(desc, sm_count=148):
    """Build the full canonical schedule for desc['rank'] (raises on invalid desc)."""
    viol = validate(desc, sm_count)
    if viol:
        raise ValueError("invalid desc: " + ", ".join(viol))
    W, r = desc["world_size"], desc["rank"]
    M, N, K, C = desc["M"], desc["N"], desc["K"], desc["chunk_rows"]
    S = M // W
    bm, bn, cg = pick_tile(desc, sm_count)
    nw = n_workers(desc, sm_count)
    n_cta = max(1, nw // cg)
    chunks, row_chunk = _chunks(desc)
    plans = _build_plans(desc, chunks)
    pos = _arrival_pos(desc, chunks, plans)
    is_ag = desc["op"] == "ag_gemm"

    n_mb, n_nb = M // bm, _ceil_div(N, bn)
    T = n_mb * n_nb
    deps = []
    tile_chunks = []
    group = []
    for t in range(T):
        mb, nb = divmod(t, n_nb)
        gs = sorted({row_chunk[i] for i in range(mb * bm, min(M, (mb + 1) * bm))})
        assert gs == list(range(gs[0], gs[-1] + 1))
        tile_chunks.append(gs)
        grp = max(pos[g] for g in gs)
        group.append(grp)
        deps.append([t, gs[0], gs[-1], grp])

    keyed = []
    for t in range(T):
        mb, nb = divmod(t, n_nb)
        keyed.append(((group[t],) + _intra_key(desc, mb, nb), t))
    keyed.sort(key=lambda x: x[0])
    order = [t for _, t in keyed]

    tiles_per_chunk = []
    if not is_ag:
        tiles_per_chunk = [sum(1 for t in range(T) if g in tile_chunks[t]) for g in range(len(chunks))]

    # CTA assignment: position k -> CTA k mod n_cta, except a stream-K tail (DESIGN.md
    # Q28).  Waits: AG tiles wait for their remote chunks; RS own-row tiles (whose epilogue
    # fuses the peer reduction) wait for the other sources' contributions to their chunks.
    sk_dp = stream_k_dp(desc, T, n_cta, cg)
    positions = worker_positions(T, n_cta, sk_dp, _ceil_div(K, BK))
    waits = []
    for c in range(n_cta):
        seen = set()
        lst = []
        for k in positions[c]:
            t = order[k]
            if is_ag:
                need = [g for g in tile_chunks[t] if chunks[g][2] != r]
            else:
                need = [g for g in tile_chunks[t] if chunks[g][2] == r] if W > 1 else []
            for g in need:
                if g not in seen:
                    seen.add(g)
                    lst.append([k, g])
        waits.append([c, lst])

    if is_ag:
        contrib = [0 if chunks[g][2] == r else (1 if desc["backend"] == "ce" else desc["n_slices"])
                   for g in range(len(chunks))]
    else:
        contrib = [W - 1 if chunks[g][2] == r else 0 for g in range(len(chunks))]

    if is_ag:
        tensors = {"A": {"elem_bytes": 2, "shape": [M, K]}, "C": {"elem_bytes": 2, "shape": [M, N]}}
        owner_regions = [{"A": [[p * S, S]]} for p in range(W)]
    else:
        tensors = {"C": {"elem_bytes": 2, "shape": [M, N]}, "P": {"elem_bytes": 4, "shape": [M, N]}}
        if desc["op"] == "gemm_ar":  # the reduced rows each owner contributes to the gather
            owner_regions = [{"C": [[p * S, S]], "P": [[0, M]]} for p in range(W)]
        else:
            owner_regions = [{"P": [[0, M]]} for p in range(W)]

    out = {
        "op": desc["op"], "world_size": W, "rank": r, "M": M, "N": N, "K": K, "chunk_rows": C,
        "tile": [bm, bn, cg], "backend": desc["backend"], "dir": desc["dir"],
        "chunk_order": desc["chunk_order"], "intra": desc["intra"], "group_m": desc["group_m"],
        "n_cta": n_cta, "comm_ctas": desc["comm_ctas"],
        "n_slices": 1 if desc["backend"] == "ce" else desc["n_slices"],
        "tensors": tensors, "owner_regions": owner_regions, "plans": plans,
        "chunks": [[g, chunks[g][0], chunks[g][1], chunks[g][2], pos[g]] for g in range(len(chunks))],
        "deps": deps, "order": order, "waits": waits, "contrib": contrib,
    }
    if not is_ag:
        out["tiles_per_chunk"] = tiles_per_chunk
        out["rs_reduce"] = desc.get("rs_reduce", "slots")
        if desc.get("rs_wire", "fp32") == "bf16":
            out["rs_wire"] = "bf16"
    if sk_dp < T:
        out["sk_dp"] = sk_dp
    return out


def stream_k_dp(desc, T, n, cg):
    """Q28 (data-parallel + stream-K tail): the number of tile positions run data-parallel.
    When T tiles do not fill whole waves of n workers, the last two waves' tiles are split
    along K instead (sk_dp = (T // n - 1) * n); T when off or not applicable.  'Auto' (-1)
    turns it on when the wave utilization T / (ceil(T / n) * n) is below 0.9."""
    from fractions import Fraction
    nkb = _ceil_div(desc["K"], BK)
    sk = desc.get("stream_k", 0)
    able = desc["op"] == "ag_gemm" and desc["backend"] == "ce" and cg <= 2 and nkb > 0 and T > n and T % n != 0
    want = sk == 1 or (sk == -1 and Fraction(T, _ceil_div(T, n) * n) < Fraction(9, 10))
    return (T // n - 1) * n if able and want else T


def worker_positions(T, n, sk_dp, nkb):
    """Tile positions each worker runs, in order.  Data-parallel part: worker c runs
    c, c + n, ... below sk_dp (Lst.1's persistent stride).  Stream-K part: the (T - sk_dp) *
    nkb (position, k-block) units, in position-major order, are cut into n contiguous
    ranges, worker c getting units [floor(U c / n), floor(U (c + 1) / n)); it runs every
    position one of its units belongs to.  Enumerated unit by unit."""
    pos = [list(range(c, sk_dp, n)) for c in range(n)]
    U = (T - sk_dp) * nkb
    bounds = [U * c // n for c in range(n + 1)]
    c = 0
    for u in range(U):
        while u >= bounds[c + 1]:
            c += 1
        k = sk_dp + u // nkb
        if not pos[c] or pos[c][-1] != k:
            pos[c].append(k)
    return pos


def worker_pieces(T, n, sk_dp, nkb, c):
    """Worker c's (position, kb0, kb1, role) pieces: role 0 = whole tile, 1 = a tail piece
    (k-blocks up to the end; stores its fp32 partial), 2 = a head piece (k-blocks from 0;
    adds the tail's partial and stores the tile).  Enumerated unit by unit."""
    dp_part = [[k, 0, nkb, 0] for k in range(c, sk_dp, n)]
    sk_part = []
    U = (T - sk_dp) * nkb
    for u in range(U * c // n, U * (c + 1) // n):
        k, kb = sk_dp + u // nkb, u % nkb
        if sk_part and sk_part[-1][0] == k:
            sk_part[-1][2] = kb + 1  # units of one position are consecutive k-blocks
        else:
            sk_part.append([k, kb, kb + 1, 0])
    out = dp_part + sk_part
    for p in out:
        p[3] = 0 if (p[1] == 0 and p[2] == nkb) else (1 if p[1] != 0 else 2)
    return out


def export_json(p) -> str:
    """Canonical export: sorted keys, no whitespace (byte-exact contract)."""
    return json.dumps(p, sort_keys=True, separators=(",", ":"))


def sm_utilization(n_tiles, sm_count):
    """tile_count / (wave_count * sm_count)."""
    waves = math.ceil(n_tiles / sm_count)
    return n_tiles / (waves * sm_count)


def group_schedule(descs, sm_count=148):
    """Launch-level schedule of a group call over the ranks `descs` (group order), by
    enumeration (Q24 -- one GPU standing in for W ranks).  Returns
    {"mode": "space_sliced"} when the ranks' persistent CTAs fit side by side, the
    time-sliced list otherwise, or None when the launch is refused (CTAs not co-resident).

    Time-sliced: every worker serves every rank, walking one global list of (rank, plan
    position) entries with Lst.1's persistent stride:
      * AG -- rank after rank, each rank's plan order intact;
      * RS / AR -- owner after owner; for owner o the positions of source ranks o+1, o+2,
        ..., o+W-1 (the rotation; reversed for odd owners -- serpentine, Q24)
        whose tile rows o owns, then o's own positions (its tiles wait on every other
        source's contribution, so they come after them).
    Waits: before each tile a worker acquires the chunks the tile's rows intersect
    that it needs from peers -- AG: chunks of another source; RS: the own tile's chunks --
    the first time the worker needs (rank, chunk)."""
    plans = [plan(d, sm_count) for d in descs]
    d0, p0 = descs[0], plans[0]
    n, W = len(descs), d0["world_size"]
    bm, _, cg = p0["tile"]
    ctas = p0["n_cta"] * cg
    is_ag = d0["op"] == "ag_gemm"
    comm = is_ag and d0["backend"] != "ce" and W > 1
    comm_ctas = d0["comm_ctas"] if comm else 0
    if n * (ctas + comm_ctas) <= sm_count:
        return {"mode": "space_sliced"}
    if not (n > 1 and n == W and ctas <= sm_count and comm_ctas == 0 and (not is_ag or d0["dir"] == "push")):
        return None
    M, C = d0["M"], d0["chunk_rows"]
    S = M // W
    n_nb = _ceil_div(d0["N"], p0["tile"][1])
    gi_of = {d["rank"]: gi for gi, d in enumerate(descs)}

    def rows_of(gi, k):
        t = plans[gi]["order"][k]
        mb = t // n_nb
        return range(mb * bm, min(M, (mb + 1) * bm))

    seq = []
    if is_ag:
        for gi in range(n):
            for k in range(len(plans[gi]["order"])):
                seq.append((gi, k))
    else:
        if S % bm != 0:
            return None
        for o in range(W):
            # even owners: sources o+1, o+2, ...; odd owners: the reverse (serpentine, so each
            # phase starts on the weights the previous one read last); own positions last
            steps = list(range(1, W)) if o % 2 == 0 else list(range(W - 1, 0, -1))
            for step in steps + [0]:
                gi = gi_of[(o + step) % W]
                for k in range(len(plans[gi]["order"])):
                    if rows_of(gi, k)[0] // S == o:
                        seq.append((gi, k))
    segments = []
    for i, (gi, k) in enumerate(seq):
        if segments and segments[-1][0] == gi and segments[-1][2] == k:
            segments[-1][2] = k + 1
        else:
            segments.append([gi, k, k + 1, i])
    if len(segments) > 256:
        return None
    n_wk = ctas // cg
    waits = []
    for w in range(n_wk):
        seen = set()
        lst = []
        for i in range(w, len(seq), n_wk):
            gi, k = seq[i]
            r = descs[gi]["rank"]
            rows = rows_of(gi, k)
            chunks = sorted({x // C for x in rows})
            if is_ag:
                need = [g for g in chunks if (g * C) // S != r]
            else:
                need = chunks if rows[0] // S == r else []
            for g in need:
                if (gi, g) not in seen:
                    seen.add((gi, g))
                    lst.append([i, r, g])
        waits.append([w, lst])
    return {"mode": "time_sliced", "n_total": len(seq), "n_workers": n_wk,
            "segments": [[descs[gi]["rank"], k0, k1, o] for gi, k0, k1, o in segments], "waits": waits}
