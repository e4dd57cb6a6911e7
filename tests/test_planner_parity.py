"""C++ planner (through the C ABI, host-only calls) vs the brute-force oracle planner:
canonical JSON exports must be byte-identical (SURVEY.md §8(c) "Schedule result"), and
both must accept / reject the same descs.  Also checks that the C-ABI library exports
every symbol include/autooverlap.h declares.  No GPU needed."""
import itertools
import json
import os
import re
import subprocess

import pytest

from oracle import schedule as osch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _sweep():
    out = []
    for W in (1, 2, 4, 8):
        for op in ("ag_gemm", "gemm_rs"):
            for S in (128, 256, 384):
                for C in (64, 128, 256):
                    if S % C:
                        continue
                    for intra, gm in (("row", 1), ("col", 1), ("grouped", 2), ("grouped", 3)):
                        for order in ("shard_major", "chunk_major"):
                            for dirn in (("push", "pull") if op == "ag_gemm" else ("push",)):
                                for tile in ((128, 128), (128, 256), (0, 0)):
                                    out.append(dict(op=op, world_size=W, M=S * W, N=392, K=136, chunk_rows=C,
                                                    intra=intra, group_m=gm, chunk_order=order, dir=dirn,
                                                    tile_m=tile[0], tile_n=tile[1], n_cta=7 if S == 256 else 0,
                                                    backend="ce" if S != 384 else "tma", n_slices=3))
    # GEMM-AR (NEXT-1): RS schedule + pull gather of the reduced chunks
    for W in (1, 2, 3, 4, 8):
        for S, C in ((128, 64), (256, 128), (384, 128), (256, 256)):
            for order in ("shard_major", "chunk_major"):
                for red in ("slots", "atomic"):
                    for tile in ((128, 128), (0, 0)):
                        out.append(dict(op="gemm_ar", world_size=W, M=S * W, N=392, K=136, chunk_rows=C,
                                        intra="grouped", group_m=2, chunk_order=order, rs_reduce=red,
                                        tile_m=tile[0], tile_n=tile[1], n_cta=7 if S == 256 else 0,
                                        backend="ldst", n_slices=4))
    return out


SWEEP = _sweep()


@pytest.mark.parametrize("i", range(0, len(SWEEP), 3))
def test_json_byte_exact(ao, i):
    d = SWEEP[i]
    for r in range(d["world_size"]):
        dd = osch.default_desc(**dict(d, rank=r))
        ref = osch.export_json(osch.plan(dd, sm_count=148))
        got = ao.plan_json(dd, sm_count=148)
        assert got == ref, (d, r)


@pytest.mark.parametrize("sms", [132, 148])
def test_json_byte_exact_full_shapes(ao, sms):
    # BASELINE configs[1]/[2] at TP=8 (planner only; tile heuristic engaged)
    for op, M, N, K, C in (("ag_gemm", 8192, 1792, 4096, 128), ("gemm_rs", 8192, 4096, 1792, 128),
                           ("ag_gemm", 8192, 1792, 4096, 1024)):
        for r in (0, 5):
            dd = osch.default_desc(op=op, world_size=8, rank=r, M=M, N=N, K=K, chunk_rows=C)
            assert ao.plan_json(dd, sm_count=sms) == osch.export_json(osch.plan(dd, sm_count=sms))


def test_validation_agrees(ao):
    cases = [dict(), dict(M=500), dict(chunk_rows=96), dict(K=100), dict(N=500), dict(op="gemm_rs", dir="pull"),
             dict(tile_m=128, tile_n=0), dict(tile_m=64, tile_n=64), dict(world_size=2, M=192, chunk_rows=32),
             dict(M=0), dict(K=0), dict(world_size=9, M=9 * 128), dict(rank=2), dict(n_slices=0),
             dict(comm_ctas=200), dict(intra="grouped", group_m=0), dict(chunk_rows=12),
             dict(op="gemm_ar"), dict(op="gemm_ar", backend="ldst"), dict(op="gemm_ar", backend="ldst", dir="pull"),
             dict(op="gemm_ar", backend="ldst", comm_ctas=4), dict(op="gemm_ar", backend="tma"),
             dict(op="gemm_rs", rs_wire="bf16"), dict(op="gemm_ar", backend="ldst", rs_wire="bf16"),
             dict(rs_wire="bf16"), dict(op="gemm_rs", rs_wire="bf16", rs_reduce="atomic"),
             dict(op="gemm_ar", backend="ldst", rs_wire="bf16", rs_reduce="atomic")]
    for kw in cases:
        dd = osch.default_desc(**kw)
        ref_ok = not osch.validate(dd)
        got_ok = not ao.validate(dd)
        assert ref_ok == got_ok, (kw, osch.validate(dd), ao.validate(dd))


def test_plan_hash_rank_independent(ao):
    hs = set()
    for r in range(4):
        p = ao.Plan(None, osch.default_desc(world_size=4, rank=r, M=1024, chunk_rows=128))
        hs.add(p.hash())
    assert len(hs) == 1
    p2 = ao.Plan(None, osch.default_desc(world_size=4, rank=0, M=1024, chunk_rows=64))
    assert p2.hash() not in hs


def test_workspace_bytes(ao):
    assert ao.workspace_bytes(osch.default_desc(M=512, K=512)) == 2 * 512 * 512 * 2
    assert ao.workspace_bytes(osch.default_desc(op="gemm_rs", M=512, N=384)) == 2 * 512 * 384 * 4
    # AR: (slots) + the owner's reduced rows [S, N] bf16, per parity
    ar = osch.default_desc(op="gemm_ar", backend="ldst", M=512, N=384)
    assert ao.workspace_bytes(ar) == 2 * (512 * 384 * 4 + 256 * 384 * 2)
    assert ao.workspace_bytes(dict(ar, rs_reduce="atomic")) == 2 * (512 * 384 * 4 + 256 * 384 * 2)


def test_library_exports_every_declared_symbol(ao):
    hdr = open(os.path.join(ROOT, "include", "autooverlap.h")).read()
    declared = set(re.findall(r"^\s*(?:const char\*|ao_status)\s+(ao_\w+)\s*\(", hdr, flags=re.M))
    assert len(declared) >= 20
    lib = ao.lib()
    for name in declared:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", ao.N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ao_\w+)", nm))
    assert declared <= exported, declared - exported
    assert set(ao.N.EXPORTED) <= exported


def test_host_only_calls_need_no_gpu(ao):
    import torch
    assert ao.plan_json(osch.default_desc())  # works on a GPU-less box
    if not torch.cuda.is_available():
        with pytest.raises(ao.AOError):
            ao.Context(0, 0, 1, 1 << 20)


def test_a2a_host_plan(ao):
    """A2A-GEMM (NEXT-3) host plan: validation rules of the header, the dynamic schedule's
    static part in the canonical JSON, rank-independent hash, workspace = 2 parities of the
    [W*T, K] bf16 receive buffer."""
    base = dict(op="a2a_gemm", world_size=8, M=1024, N=28672, K=4096, topk=2, chunk_rows=64, backend="ldst",
                tile_m=256, tile_n=256, n_cta=148)
    assert ao.validate(dict(base, rank=0)) == []
    for bad, why in ((dict(topk=9), "topk"), (dict(topk=0), "topk"), (dict(backend="ce"), "backend"),
                     (dict(dir="pull"), "dir"), (dict(chunk_rows=20), "chunk_rows"), (dict(comm_ctas=2), "comm_ctas")):
        v = ao.validate(dict(base, rank=0, **bad))
        assert any(why in x for x in v), (bad, v)
    assert any("topk" in x for x in ao.validate(dict(op="ag_gemm", world_size=2, rank=0, M=512, N=512, K=512,
                                                     chunk_rows=64, topk=2)))
    j = json.loads(ao.plan_json(dict(base, rank=3)))
    assert j["op"] == "a2a_gemm" and j["dynamic"] == 1 and j["topk"] == 2
    assert j["max_chunks_per_source"] == 1024 // 64 and j["tile"] == [256, 256, 2] and j["n_cta"] == 74
    hashes = {ao.Plan(None, dict(base, rank=r)).hash() for r in range(8)}
    assert len(hashes) == 1
    assert ao.workspace_bytes(dict(base, rank=0)) == 2 * 8 * 1024 * 4096 * 2


def test_sp_attn_host_plan(ao):
    """SP attention (NEXT-4) host plan: validation, canonical JSON, rank-independent hash,
    workspace = 2 parities x (gathered K + gathered V)."""
    base = dict(op="sp_attn", world_size=8, M=4096, N=32, K=128, chunk_rows=4096, backend="ce", n_cta=148)
    assert ao.validate(dict(base, rank=0)) == []
    for bad, why in ((dict(K=64), "head dim"), (dict(M=100), "S_loc"), (dict(chunk_rows=192), "chunk_rows"),
                     (dict(backend="tma"), "backend"), (dict(dir="pull"), "dir"), (dict(N=0), "heads")):
        v = ao.validate(dict(base, rank=0, **bad))
        assert any(why in x for x in v), (bad, v)
    j = json.loads(ao.plan_json(dict(base, rank=2)))
    assert j["op"] == "sp_attn" and j["chunks_per_source"] == 32 * 4096 // 4096 and j["items"] == 32 * 32
    assert len({ao.Plan(None, dict(base, rank=r)).hash() for r in range(8)}) == 1
    assert ao.workspace_bytes(dict(base, rank=0)) == 2 * 2 * 8 * 32 * 4096 * 128 * 2


# ---- stream-K tail (Q28) ------------------------------------------------------
def _sk_descs():
    out = []
    # per-GPU TP shapes (BASELINE configs[1]) at W = 8 / 4 / 2, tiles of 1 and 2 CTAs, and
    # small shapes where the tail is a handful of tiles; K ragged (not a multiple of 64)
    for W, N in ((8, 1792), (4, 3584), (2, 7168)):
        for tile in ((256, 256), (256, 224), (128, 256), (0, 0)):
            for sk in (1, -1):
                out.append(dict(op="ag_gemm", world_size=W, M=8192, N=N, K=4096, chunk_rows=1024 // W * 2,
                                intra="grouped", group_m=4, tile_m=tile[0], tile_n=tile[1], stream_k=sk))
    for n_cta in (3, 5, 7, 11):
        for K in (136, 512, 1000 // 8 * 8):
            out.append(dict(op="ag_gemm", world_size=2, M=1024, N=392, K=K, chunk_rows=128, tile_m=128,
                            tile_n=128, n_cta=n_cta, stream_k=1))
    return out


@pytest.mark.parametrize("d", _sk_descs())
def test_stream_k_json_byte_exact(ao, d):
    for r in range(d["world_size"]):
        dd = osch.default_desc(**dict(d, rank=r))
        assert ao.plan_json(dd, sm_count=148) == osch.export_json(osch.plan(dd, sm_count=148)), (d, r)


def test_stream_k_partition_invariants():
    """Independent of the oracle's formulas: every (position, k-block) unit of the tiles is
    computed by exactly one piece; each worker's pieces are contiguous in unit order; a
    split tile has exactly one head (from k-block 0, stores the tile) and one tail (to the
    last k-block, stores a partial) on consecutive workers; every worker's stream-K work
    differs from the mean by less than one k-block."""
    for T, n, nkb in ((224, 74, 64), (448, 74, 64), (13, 5, 7), (29, 4, 3), (150, 74, 1)):
        dp = (T // n - 1) * n
        cover = {}
        sk_units = []
        for c in range(n):
            pcs = osch.worker_pieces(T, n, dp, nkb, c)
            units = []
            for k, kb0, kb1, role in pcs:
                assert 0 <= kb0 < kb1 <= nkb
                for kb in range(kb0, kb1):
                    assert (k, kb) not in cover
                    cover[(k, kb)] = (c, role)
                    if k >= dp:
                        units.append(k * nkb + kb)
            assert units == list(range(units[0], units[0] + len(units))) if units else True
            sk_units.append(len(units))
        assert set(cover) == {(k, kb) for k in range(T) for kb in range(nkb)}
        mean = (T - dp) * nkb / n
        assert all(abs(u - mean) < 1 for u in sk_units)
        for k in range(dp, T):
            owners = {cover[(k, kb)] for kb in range(nkb)}
            if len(owners) > 1:
                (c_head, r_head), (c_tail, r_tail) = sorted(owners)
                assert (r_head, r_tail) == (2, 1) and c_tail == c_head + 1
                assert cover[(k, 0)][1] == 2 and cover[(k, nkb - 1)][1] == 1
            else:
                assert owners.pop()[1] == 0


def test_stream_k_auto_rule():
    # S:334 utilization at the per-GPU TP=8 AG shape: 224 pair tiles on 74 workers = 0.757 -> on;
    # TP=2 (896 tiles, 0.93) -> off; an exact multiple -> off
    assert osch.stream_k_dp(osch.default_desc(K=4096, stream_k=-1), 224, 74, 2) == 148
    assert osch.stream_k_dp(osch.default_desc(K=4096, stream_k=-1), 896, 74, 2) == 896
    assert osch.stream_k_dp(osch.default_desc(K=4096, stream_k=1), 222, 74, 2) == 222
    assert osch.stream_k_dp(osch.default_desc(K=4096, stream_k=0), 224, 74, 2) == 224
    assert osch.stream_k_dp(osch.default_desc(op="gemm_rs", K=4096, stream_k=1), 224, 74, 2) == 224


def test_stream_k_validation_agrees(ao):
    for kw in (dict(stream_k=1), dict(stream_k=-1), dict(stream_k=2), dict(stream_k=1, op="gemm_rs"),
               dict(stream_k=1, backend="tma"), dict(stream_k=-1, op="gemm_rs")):
        dd = osch.default_desc(**kw)
        assert (not osch.validate(dd)) == (not ao.validate(dd)), kw


def test_rs_bf16_wire_json_and_flag(ao):
    """The non-conforming bf16 RS wire (Q14): accepted for GEMM-RS with the atomic
    reduction, exported in the canonical JSON, part of the plan hash, flagged in
    ao_last_error while the call returns AO_OK."""
    d = osch.default_desc(op="gemm_rs", world_size=4, M=1024, N=392, K=136, chunk_rows=128, rs_reduce="atomic",
                          rs_wire="bf16")
    got = ao.plan_json(d)
    assert got == osch.export_json(osch.plan(d))
    assert json.loads(got)["rs_wire"] == "bf16"
    assert "non-conforming" in ao.N.lib().ao_last_error().decode()
    h32 = ao.Plan(None, dict(d, rs_wire="fp32")).hash()
    assert ao.Plan(None, d).hash() != h32


def test_hp_attn_host_plan(ao):
    """HP attention (NEXT-4) host plan: validation (heads divisible by W, S_loc % 256, chunk
    rows dividing a source block of H/W heads), JSON, rank-independent hash, workspace = 2
    parities of gathered Q, K, V and the output return buffer."""
    base = dict(op="hp_attn", world_size=8, M=4096, N=32, K=128, chunk_rows=2048, backend="ce", n_cta=148)
    assert ao.validate(dict(base, rank=0)) == []
    for bad in (dict(N=30), dict(M=384), dict(K=64), dict(chunk_rows=96), dict(chunk_rows=4096 * 4 + 128),
                dict(backend="tma"), dict(causal=2)):
        assert ao.validate(dict(base, rank=0, **bad)), bad
    j = json.loads(ao.plan_json(dict(base, rank=3)))
    assert j["op"] == "hp_attn" and j["heads_per_rank"] == 4 and j["chunks_per_source"] == 4 * 4096 // 2048
    assert j["items"] == 8 * 4 * (4096 // 256)
    hs = {ao.Plan(None, dict(base, rank=r)).hash() for r in range(8)}
    assert len(hs) == 1
    assert ao.workspace_bytes(dict(base, rank=0)) == 2 * 4 * 32 * 4096 * 128 * 2
