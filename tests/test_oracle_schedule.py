"""Pins of the brute-force schedule oracle (oracle/schedule.py).

Pinned against: worked examples printed in SPEC.md / PAPER.md (tests/golden/
spec_examples.json), the hand-derived tiny example of SURVEY.md §8(c)
(tests/golden/tiny_worked_example.json), closed forms (wave quantization), and
invariants (permutation, group monotonicity, partition, safety under randomized
arrival, and a 100 % wait-mutation kill rate).
"""
import itertools
import json
import os
import random

import pytest

from oracle import schedule as osch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


SPEC = _gold("spec_examples.json")
TINY = _gold("tiny_worked_example.json")


def _desc(**kw):
    return osch.default_desc(**kw)


def test_pull_rotation_spec_s158():
    ex = SPEC["pull_rotation"]
    W, r = ex["world_size"], ex["rank"]
    p = osch.plan(_desc(world_size=W, rank=r, M=W * 128, dir="pull", chunk_rows=128), sm_count=148)
    peers = []
    for op in p["plans"][r]:
        if op["peer"] not in peers:
            peers.append(op["peer"])
    assert peers == ex["peers"]
    assert all(op["direction"] == "pull" for op in p["plans"][r])


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("direction", ["push", "pull"])
def test_rotation_is_contention_free_s160(W, direction):
    p = osch.plan(_desc(world_size=W, rank=0, M=W * 128, dir=direction, chunk_rows=128))
    n_ops = len(p["plans"][0])
    assert n_ops == W - 1
    for i in range(n_ops):
        peers = [p["plans"][q][i]["peer"] for q in range(W)]
        assert sorted(peers) == list(range(W))  # each peer exactly once at position i
        assert all(peers[q] != q for q in range(W))


def test_ag_dependency_example_s399():
    ex = SPEC["ag_dep_example"]
    p = osch.plan(_desc(world_size=2, rank=0, M=ex["M"], N=256, K=64, chunk_rows=128,
                        tile_m=ex["block_m"], tile_n=128))
    n_nb = 2
    chunks = {c[0]: c for c in p["chunks"]}
    dependent = sorted({t // n_nb for (t, glo, ghi, _) in p["deps"]
                        if any(chunks[g][3] != 0 for g in range(glo, ghi + 1))})
    assert dependent == ex["dependent_pid_m"]


def test_utilization_closed_form_s337():
    for tiles, sms, val in SPEC["utilization"]["cases"]:
        assert abs(osch.sm_utilization(tiles, sms) - val) <= SPEC["utilization"]["tol"]
    w = SPEC["waves"]
    import math
    assert math.ceil(w["tiles"] / w["sms"]) == w["waves"]
    assert w["tiles"] - (w["waves"] - 1) * w["sms"] == w["last"]


def test_grouped_prefix_s421():
    # W=1: no remote chunks, one group; 4x4 tiles of 128x128
    p = osch.plan(_desc(world_size=1, rank=0, M=512, N=512, K=64, chunk_rows=512,
                        tile_m=128, tile_n=128, intra="grouped", group_m=2))
    coords = [[t // 4, t % 4] for t in p["order"]]
    assert coords[:4] == SPEC["grouped2_prefix"]["prefix"]
    assert sorted(p["order"]) == list(range(16))


def test_min_wait_example_s409():
    # One CTA; a chunk consumed at positions {5, 9, 12}: single wait before position 5.
    # Build it: W=2 rank 1, n_cta=1, the chunk's consumers are found from the order.
    p = osch.plan(_desc(world_size=2, rank=1, M=512, N=512, chunk_rows=64, tile_m=128, tile_n=128, n_cta=1))
    (cta, waits), = p["waits"]
    first = {}
    for k, t in enumerate(p["order"]):
        glo, ghi = p["deps"][t][1], p["deps"][t][2]
        for g in range(glo, ghi + 1):
            if p["chunks"][g][3] != 1:
                first.setdefault(g, k)
    assert waits == sorted([[k, g] for g, k in first.items()])
    assert len(waits) == len(first)  # exactly one wait per consumed remote chunk
    ex = SPEC["min_wait"]
    consumers = ex["positions"]
    assert min(consumers) == ex["wait_before"]


def test_tiny_worked_example_ag():
    d = TINY["desc"]
    base = dict(op=d["op"], world_size=d["world_size"], M=d["M"], N=d["N"], K=d["K"],
                chunk_rows=d["chunk_rows"], tile_m=d["tile_m"], tile_n=d["tile_n"])
    for r, key in ((0, "rank0"), (1, "rank1")):
        p = osch.plan(_desc(rank=r, **base))
        exp = TINY[key]
        assert [c[4] for c in p["chunks"]] == exp["pos"]
        grp_mb = [p["deps"][mb * 4][3] for mb in range(4)]
        assert grp_mb == exp["group_by_mb"]
        assert p["order"] == exp["order"]
    p0 = osch.plan(_desc(rank=0, **base))
    t = 2 * 4  # mb = 2
    assert [p0["deps"][t][1], p0["deps"][t][2]] == TINY["rank0"]["mb2_chunks"]
    pg = osch.plan(_desc(rank=1, intra="grouped", group_m=2, **base))
    assert pg["order"][:8] == TINY["rank1"]["grouped2_group0"]
    ex = TINY["rank1_ncta4"]
    p4 = osch.plan(_desc(rank=1, n_cta=ex["n_cta"], **base))
    for c in range(4):
        assert [p4["order"][k] for k in range(c, 16, 4)] == ex["tiles_of_cta"][c]
        assert p4["waits"][c] == [c, ex["waits_of_cta"][c]]
    assert sum(len(w[1]) for w in p4["waits"]) == ex["waits_per_rank"]


def test_tiny_worked_example_rs():
    ex = TINY["rs_rank0"]
    d = ex["desc"]
    p = osch.plan(_desc(rank=0, **d))
    assert [c[4] for c in p["chunks"]] == ex["pos"]
    assert all(x == ex["tiles_per_chunk"] for x in p["tiles_per_chunk"])
    assert p["order"] == ex["gemm_order"]
    own = [t for t in p["order"] if t // 4 < 2]
    assert sorted(own) == ex["own_tiles"]
    assert p["order"][-len(own):] == own  # own rows last
    for t in own:
        mb = t // 4
        assert [p["deps"][t][1], p["deps"][t][2]] == ex["own_tile_chunks"]["mb%d" % mb]
    p1 = osch.plan(_desc(rank=0, n_cta=1, **d))
    assert p1["waits"] == [[0, ex["ncta1_waits"]]]
    assert p["contrib"] == ex["contrib"]


SWEEP = []
for W in (1, 2, 4, 8):
    for op in ("ag_gemm", "gemm_rs"):
        for C in (64, 128, 256):
            for intra in ("row", "col", "grouped"):
                for order in ("shard_major", "chunk_major"):
                    SWEEP.append(dict(op=op, world_size=W, M=256 * W, N=384, K=128, chunk_rows=C,
                                      intra=intra, group_m=2, chunk_order=order, tile_m=128, tile_n=128, n_cta=5))


@pytest.mark.parametrize("d", SWEEP[::7])
def test_invariants(d):
    W = d["world_size"]
    for r in range(W):
        p = osch.plan(_desc(rank=r, **d))
        T = len(p["deps"])
        assert sorted(p["order"]) == list(range(T))  # permutation
        groups = [p["deps"][t][3] for t in p["order"]]
        assert groups == sorted(groups)  # group monotonicity
        # partition (Q4): each row in exactly one chunk
        covered = []
        for g, row0, rows, src, pos in p["chunks"]:
            covered.extend(range(row0, row0 + rows))
        assert covered == list(range(d["M"]))
        # each tile's chunks: BM/C chunks of one source when C < BM, else exactly one
        bm = p["tile"][0]
        for t, glo, ghi, grp in p["deps"]:
            n = ghi - glo + 1
            assert n == max(1, bm // d["chunk_rows"])
            assert len({p["chunks"][g][3] for g in range(glo, ghi + 1)}) == 1
        # arrival positions are injective over remote chunks
        pos = [c[4] for c in p["chunks"] if (d["op"] == "gemm_rs" or c[3] != r)]
        assert len(pos) == len(set(pos))
        if d["op"] == "gemm_rs" and d["chunk_order"] == "shard_major":
            own = {t for t, glo, ghi, _ in p["deps"] if p["chunks"][glo][3] == r}
            assert set(p["order"][len(p["order"]) - len(own):]) == own  # own rows last


def _simulate(p, rank, drop=None, seed=0):
    """Randomized-timing execution of one rank's plan: remote chunks (AG) or
    the other sources' contributions to own chunks (RS) arrive at random times; each CTA
    runs its positions in order, blocking at its waits.  Returns the reads of a chunk
    before its arrival."""
    rnd = random.Random(seed)
    is_ag = p["op"] == "ag_gemm"
    arrival = {}
    for g, row0, rows, src, pos in p["chunks"]:
        if is_ag:
            arrival[g] = 0.0 if src == rank else rnd.uniform(0, 100) + pos
        else:
            arrival[g] = rnd.uniform(0, 150) + pos if src == rank else 0.0
    violations = []
    n_cta = p["n_cta"]
    order = p["order"]
    for cta, waits in p["waits"]:
        ws = {}
        for k, g in waits:
            if (k, g) == drop:
                continue
            ws.setdefault(k, []).append(g)
        now = 0.0
        for k in range(cta, len(order), n_cta):
            for g in ws.get(k, []):
                now = max(now, arrival[g])
            t = order[k]
            glo, ghi = p["deps"][t][1], p["deps"][t][2]
            if is_ag:
                need = [g for g in range(glo, ghi + 1) if p["chunks"][g][3] != rank]
            else:
                need = [g for g in range(glo, ghi + 1) if p["chunks"][g][3] == rank]
            for g in need:
                if arrival[g] > now:
                    violations.append((k, t, g))
            now += rnd.uniform(0.5, 2.0)
    return violations


@pytest.mark.parametrize("op", ["ag_gemm", "gemm_rs"])
@pytest.mark.parametrize("n_cta", [1, 3, 4])
def test_safety_and_mutation_kill(op, n_cta):
    base = dict(op=op, world_size=2, M=512, N=512, K=256, chunk_rows=64, tile_m=128, tile_n=128, n_cta=n_cta)
    for r in range(2):
        p = osch.plan(_desc(rank=r, **base))
        for seed in range(100):
            assert _simulate(p, r, seed=seed) == []
        all_waits = [(k, g) for _, ws in p["waits"] for k, g in ws]
        assert all_waits
        for w in all_waits:  # every single wait is necessary (100 % kill rate)
            assert any(_simulate(p, r, drop=w, seed=s) for s in range(100)), w


def test_validation_rejects():
    bad = [
        dict(M=500),                       # M % W
        dict(chunk_rows=96),               # S % C (S=256)
        dict(K=100),                       # K % 8
        dict(N=500),                       # N % 8
        dict(op="gemm_rs", dir="pull"),    # pull with RS
        dict(tile_m=128, tile_n=0),
        dict(tile_m=64, tile_n=64),        # unsupported tile
        dict(world_size=2, M=2 * 96, chunk_rows=32),  # S=96 not divisible by any BM
    ]
    for kw in bad:
        assert osch.validate(_desc(**kw)), kw
    assert osch.validate(_desc()) == []
    assert osch.validate(_desc(M=0)) == []  # empty problem is valid (no tiles)


def test_tile_eff_is_the_measurement_record():
    """TILE_EFF is typed from the committed measurement (scripts/measure_tile_eff.py ->
    profiles/r02_tile_eff.json), not from the planner's own formula."""
    rec = json.load(open(os.path.join(ROOT, "profiles", "r02_tile_eff.json")))["eff_pct"]
    assert {f"{a}x{b}": v for (a, b, _), v in osch.TILE_EFF.items() if v} == {k: v for k, v in rec.items() if k in
                                                                               {f"{a}x{b}" for (a, b, _), w in osch.TILE_EFF.items() if w}}
    assert all(f"{a}x{b}" in rec for (a, b, _), v in osch.TILE_EFF.items() if v)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "pick_tile.json")))
    assert gold["eff_pct"] == rec


def test_tile_heuristic_golden_picks():
    """Hand-derived picks (tests/golden/pick_tile.json, each with its worked costs): wave
    quantization weighted by the measured efficiency.  A changed efficiency,
    candidate list or cost rule flips at least one of them."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "pick_tile.json")))
    for case in gold["cases"]:
        d = osch.default_desc(**case["desc"])
        assert list(osch.pick_tile(d, case["sm_count"])) == case["pick"], case["name"]


def test_tile_heuristic_is_wave_quantization_when_efficiencies_tie():
    """With equal efficiencies the rule reduces to S:334: least waves x per-SM tile area,
    i.e. the utilization argmax among shapes of equal area."""
    saved = dict(osch.TILE_EFF)
    try:
        for k in osch.TILE_EFF:
            osch.TILE_EFF[k] = 50
        # AG@8: 256x224 (4 waves) vs 256x256 (4 waves): equal waves -> smaller area wins
        d = osch.default_desc(op="ag_gemm", world_size=8, M=8192, N=1792, K=4096, chunk_rows=128)
        picked = osch.pick_tile(d, 148)
        def waves_of(c):
            tiles = (8192 // c[0]) * ((1792 + c[1] - 1) // c[1])
            n = 148 // c[2]
            return (tiles + n - 1) // n
        waves = {c: waves_of(c) for c in osch.tile_candidates(d)}
        best = min(waves[c] * c[0] * c[1] // c[2] for c in waves)
        assert waves[picked] * picked[0] * picked[1] // picked[2] == best
        # S:334 numbers: 1024 tiles on 132 SMs -> 8 waves (utilization 0.9697)
        assert osch.sm_utilization(1024, 132) == 1024 / 1056
    finally:
        osch.TILE_EFF.clear()
        osch.TILE_EFF.update(saved)


def test_export_is_canonical_and_deterministic():
    p = osch.plan(_desc(rank=1))
    s = osch.export_json(p)
    assert " " not in s and "\n" not in s
    assert s == osch.export_json(osch.plan(_desc(rank=1)))
    assert json.loads(s) == p


@pytest.mark.parametrize("W", [2, 3, 4, 8])
@pytest.mark.parametrize("C", [64, 128])
def test_gemm_ar_gather_plan(W, C):
    """GEMM-AR (NEXT-1, Fig.4d): the RS part equals gemm_rs's plan; the gather part
    pulls every other owner's reduced chunk exactly once; at every gather step each owner
    serves exactly one puller (contention-free rotation); reduce-side tables equal RS."""
    base = dict(world_size=W, M=256 * W, N=384, K=128, chunk_rows=C, tile_m=128, tile_n=128, n_cta=5,
                backend="ldst", intra="grouped", group_m=2)
    S, n_c = 256, 256 // C
    steps = {}
    for r in range(W):
        ar = osch.plan(_desc(op="gemm_ar", rank=r, **base))
        rs = osch.plan(_desc(op="gemm_rs", rank=r, **base))
        for key in ("chunks", "deps", "order", "waits", "contrib", "tiles_per_chunk"):
            assert ar[key] == rs[key], key
        for q in range(W):
            n_rs = len(rs["plans"][q])
            assert ar["plans"][q][:n_rs] == rs["plans"][q]
            pulls = ar["plans"][q][n_rs:]
            assert all(op["direction"] == "pull" and op["tensor"] == "C" and not op["accumulate"] for op in pulls)
            got = sorted(op["src_chunk"][0] for op in pulls)
            want = sorted(o * S + j * C for o in range(W) if o != q for j in range(n_c))
            assert got == want
            assert all(op["peer"] == op["src_chunk"][0] // S for op in pulls)
            if r == 0:
                for i, op in enumerate(pulls):
                    steps.setdefault(i, []).append(op["peer"])
        assert ar["owner_regions"][r]["C"] == [[r * S, S]]
    for i, owners in steps.items():
        assert sorted(owners) == list(range(W)) or len(set(owners)) == W, (i, owners)
