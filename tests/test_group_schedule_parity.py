"""Launch-level (time-sliced / space-sliced) group schedule of the C++ runtime, exported
through the C ABI (ao_group_schedule_export, host-only), vs the oracle's enumeration
(oracle.schedule.group_schedule): byte-identical canonical JSON, same accept / refuse
decisions.  Plus properties the enumeration must satisfy on its own (every rank's tile
list appears exactly once in plan order; no RS own tile precedes a contribution it waits
on; the waits are exactly the first uses).  No GPU needed."""
import itertools
import json

import pytest

from oracle import schedule as osch


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _export(ao, descs, sms):
    plans = [ao.Plan(None, d, sms) for d in descs]
    try:
        return ao.group_schedule_json(plans, sms)
    except ao.AOError as e:
        assert e.status == "AO_ERR_INVALID_ARG", e
        return None
    finally:
        for p in plans:
            p.close()


def _cases():
    out = []
    for W in (2, 3, 4, 8):
        for op in ("ag_gemm", "gemm_rs", "gemm_ar"):
            for S, C in ((256, 64), (256, 128), (512, 256)):
                for tile in ((128, 128), (256, 128), (128, 256)):
                    if S % tile[0]:
                        continue
                    for n_cta in (5, 16, 0):
                        for intra, gm in (("row", 1), ("grouped", 2)):
                            for order in ("shard_major", "chunk_major"):
                                out.append(dict(op=op, world_size=W, M=S * W, N=384, K=128, chunk_rows=C,
                                                tile_m=tile[0], tile_n=tile[1], n_cta=n_cta, intra=intra,
                                                group_m=gm, chunk_order=order,
                                                backend="ldst" if op == "gemm_ar" else "ce"))
    return out


CASES = _cases()


@pytest.mark.parametrize("i", range(0, len(CASES), 2))
def test_group_schedule_byte_exact(ao, i):
    d = CASES[i]
    W = d["world_size"]
    # group order: identity, and a permutation (the list follows ranks, not call order)
    for perm in (list(range(W)), list(range(W))[::-1]):
        descs = [osch.default_desc(**dict(d, rank=r)) for r in perm]
        for sms in (148, 40):
            ref = osch.group_schedule(descs, sms)
            got = _export(ao, descs, sms)
            if ref is None:
                assert got is None, (d, perm, sms)
            else:
                assert got == osch.export_json(ref), (d, perm, sms)


@pytest.mark.parametrize("op,N,K,C,gm", [("ag_gemm", 1792, 4096, 1024, 4), ("gemm_rs", 4096, 1792, 1024, 4),
                                         ("ag_gemm", 1792, 4096, 128, 4), ("gemm_rs", 4096, 1792, 256, 4)])
def test_group_schedule_bench_config(ao, op, N, K, C, gm):
    """The bench's loopback TP=8 configuration (Llama-3-8B FFN, time-sliced over 148 SMs)."""
    descs = [osch.default_desc(op=op, world_size=8, rank=r, M=8192, N=N, K=K, chunk_rows=C, tile_m=256,
                               tile_n=256, n_cta=148, intra="grouped", group_m=gm, rs_reduce="atomic")
             for r in range(8)]
    ref = osch.group_schedule(descs, 148)
    assert ref["mode"] == "time_sliced"
    assert _export(ao, descs, 148) == osch.export_json(ref)


def _properties(descs, s):
    plans = [osch.plan(d) for d in descs]
    W = descs[0]["world_size"]
    # every rank's positions appear exactly once (AG: in plan order; RS: in plan order
    # within each owner's phase)
    seen = {d["rank"]: [] for d in descs}
    seq = []
    for r, k0, k1, o in s["segments"]:
        assert o == len(seq)
        for k in range(k0, k1):
            seen[r].append(k)
            seq.append((r, k))
    for d, p in zip(descs, plans):
        if d["op"] == "ag_gemm":
            assert seen[d["rank"]] == list(range(len(p["order"]))), d["rank"]
        else:
            assert sorted(seen[d["rank"]]) == list(range(len(p["order"]))), d["rank"]
    return plans, seq


def test_group_schedule_properties():
    for op, order in itertools.product(("ag_gemm", "gemm_rs"), ("shard_major", "chunk_major")):
        W, S, C = 4, 256, 64
        descs = [osch.default_desc(op=op, world_size=W, rank=r, M=S * W, N=384, K=128, chunk_rows=C, tile_m=128,
                                   tile_n=128, n_cta=16, chunk_order=order) for r in range(W)]
        s = osch.group_schedule(descs, 40)
        assert s["mode"] == "time_sliced"
        plans, seq = _properties(descs, s)
        by_rank = {d["rank"]: p for d, p in zip(descs, plans)}
        n_nb = 3
        if op == "gemm_rs":
            # an own tile (rows of rank r) comes after every other source's tiles of those rows
            for i, (r, k) in enumerate(seq):
                mb = by_rank[r]["order"][k] // n_nb
                if (mb * 128) // S != r:
                    continue
                for j in range(i + 1, len(seq)):
                    q, kk = seq[j]
                    if q != r:
                        assert (by_rank[q]["order"][kk] // n_nb * 128) // S != r, (i, j)
        # waits: exactly the first use per (worker, rank, chunk), in walk order
        nw = s["n_workers"]
        for w, lst in s["waits"]:
            assert [x[0] for x in lst] == sorted(x[0] for x in lst)
            assert all(x[0] % nw == w for x in lst)
            assert len({(x[1], x[2]) for x in lst}) == len(lst)


def test_group_schedule_space_sliced_and_refused():
    d = dict(op="ag_gemm", world_size=4, M=1024, N=384, K=128, chunk_rows=64, tile_m=128, tile_n=128)
    descs = [osch.default_desc(**dict(d, rank=r, n_cta=30)) for r in range(4)]
    assert osch.group_schedule(descs, 148) == {"mode": "space_sliced"}
    # pull plans cannot run time-sliced (a pull waits on a peer's stage that may not run)
    descs = [osch.default_desc(**dict(d, rank=r, n_cta=100, dir="pull")) for r in range(4)]
    assert osch.group_schedule(descs, 148) is None
    # a partial group cannot be time-sliced
    descs = [osch.default_desc(**dict(d, rank=r, n_cta=100)) for r in range(2)]
    assert osch.group_schedule(descs, 148) is None
