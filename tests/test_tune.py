"""Auto-tuner (§5.3): candidate enumeration (chunk x backend x dir x
intra x tile x RS order x comm_ctas x n_slices), pruning (validation, CE minimum size,
E4-seeded transfer estimates), the tuned table consumed by backend "auto" plans -- on CPU;
a small measured tune on the GPU whose winner is checked against the fp64 oracle."""
import json

import pytest

from oracle import numeric as on
from oracle import schedule as osch


@pytest.fixture(scope="module")
def tune():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.tune as t
    return t


def test_space_and_pruning(tune):
    descs = tune.candidate_space("ag_gemm", 8, 8192, 1792, 4096)
    assert len(descs) == len({tuple(sorted(d.items())) for d in descs})  # no duplicates
    # in-kernel backends carry the comm_ctas and n_slices axes, the copy engine does not
    assert {d["comm_ctas"] for d in descs if d["backend"] == "tma"} == {0, 8, 16}
    assert {d["n_slices"] for d in descs if d["backend"] == "ldst"} == {1, 2, 4}
    assert {(d["comm_ctas"], d["n_slices"]) for d in descs if d["backend"] == "ce"} == {(0, 1)}
    kept, pruned = tune.prune(descs, 18)
    assert kept and pruned is not None
    for d in kept:  # everything kept is a valid plan for the oracle planner too
        assert not osch.validate(osch.default_desc(**{k: v for k, v in d.items()}), 18)
    for d in kept:  # the copy engine never gets chunks below the minimum efficient transfer size
        if d["backend"] == "ce":
            assert d["chunk_rows"] * d["K"] * 2 >= tune.CE_MIN_CHUNK_BYTES
    reasons = {r.split(":")[0] for _, r in pruned}
    assert reasons <= {"invalid", "inefficient"}


def test_rs_space_has_both_orders(tune):
    descs = tune.candidate_space("gemm_rs", 4, 4096, 4096, 1024)
    assert {d["chunk_order"] for d in descs} == {"shard_major", "chunk_major"}
    assert {d["backend"] for d in descs} == {"ce"}


def _write_e4(path, ce, tma, ldst):
    """Synthetic E4 curves: GB/s flat in message size for each (backend, units)."""
    with open(path, "w") as f:
        for m in (1 << 16, 1 << 20, 1 << 24):
            f.write(json.dumps(dict(mode="loopback", backend="ce", streams=1, bytes=m, ms=1.0, GBps=ce)) + "\n")
            for n in (1, 8, 16, 74):
                for b, g in (("tma", tma), ("ldst", ldst)):
                    f.write(json.dumps(dict(mode="loopback", backend=b, ctas=n, bytes=m, ms=1.0, GBps=g * n / 16)) + "\n")


def test_e4_interpolation_and_seeded_pruning(tune, tmp_path):
    p = str(tmp_path / "e4.jsonl")
    _write_e4(p, ce=400.0, tma=300.0, ldst=100.0)
    e4 = tune.load_e4(p)
    assert tune.e4_bandwidth(e4, "ce", 1, 1 << 20) == pytest.approx(400.0)
    assert tune.e4_bandwidth(e4, "tma", 16, 1 << 22) == pytest.approx(300.0)
    assert tune.e4_bandwidth(e4, "tma", 12, 1 << 20) == pytest.approx(300.0 * 8 / 16)  # nearest unit count below
    assert tune.e4_bandwidth(e4, "ce", 1, 1 << 15) == pytest.approx(400.0 / 2)  # latency-bound below the curve
    descs = tune.candidate_space("ag_gemm", 8, 8192, 1792, 4096, chunks=[512], intras=[("row", 1)], tiles=[(0, 0)],
                                 dirs=["push"])
    kept, pruned = tune.prune(descs, 148, e4=e4)
    # LDST (100 GB/s at 16 CTAs) and TMA with 8 comm CTAs are > 1.5x slower than the copy engine
    assert all(d["backend"] != "ldst" for d in kept)
    assert any(r.startswith("e4:") for _, r in pruned)
    est = {d["backend"]: tune.e4_transfer_ms(d, e4, 148) for d in kept}
    assert est["ce"] == pytest.approx(7 * 1024 * 4096 * 2 / 400e9 * 1e3)


def test_tuned_table_and_auto_plans(tune, tmp_path):
    p = str(tmp_path / "table.json")
    desc = dict(op="ag_gemm", world_size=4, M=4096, N=1024, K=512, chunk_rows=256, backend="tma", dir="pull",
                chunk_order="chunk_major", intra="grouped", group_m=4, tile_m=128, tile_n=256, n_slices=2, comm_ctas=0)
    tune.save_table([{"desc": desc, "ms": 1.0, "tflops": 5.0}], p)
    got = tune.resolve(dict(op="ag_gemm", world_size=4, M=4096, N=1024, K=512, backend="auto", rank=3), p)
    assert got["rank"] == 3 and got["backend"] == "tma" and got["chunk_rows"] == 256 and got["dir"] == "pull"
    assert not osch.validate(osch.default_desc(**got))
    # an untuned shape falls back to the planner defaults
    other = tune.resolve(dict(op="gemm_rs", world_size=2, M=512, N=512, K=256, backend="auto"), p)
    assert other["backend"] == "ce" and "chunk_rows" not in other
    assert tune.resolve(dict(desc, backend="ce"), p)["backend"] == "ce"  # explicit backends pass through


@pytest.mark.gpu
def test_small_measured_tune_winner_matches_oracle(tune, tmp_path):
    import torch

    from synthetic import inputs as si
    W, M, N, K = 2, 1024, 512, 512
    space = tune.candidate_space("ag_gemm", W, M, N, K, chunks=[128, 256], intras=[("row", 1)], tiles=[(128, 128)],
                                 comm_ctas=[0, 8], slices=[1, 2])
    rows, pruned = tune.tune_loopback("ag_gemm", W, M, N, K, space=space, budget_s=60)
    assert rows and all(r["ms"] > 0 for r in rows)
    assert rows == sorted(rows, key=lambda r: r["ms"])
    table = str(tmp_path / "t.json")
    tune.save_table(rows, table)
    import paper_2601_20595_b200.api as api
    descs = [tune.resolve(dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, backend="auto", rank=r,
                               timeout_ns=2_000_000_000), table) for r in range(W)]
    if not rows[0]["desc"].get("sched"):
        for d in descs:
            d["n_cta"] = 148 // W - d.get("comm_ctas", 0)
    ctxs = api.loopback_world(0, W, api.workspace_bytes(descs[0]))
    plans = [api.Plan(ctxs[r], descs[r]) for r in range(W)]
    A, B = si.ag_inputs(W, M, K, N, salt=91)
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    api.ag_gemm_group(plans, [a.cuda() for a in A], [b.cuda() for b in B], Cs)
    torch.cuda.synchronize()
    A64 = [si.to_f64(a) for a in A]
    for r in range(W):
        ok, e, f = on.check_tolerance(Cs[r].float().cpu().numpy(), on.ag_gemm(A64, si.to_f64(B[r])))
        assert ok, (rows[0]["desc"], e, f)
    for c in ctxs:
        c.close()


def test_stream_k_axis(tune):
    descs = tune.candidate_space("ag_gemm", 8, 8192, 1792, 4096, backends=["ce", "tma"], stream_ks=[0, -1])
    assert {d.get("stream_k", 0) for d in descs if d["backend"] == "ce"} == {0, -1}
    assert {d.get("stream_k", 0) for d in descs if d["backend"] == "tma"} == {0}
    assert all("stream_k" not in d for d in tune.candidate_space("gemm_rs", 4, 4096, 4096, 1024, stream_ks=[0, 1]))
