"""Auto-tuner (§5.3): candidate enumeration and pruning on CPU; a small measured
tune on the GPU."""
import pytest

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
    kept, pruned = tune.prune(descs, 18)
    assert kept and pruned is not None
    for d in kept:  # everything kept is a valid plan for the oracle planner too
        assert not osch.validate(osch.default_desc(**{k: v for k, v in d.items()}), 18)
    # the copy engine never gets chunks below the minimum efficient transfer size
    for d in kept:
        if d["backend"] == "ce":
            assert d["chunk_rows"] * d["K"] * 2 >= tune.CE_MIN_CHUNK_BYTES
    reasons = {r.split(":")[0] for _, r in pruned}
    assert reasons <= {"invalid", "inefficient"}


def test_rs_space_has_both_orders(tune):
    descs = tune.candidate_space("gemm_rs", 4, 4096, 4096, 1024)
    assert {d["chunk_order"] for d in descs} == {"shard_major", "chunk_major"}
    assert {d["backend"] for d in descs} == {"ce"}


@pytest.mark.gpu
def test_small_measured_tune(tune):
    space = tune.candidate_space("ag_gemm", 2, 1024, 512, 512, chunks=[128, 256], intras=[("row", 1)],
                                 tiles=[(128, 128)])
    rows, pruned = tune.tune_loopback("ag_gemm", 2, 1024, 512, 512, space=space, budget_s=60)
    assert rows and all(r["ms"] > 0 for r in rows)
    assert rows == sorted(rows, key=lambda r: r["ms"])
