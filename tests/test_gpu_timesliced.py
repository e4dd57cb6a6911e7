"""GPU parity of TIME-SLICED loopback groups (Q24) vs the fp64 CPU oracle.

A whole-world loopback group whose plans each ask for more CTAs than SMs / W runs all
its CTAs over every rank's tile list in one global order (AG: rank after rank; RS: owner
after owner, the owner's own tiles after the peers' contributions), with per-tile chunk
waits.  Same tolerance as tests/test_gpu_ops.py (north star: 1e-2 per element relative to
max(1, |ref|), Frobenius 2e-3); provenance patterns and gathered copies are bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle import numeric as on
from synthetic import inputs as si

pytestmark = pytest.mark.gpu

SMS = 148


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _dev(ts):
    return [t.cuda() for t in ts]


def _check(gpu, ref, what):
    ok, e, f = on.check_tolerance(gpu.float().cpu().numpy(), ref)
    assert ok, f"{what}: max elem err {e:.3e}, frob {f:.3e}"


def _world(ao, desc, W):
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(desc))
    return ctxs, [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]


def _ag(ao, ctxs, plans, A, B, gather=False):
    W = len(plans)
    M = sum(a.shape[0] for a in A)
    Cs = [torch.empty(M, B[r].shape[0], dtype=torch.bfloat16, device="cuda") for r in range(W)]
    G = [torch.empty(M, A[0].shape[1], dtype=torch.bfloat16, device="cuda") for _ in range(W)] if gather else None
    ao.ag_gemm_group(plans, A, B, Cs, G)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Cs, G


def _rs(ao, ctxs, plans, A, B):
    W = len(plans)
    M, N = A[0].shape[0], B[0].shape[0]
    Cs = [torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.gemm_rs_group(plans, A, B, Cs)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Cs


@pytest.mark.parametrize("backend", ["ce", "tma", "ldst"])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_ag_timesliced_vs_oracle(ao, W, tile, backend):
    M, K, N, C = 256 * W, 512, 520, 64
    A, B = si.ag_inputs(W, M, K, N, salt=41)
    ctxs, plans = _world(ao, dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=C, backend=backend,
                                  n_slices=2, tile_m=tile[0], tile_n=tile[1], n_cta=SMS,
                                  timeout_ns=2_000_000_000), W)
    Cs, G = _ag(ao, ctxs, plans, _dev(A), _dev(B), gather=True)
    A64 = [si.to_f64(a) for a in A]
    full = torch.cat(A, 0)
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag ts W={W} r{r}")
        assert torch.equal(G[r].cpu(), full), "gathered A must be a bit-exact copy"


@pytest.mark.parametrize("backend", ["ce", "tma", "ldst"])
@pytest.mark.parametrize("W", [4, 8])
def test_ag_timesliced_provenance_epochs(ao, W, backend):
    """Row-id / epoch digits decode exactly across back-to-back epochs (both parities),
    with chunks smaller than a tile (multi-chunk waits) and N spanning several tiles."""
    M, K, N = 256 * W, 64, 768
    ctxs, plans = _world(ao, dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=64, backend=backend,
                                  n_slices=3, tile_m=256, tile_n=256, n_cta=SMS, timeout_ns=2_000_000_000), W)
    for it in range(5):
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=it + 1)
        Cs, _ = _ag(ao, ctxs, plans, _dev(A), _dev(B))
        for r in range(W):
            c = Cs[r].float().cpu()
            rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
            assert torch.equal(rid, torch.arange(M, dtype=torch.float32)), (it, r)
            assert torch.all(c[:, 3] == (it + 1) % 32)


@pytest.mark.parametrize("order", ["shard_major", "chunk_major"])
@pytest.mark.parametrize("reduce", ["slots", "atomic"])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_rs_timesliced_vs_oracle(ao, W, tile, reduce, order):
    M, K, N, C = 256 * W, 256, 520, 64
    A, B = si.rs_inputs(W, M, K, N, salt=43)
    ctxs, plans = _world(ao, dict(op="gemm_rs", world_size=W, M=M, N=N, K=K, chunk_rows=C, tile_m=tile[0],
                                  tile_n=tile[1], rs_reduce=reduce, chunk_order=order, n_cta=SMS,
                                  timeout_ns=2_000_000_000), W)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    dA, dB = _dev(A), _dev(B)
    for it in range(2):  # the accumulator is re-armed between calls
        Cs = _rs(ao, ctxs, plans, dA, dB)
        for r in range(W):
            _check(Cs[r], on.gemm_rs(A64, B64, r), f"rs ts W={W} {reduce} {order} it={it} r{r}")


@pytest.mark.parametrize("reduce", ["slots", "atomic"])
def test_rs_timesliced_bitmask_and_determinism(ao, reduce):
    W, M, K, N = 8, 2048, 64, 520
    ctxs, plans = _world(ao, dict(op="gemm_rs", world_size=W, M=M, N=N, K=K, chunk_rows=128, tile_m=256,
                                  tile_n=256, rs_reduce=reduce, n_cta=SMS, timeout_ns=2_000_000_000), W)
    A, B = si.rs_provenance_inputs(W, M, K, N)
    for it in range(3):
        Cs = _rs(ao, ctxs, plans, _dev(A), _dev(B))
        for r in range(W):
            assert torch.all(Cs[r].float().cpu() == 2 ** W - 1), (it, r)
    if reduce == "slots":
        A, B = si.rs_inputs(W, M, K, N, salt=5)
        A, B = _dev(A), _dev(B)
        first = [c.clone() for c in _rs(ao, ctxs, plans, A, B)]
        second = _rs(ao, ctxs, plans, A, B)
        for r in range(W):
            assert torch.equal(first[r], second[r]), "slots RS stays bitwise deterministic when time-sliced"


def test_timesliced_and_space_sliced_mix_on_one_world(ao):
    """Space- and time-sliced launches interleaved on the same ctxs keep epochs, flags and
    the atomic accumulator consistent."""
    W, M, K, N = 4, 1024, 128, 256
    base = dict(world_size=W, M=M, N=N, K=K, chunk_rows=128, tile_m=256, tile_n=256, timeout_ns=2_000_000_000)
    ag_d = dict(base, op="ag_gemm", backend="ce")
    rs_d = dict(base, op="gemm_rs", rs_reduce="atomic")
    ctxs = ao.loopback_world(0, W, max(ao.workspace_bytes(ag_d), ao.workspace_bytes(rs_d)))
    plans = {}
    for name, d in (("ag", ag_d), ("rs", rs_d)):
        for ts, n_cta in (("ts", SMS), ("sp", SMS // W)):
            plans[name + ts] = [ao.Plan(ctxs[r], dict(d, rank=r, n_cta=n_cta)) for r in range(W)]
    Ag, Bg = si.ag_inputs(W, M, K, N, salt=2)
    Ar, Br = si.rs_inputs(W, M, K, N, salt=3)
    A64 = [si.to_f64(a) for a in Ag]
    Ar64, Br64 = [si.to_f64(a) for a in Ar], [si.to_f64(b) for b in Br]
    dAg, dBg, dAr, dBr = _dev(Ag), _dev(Bg), _dev(Ar), _dev(Br)
    for key in ("agts", "rsts", "agsp", "rssp", "rsts", "agts", "rssp", "agsp", "rsts"):
        if key.startswith("ag"):
            Cs, _ = _ag(ao, ctxs, plans[key], dAg, dBg)
            for r in range(W):
                _check(Cs[r], on.ag_gemm(A64, si.to_f64(Bg[r])), f"{key} r{r}")
        else:
            Cs = _rs(ao, ctxs, plans[key], dAr, dBr)
            for r in range(W):
                _check(Cs[r], on.gemm_rs(Ar64, Br64, r), f"{key} r{r}")


@pytest.mark.parametrize("reduce", ["slots", "atomic"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_gemm_ar_timesliced_vs_oracle(ao, W, reduce):
    """GEMM-AR (NEXT-1) time-sliced: the RS phase owner after owner, every CTA's gather warps
    pulling the owners' reduced chunks in the same order; every rank's full C vs fp64."""
    M, K, N = 256 * W, 256, 520
    A, B = si.rs_inputs(W, M, K, N, salt=47)
    ctxs, plans = _world(ao, dict(op="gemm_ar", world_size=W, M=M, N=N, K=K, chunk_rows=64, backend="ldst",
                                  n_slices=4, rs_reduce=reduce, tile_m=256, tile_n=256, n_cta=SMS,
                                  timeout_ns=2_000_000_000), W)
    ref = on.gemm_ar([si.to_f64(a) for a in A], [si.to_f64(b) for b in B])
    dA, dB = _dev(A), _dev(B)
    for it in range(2):
        Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
        ao.gemm_ar_group(plans, dA, dB, Cs)
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_async()
        for r in range(W):
            _check(Cs[r], ref, f"ar ts W={W} {reduce} it={it} r{r}")
        for r in range(1, W):
            assert torch.equal(Cs[r], Cs[0]), "every rank gathers the same reduced rows"


@pytest.mark.parametrize("n", [2, 8])
def test_gemm_batched_timesliced(ao, n):
    M, N, K = 512, 520, 1000
    A, B = si.ag_inputs(n, n * M, K, N, salt=37)
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    ao.gemm_batched(_dev(A), _dev(B), Cs, tile_m=256, tile_n=256, group_m=4, n_cta=SMS)
    torch.cuda.synchronize()
    for i in range(n):
        _check(Cs[i], on.gemm(si.to_f64(A[i]), si.to_f64(B[i])), f"gemm_batched ts n={n} #{i}")


def test_timesliced_rejects_a_partial_world(ao):
    """Only a whole world can be time-sliced: two ranks of a 4-rank world whose plans ask
    for all SMs keep the co-residency error."""
    W, M, K, N = 4, 512, 64, 256
    B = [torch.zeros(N, K, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    C = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    A = [torch.zeros(M // W, K, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    d = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=64, backend="ce", n_cta=SMS)
    ctxs, plans = _world(ao, d, W)
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.ag_gemm_group(plans[:2], A, B, C)


def test_bench_config_timesliced_fullsize(ao):
    """The bench launch configuration (Llama-3-8B FFN, TP=8 loopback, time-sliced over all
    SMs, CE push AG + atomic RS, 256x256 pair tiles): sampled rows vs the fp64 oracle,
    every chunk boundary row included."""
    W, M, H, F = 8, 8192, 4096, 14336 // 8
    base = dict(world_size=W, M=M, chunk_rows=1024, intra="grouped", group_m=4, n_cta=SMS, tile_m=256,
                tile_n=256, timeout_ns=10_000_000_000)
    ag_d = dict(base, op="ag_gemm", N=F, K=H, backend="ce")
    rs_d = dict(base, op="gemm_rs", N=H, K=F, rs_reduce="atomic")
    ctxs = ao.loopback_world(0, W, max(ao.workspace_bytes(ag_d), ao.workspace_bytes(rs_d)))
    pa = [ao.Plan(ctxs[r], dict(ag_d, rank=r)) for r in range(W)]
    pr = [ao.Plan(ctxs[r], dict(rs_d, rank=r)) for r in range(W)]
    A, Bu = si.ag_inputs(W, M, H, F)
    Bd = si.rs_weights(W, F, H)
    dA, dBu, dBd = _dev(A), _dev(Bu), _dev(Bd)
    Cu = [torch.empty(M, F, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    Cd = [torch.empty(M // W, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for _ in range(2):  # second call exercises the other parity and the re-armed accumulator
        ao.ag_gemm_group(pa, dA, dBu, Cu)
        ao.gemm_rs_group(pr, Cu, dBd, Cd)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    rng = np.random.default_rng(7)
    # every rank; each shard's first / last rows and a tile-boundary row of every 256-row
    # block (both CTAs of a pair, chunk edges) plus random rows
    edges = np.concatenate([np.arange(0, M, 256), np.arange(127, M, 256), np.arange(128, M, 256), np.arange(255, M, 256)])
    rows = np.unique(np.concatenate([edges[::3], rng.integers(0, M, 48)]))
    A64 = [si.to_f64(a) for a in A]
    for r in range(W):
        ref = on.ag_gemm_rows(A64, si.to_f64(Bu[r]), rows)
        _check(Cu[r][torch.as_tensor(rows)], ref, f"fullsize ag ts r{r}")
    # RS consumes the GPU's up-proj output (bit-identical input on both sides); every owner,
    # 96+ of its 1024 rows (every sub-tile half of each 256-row block, random rows)
    Cu64 = [Cu[s].float().cpu().numpy().astype(np.float64) for s in range(W)]
    Bd64 = [si.to_f64(b) for b in Bd]
    lrows = np.unique(np.concatenate([np.arange(0, M // W, 16), [127, 128, 1023], rng.integers(0, M // W, 32)]))
    for r in range(W):
        ref = on.gemm_rs_rows(Cu64, Bd64, r, lrows)
        _check(Cd[r][torch.as_tensor(lrows)], ref, f"fullsize rs ts r{r}")


@pytest.mark.parametrize("op", ["ag_gemm", "gemm_rs", "gemm_ar"])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [2, 4])
def test_timesliced_mma_order_matches_oracle(ao, op, tile, W, tmp_path):
    """The time-sliced launch order executed on the device equals the oracle's enumeration
    (oracle.schedule.group_schedule) tile for tile: the MMA trace gives each worker's tiles
    in issue order, and worker w's m-th tile must be global list entry w + m * n_workers."""
    import json

    from oracle import schedule as osch
    M, K, N, C = 256 * W, 256, 768, 64
    desc = dict(op=op, world_size=W, M=M, N=N, K=K, chunk_rows=C, tile_m=tile[0], tile_n=tile[1], n_cta=SMS,
                intra="grouped", group_m=2, backend="ldst" if op == "gemm_ar" else "ce",
                rs_reduce="atomic" if op == "gemm_rs" else "slots", timeout_ns=2_000_000_000)
    ctxs, plans = _world(ao, desc, W)
    if op == "ag_gemm":
        A, B = si.ag_inputs(W, M, K, N, salt=43)
        run = lambda: _ag(ao, ctxs, plans, _dev(A), _dev(B))  # noqa: E731
    else:
        A, B = si.rs_inputs(W, M, K, N, salt=44)
        if op == "gemm_rs":
            run = lambda: _rs(ao, ctxs, plans, _dev(A), _dev(B))  # noqa: E731
        else:
            def run():
                Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
                ao.gemm_ar_group(plans, _dev(A), _dev(B), Cs)
                torch.cuda.synchronize()
    run()
    ctxs[0].trace_enable(1 << 20)
    run()
    path = str(tmp_path / "ts_trace.json")
    ctxs[0].trace_dump(path)
    ctxs[0].trace_enable(0)
    ev = [e for e in json.load(open(path))["traceEvents"] if e["cat"] == "mma"]
    descs = [osch.default_desc(**{k: v for k, v in dict(desc, rank=r).items() if k != "timeout_ns"})
             for r in range(W)]
    sched = osch.group_schedule(descs, SMS)
    assert sched["mode"] == "time_sliced"
    # the library's own export says the same
    hp = [ao.Plan(None, d, SMS) for d in descs]
    assert ao.group_schedule_json(hp, SMS) == osch.export_json(sched)
    orders = {d["rank"]: osch.plan(d, SMS)["order"] for d in descs}
    seq = [(r, orders[r][k]) for r, k0, k1, o in sched["segments"] for k in range(k0, k1)]
    nw, cg = sched["n_workers"], tile[0] // 128
    got = {}
    for cta in sorted({e["tid"] // 8 for e in ev}):
        mine = sorted((e for e in ev if e["tid"] // 8 == cta), key=lambda e: e["ts"])
        for m, e in enumerate(mine):
            got[cta // cg + m * nw] = (e["pid"], int(e["name"].split()[1]))
    assert len(got) == len(seq)
    for i, want in enumerate(seq):
        assert got[i] == want, (i, got[i], want)
