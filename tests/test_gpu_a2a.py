"""GPU parity of A2A-GEMM (NEXT-3: MoE All-to-All dispatch + expert GEMM) vs the fp64 oracle
(oracle/a2a.py), through the C ABI.  Received row counts and route positions are integer
results (bit-exact); Y within the north-star tolerance (1e-2 per element relative to
max(1, |ref|), Frobenius 2e-3); provenance rows bit-exact."""
import numpy as np
import pytest
import torch

from oracle import a2a as oa
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


def _world(ao, W, T, H, N, k, C, ts, **kw):
    d = dict(op="a2a_gemm", world_size=W, M=T, N=N, K=H, topk=k, chunk_rows=C, backend="ldst",
             n_cta=SMS if ts else SMS // W, timeout_ns=2_000_000_000)
    d.update(kw)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    return ctxs, [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]


def _run(ao, ctxs, plans, X, idx, B, N):
    W = len(plans)
    T, k = idx[0].shape
    Y = [torch.full((W * T, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    rp = [torch.full((T, k), -1, dtype=torch.int32, device="cuda") for _ in range(W)]
    rr = [torch.full((1,), -1, dtype=torch.int32, device="cuda") for _ in range(W)]
    ao.a2a_gemm_group(plans, [x.cuda() for x in X], [i.cuda() for i in idx], [b.cuda() for b in B], Y, rp, rr)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Y, rp, [int(r.item()) for r in rr]


def _check_all(Y, rp, rr, X, idx, B, what):
    W = len(Y)
    Xn = [si.to_f64(x) for x in X]
    In = [i.numpy().astype(np.int64) for i in idx]
    ref = oa.a2a_gemm(Xn, In, [si.to_f64(b) for b in B])
    pos = oa.route_positions(In)
    for e in range(W):
        assert rr[e] == ref[e].shape[0], f"{what}: expert {e} received {rr[e]} rows, oracle {ref[e].shape[0]}"
        np.testing.assert_array_equal(rp[e].cpu().numpy(), pos[e], err_msg=f"{what}: route_pos of rank {e}")
        if rr[e]:
            ok, el, fr = on.check_tolerance(Y[e][: rr[e]].float().cpu().numpy(), ref[e])
            assert ok, f"{what}: expert {e}: max elem err {el:.3e}, frob {fr:.3e}"


@pytest.mark.parametrize("ts", [False, True])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W,T,k,C", [(2, 128, 1, 64), (4, 128, 2, 16), (8, 128, 2, 32), (8, 96, 2, 24)])
def test_a2a_vs_oracle(ao, W, T, k, C, tile, ts):
    if (W * T) % tile[0]:
        pytest.skip("receive capacity not a multiple of the tile rows")
    H, N = 256, 520
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k, salt=W + T + C)
    ctxs, plans = _world(ao, W, T, H, N, k, C, ts, tile_m=tile[0], tile_n=tile[1])
    Y, rp, rr = _run(ao, ctxs, plans, X, idx, B, N)
    _check_all(Y, rp, rr, X, idx, B, f"a2a W={W} T={T} k={k} C={C} tile={tile} ts={ts}")


@pytest.mark.parametrize("ts", [False, True])
def test_a2a_zipf_skew_and_epochs(ao, ts):
    """Zipf-skewed routing (one expert receives most rows, another may receive none),
    three back-to-back calls (both parities, re-sent count tables)."""
    W, T, H, N, k = 8, 256, 128, 256, 2
    ctxs, plans = _world(ao, W, T, H, N, k, 64, ts, tile_m=256, tile_n=256, intra="grouped", group_m=4)
    for it, z in enumerate((1.5, 0.0, 3.0)):
        X, idx, B = si.moe_inputs(W, T, H, N, topk=k, zipf=z, salt=100 + it)
        Y, rp, rr = _run(ao, ctxs, plans, X, idx, B, N)
        _check_all(Y, rp, rr, X, idx, B, f"zipf={z} it={it} ts={ts}")


def test_a2a_degenerate_routings(ao):
    """All tokens to expert 0 (others receive nothing), then all-local routing."""
    W, T, H, N = 4, 128, 64, 256
    ctxs, plans = _world(ao, W, T, H, N, 1, 32, False, tile_m=128, tile_n=128)
    X, _, B = si.moe_inputs(W, T, H, N, topk=1, salt=77)
    for idx in ([torch.zeros(T, 1, dtype=torch.int32) for _ in range(W)],
                [torch.full((T, 1), s, dtype=torch.int32) for s in range(W)]):
        Y, rp, rr = _run(ao, ctxs, plans, X, idx, B, N)
        _check_all(Y, rp, rr, X, idx, B, "degenerate")


@pytest.mark.parametrize("ts", [False, True])
def test_a2a_provenance_exact(ao, ts):
    W, T, H, N, k = 8, 128, 64, 256, 2
    _, idx, _ = si.moe_inputs(W, T, H, N, topk=k, salt=5)
    ctxs, plans = _world(ao, W, T, H, N, k, 16, ts, tile_m=256, tile_n=256)
    In = [i.numpy().astype(np.int64) for i in idx]
    for ep in range(1, 4):
        X, idx2, B = si.moe_provenance_inputs(W, T, H, N, idx, epoch=ep)
        Y, rp, rr = _run(ao, ctxs, plans, X, idx2, B, N)
        for e in range(W):
            y = Y[e][: rr[e]].float().cpu()
            gid = (y[:, 0] + 32 * y[:, 1] + 1024 * y[:, 2]).numpy()
            want = [s * T + t for s in range(W) for t in range(T) if e in In[s][t]]
            np.testing.assert_array_equal(gid, want)
            assert torch.all(y[:, 3] == ep % 32)


def test_a2a_rejects_bad_plans(ao):
    W, T = 2, 128
    base = dict(op="a2a_gemm", world_size=W, M=T, N=256, K=64, topk=2, chunk_rows=32, backend="ldst")
    for bad in (dict(topk=3), dict(topk=0), dict(backend="ce"), dict(chunk_rows=12), dict(tile_m=256, tile_n=256, M=64)):
        assert ao.validate(dict(base, rank=0, **bad)), bad
    assert not ao.validate(dict(base, rank=0))


def test_a2a_mixtral_fullsize_sampled(ao):
    """BASELINE configs[3]: Mixtral-8x7B MoE, 8 experts over 8 ranks (loopback, time-sliced
    over all SMs), top-2 of 8192 tokens (1024 per rank), H = 4096, w1||w3 (N = 28672):
    counts and route positions exact, sampled Y rows (every block boundary) vs fp64."""
    W, T, H, N, k = 8, 1024, 4096, 2 * 14336, 2
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k)
    ctxs, plans = _world(ao, W, T, H, N, k, 128, True, tile_m=256, tile_n=256, intra="grouped", group_m=8,
                         timeout_ns=10_000_000_000)
    Y, rp, rr = _run(ao, ctxs, plans, X, idx, B, N)
    Xn = [si.to_f64(x) for x in X]
    In = [i.numpy().astype(np.int64) for i in idx]
    cnt = oa.counts(In, W)
    pos = oa.route_positions(In)
    rng = np.random.default_rng(3)
    for e in range(W):
        assert rr[e] == cnt[:, e].sum()
        np.testing.assert_array_equal(rp[e].cpu().numpy(), pos[e])
    for e in (0, 3, 7):
        starts = np.concatenate([[0], np.cumsum(cnt[:, e])])
        rows = np.unique(np.concatenate([starts[:-1], np.maximum(starts[1:] - 1, 0), rng.integers(0, rr[e], 8)]))
        rows = rows[rows < rr[e]]
        ref = oa.a2a_gemm_rows(Xn, In, si.to_f64(B[e]), e, rows)
        ok, el, fr = on.check_tolerance(Y[e][torch.as_tensor(rows)].float().cpu().numpy(), ref)
        assert ok, f"fullsize expert {e}: {el:.3e} {fr:.3e}"


@pytest.mark.parametrize("ts", [False, True])
def test_a2a_device_schedule_matches_oracle(ao, ts, tmp_path):
    """The routing-dependent tile order built on the device (chunk->tile join on ragged
    source blocks, arrival sort, GROUP_M) equals oracle.a2a.schedule tile for tile: the
    MMA trace events give each worker's tiles in execution order, and worker w's m-th tile
    is list position w + m * n_workers (Lst.1's persistent stride)."""
    import json
    W, T, H, N, k, C, gm = 4, 256, 64, 384, 2, 32, 2
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k, zipf=1.3, salt=61)
    n_cta = SMS if ts else 3
    ctxs, plans = _world(ao, W, T, H, N, k, C, ts, tile_m=128, tile_n=128, intra="grouped", group_m=gm,
                         n_cta=n_cta)
    _run(ao, ctxs, plans, X, idx, B, N)  # warm (epoch 1)
    ctxs[0].trace_enable(1 << 20)
    _run(ao, ctxs, plans, X, idx, B, N)
    path = str(tmp_path / "a2a_trace.json")
    ctxs[0].trace_dump(path)
    ctxs[0].trace_enable(0)
    ev = [e for e in json.load(open(path))["traceEvents"] if e["cat"] == "mma"]
    cnt = oa.counts([i.numpy().astype(np.int64) for i in idx], W)
    n_nb = -(-N // 128)
    sched = [oa.schedule(cnt, e, T, C, 128, n_nb, gm) for e in range(W)]
    if ts:
        glob = [(e, t) for e in range(W) for t in sched[e]]
        got = {}
        for cta in sorted({e["tid"] // 8 for e in ev}):
            mine = sorted((e for e in ev if e["tid"] // 8 == cta), key=lambda e: e["ts"])
            for m, e in enumerate(mine):
                got[cta + m * n_cta] = (e["pid"], int(e["name"].split()[1]))
        assert len(got) == len(glob)
        for i, (e, (mb, nb)) in enumerate(glob):
            assert got[i] == (e, mb * n_nb + nb), (i, got[i], (e, mb, nb))
    else:
        for e in range(W):
            got = {}
            for cta in range(n_cta):
                mine = sorted((x for x in ev if x["pid"] == e and x["tid"] // 8 == cta), key=lambda x: x["ts"])
                for m, x in enumerate(mine):
                    got[cta + m * n_cta] = int(x["name"].split()[1])
            assert [got[i] for i in range(len(sched[e]))] == [mb * n_nb + nb for mb, nb in sched[e]], e


def test_a2a_delays_are_safe_and_a_dropped_wait_is_caught(ao):
    """Fault injection: random delays before every chunk-flag release never
    change the result; dropping the waits of one tile while pushes are delayed is caught by
    the provenance decode (the chunk waits are load-bearing); recovery afterwards."""
    W, T, H, N, k = 4, 256, 64, 256, 2
    _, idx, _ = si.moe_inputs(W, T, H, N, topk=k, salt=9)
    ctxs, plans = _world(ao, W, T, H, N, k, 64, False, tile_m=128, tile_n=128, n_cta=4)
    In = [i.numpy().astype(np.int64) for i in idx]

    def decode_ok(ep):
        X, idx2, B = si.moe_provenance_inputs(W, T, H, N, idx, epoch=ep)
        Y, rp, rr = _run(ao, ctxs, plans, X, idx2, B, N)
        ok = True
        for e in range(W):
            y = Y[e][: rr[e]].float().cpu()
            gid = (y[:, 0] + 32 * y[:, 1] + 1024 * y[:, 2]).numpy()
            want = [s * T + t for s in range(W) for t in range(T) if e in In[s][t]]
            ok &= bool(np.array_equal(gid, want)) and bool(torch.all(y[:, 3] == ep % 32))
        return ok

    try:
        ao.debug_set("delay_ns", 2_000_000)
        assert decode_ok(1), "delayed pushes must not change the result"
        ao.debug_set("skip_wait", 0)
        assert not decode_ok(2), "a dropped wait must be observable (mutation kill)"
    finally:
        ao.debug_set("skip_wait", -1)
        ao.debug_set("delay_ns", 0)
    assert decode_ok(3)



def test_a2a_invalid_routing_is_reported_not_read_out_of_bounds(ao):
    """topk_idx entries outside [0, W) or repeated within a token are dropped by the prep
    kernel (route_pos = -1, the token is not dispatched for that choice) and reported as
    AO_ERR_INVALID_ARG by check_async; valid entries are routed as usual."""
    W, T, H, N, k, C = 2, 256, 64, 256, 2, 32
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k, salt=71)
    bad = [i.clone() for i in idx]
    bad[0][5, 1] = 7           # out of range
    bad[0][9, 1] = bad[0][9, 0]  # duplicate
    bad[1][3, 0] = -1          # negative
    ctxs, plans = _world(ao, W, T, H, N, k, C, False, tile_m=128, tile_n=128, n_cta=16)
    Y = [torch.zeros((W * T, N), dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    rp = [torch.zeros((T, k), dtype=torch.int32, device="cuda") for _ in range(W)]
    rr = [torch.zeros((1,), dtype=torch.int32, device="cuda") for _ in range(W)]
    ao.a2a_gemm_group(plans, [x.cuda() for x in X], [i.cuda() for i in bad], [b.cuda() for b in B], Y, rp, rr)
    torch.cuda.synchronize()
    with pytest.raises(ao.AOError) as ei:
        for c in ctxs:
            c.check_async()
    assert ei.value.status == "AO_ERR_INVALID_ARG"
    assert int(rp[0][5, 1]) == -1 and int(rp[0][9, 1]) == -1 and int(rp[1][3, 0]) == -1
    # the valid entries still received rows: total rows = valid (token, choice) pairs
    n_valid = sum(int((b >= 0).sum()) for b in bad) - 2  # 7 and the duplicate dropped (-1 counted out already)
    assert sum(int(r.item()) for r in rr) == n_valid
