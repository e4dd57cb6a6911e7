"""GPU parity of the stream-K tail (Q28): plans whose last two waves of tiles are
split along K over all workers (a tail piece stores its fp32 partial, the head piece of the
same tile adds it) against the fp64 oracle, element by element; AG provenance stays exact
over back-to-back epochs (the partial workspace and its flags are reused every launch).
"""
import numpy as np
import pytest
import torch

from oracle import numeric as on
from oracle import schedule as osch
from synthetic import inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _check(gpu, ref, what):
    ok, e, f = on.check_tolerance(gpu.float().cpu().numpy(), ref)
    assert ok, f"{what}: max elem err {e:.3e}, frob {f:.3e}"


@pytest.fixture
def gemm_sk(ao):
    ao.debug_set("gemm_stream_k", 1)
    yield
    ao.debug_set("gemm_stream_k", 0)


# (M, N, K, tile): tile counts that leave a partial wave on the 74 pair / 148 single workers;
# K ragged (1000 = 15.6 k-blocks), K short (one k-block: the tail is whole tiles)
@pytest.mark.parametrize("M,N,K,tile", [(4096, 1792, 1000, (256, 256)), (8192, 1792, 4096, (256, 256)),
                                        (2048, 2816, 520, (256, 128)), (8192, 1024, 2048, (128, 256)),
                                        (8192, 2560, 64, (256, 256)), (8192, 1792, 4096, (256, 224))])
def test_gemm_stream_k_vs_oracle(ao, gemm_sk, M, N, K, tile):
    A, B = si.ag_inputs(1, M, K, N, salt=M + N + K + 7)
    C = ao.gemm(A[0].cuda(), B[0].cuda(), tile_m=tile[0], tile_n=tile[1])
    torch.cuda.synchronize()
    rows = np.arange(M) if M * N * K <= 4096 * 1792 * 1000 else np.unique(
        np.concatenate([np.arange(0, M, 61), np.arange(M - 300, M)]))
    ref = on.gemm_rows(si.to_f64(A[0]), si.to_f64(B[0]), rows)
    _check(C[torch.as_tensor(rows)], ref, f"gemm stream-K {M}x{N}x{K} {tile}")


def test_gemm_stream_k_repeat_is_bitwise_stable(ao, gemm_sk):
    # each split tile is the head's TMEM value + one tail partial: fixed summation order
    M, N, K = 4096, 1792, 1000
    A, B = si.ag_inputs(1, M, K, N, salt=3)
    a, b = A[0].cuda(), B[0].cuda()
    c0 = ao.gemm(a, b, tile_m=256, tile_n=256).clone()
    for _ in range(3):
        assert torch.equal(ao.gemm(a, b, tile_m=256, tile_n=256), c0)


def _ag_world(ao, W, desc):
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(desc))
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    return ctxs, plans


@pytest.mark.parametrize("dirn", ["push", "pull"])
@pytest.mark.parametrize("W,n_cta,tile,K", [(2, 10, (256, 256), 512), (2, 7, (128, 256), 1000), (4, 18, (256, 128), 136)])
def test_ag_gemm_stream_k_vs_oracle(ao, W, n_cta, tile, K, dirn):
    # space-sliced loopback group (n_cta CTAs = n_cta / cta_group workers per rank): each rank's workers run the data-parallel waves, then
    # the stream-K tail; the plan's per-worker chunk waits follow the stream-K walk
    M, N, C = 1024 * W, 768, 128
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=C, backend="ce", tile_m=tile[0],
                tile_n=tile[1], n_cta=n_cta, stream_k=1, intra="grouped", group_m=2, dir=dirn,
                timeout_ns=2_000_000_000)
    p = osch.plan(osch.default_desc(**dict(desc, rank=0)))
    assert p.get("sk_dp", None) is not None and p["sk_dp"] < len(p["order"])
    A, B = si.ag_inputs(W, M, K, N, salt=11)
    ctxs, plans = _ag_world(ao, W, desc)
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.ag_gemm_group(plans, [a.cuda() for a in A], [b.cuda() for b in B], Cs)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    A64 = [si.to_f64(a) for a in A]
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag stream-K W={W} rank {r}")
    for c in ctxs:
        c.close()


def test_ag_gemm_stream_k_provenance_epochs(ao):
    W, M, K, N = 2, 2048, 256, 768
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=128, backend="ce", tile_m=256, tile_n=256,
                n_cta=10, stream_k=1, timeout_ns=2_000_000_000)
    ctxs, plans = _ag_world(ao, W, desc)
    for it in range(5):
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=it + 1)
        Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
        ao.ag_gemm_group(plans, [a.cuda() for a in A], [b.cuda() for b in B], Cs)
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_async()
        for r in range(W):
            c = Cs[r].float().cpu()
            rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
            assert torch.equal(rid, torch.arange(M, dtype=torch.float32)), (it, r)
            assert torch.all(c[:, 3] == (it + 1) % 32)
    for c in ctxs:
        c.close()


def test_ag_gemm_stream_k_per_rank_full_size(ao):
    # the per-GPU TP=8 up-proj (8192 x 1792 x 4096) of rank 0 alone on all SMs with auto
    # stream-K (224 pair tiles on 74 workers: 148 data-parallel, 76 split), peers simulated
    # as arrived (the bench's per-rank leg).  Two whole-world launches (time-sliced, epochs 1
    # and 2) first fill both parities' gathered buffers with the real gather, so epoch 3's
    # buffer holds concat_p A_p.  Sampled rows vs the oracle.
    W, M, K, N = 8, 8192, 4096, 1792
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=1024, backend="ce", tile_m=256,
                tile_n=256, n_cta=148, stream_k=-1, intra="grouped", group_m=4, timeout_ns=5_000_000_000)
    assert osch.plan(osch.default_desc(**dict(desc, rank=0)))["sk_dp"] == 148
    ctxs, plans = _ag_world(ao, W, desc)
    A, B = si.ag_inputs(W, M, K, N)
    Ad, Bd = [a.cuda() for a in A], [b.cuda() for b in B]
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for _ in range(2):
        ao.ag_gemm_group(plans, Ad, Bd, Cs)
    torch.cuda.synchronize()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ao.debug_set("prearrive", 1)
    try:
        ao.ag_gemm(plans[0], Ad[0], Bd[0], C)
        torch.cuda.synchronize()
    finally:
        ao.debug_set("prearrive", 0)
    ctxs[0].check_async()
    rows = np.unique(np.concatenate([np.arange(0, M, 113), np.arange(M - 64, M)]))
    ref = on.gemm_rows(si.to_f64(torch.cat(A, 0)), si.to_f64(B[0]), rows)
    _check(C[torch.as_tensor(rows)], ref, "ag stream-K per-rank full size")
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("tile,n_cta", [((256, 256), 10), ((128, 256), 7)])
def test_stream_k_mma_order_matches_oracle(ao, tile, n_cta, tmp_path):
    """The device executes the stream-K walk of oracle.schedule.worker_pieces: the MMA trace
    gives each worker's tiles in issue order, which must be the tiles of the worker's pieces
    (data-parallel positions, then its contiguous stream-K range; a split tile appears in
    two adjacent workers)."""
    import json
    W, M, N, K, C = 2, 2048, 768, 512, 128
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=C, backend="ce", tile_m=tile[0],
                tile_n=tile[1], n_cta=n_cta, stream_k=1, intra="grouped", group_m=2, timeout_ns=2_000_000_000)
    ctxs, plans = _ag_world(ao, W, desc)
    A, B = si.ag_inputs(W, M, K, N, salt=19)
    dA, dB = [a.cuda() for a in A], [b.cuda() for b in B]
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.ag_gemm_group(plans, dA, dB, Cs)
    ctxs[0].trace_enable(1 << 16)
    ao.ag_gemm_group(plans, dA, dB, Cs)
    torch.cuda.synchronize()
    path = str(tmp_path / "sk_trace.json")
    ctxs[0].trace_dump(path)
    ctxs[0].trace_enable(0)
    ev = [e for e in json.load(open(path))["traceEvents"] if e["cat"] == "mma"]
    cg = tile[0] // 128
    for r in range(W):
        p = osch.plan(osch.default_desc(**{k: v for k, v in dict(desc, rank=r).items() if k != "timeout_ns"}))
        T, nw, nkb = len(p["order"]), p["n_cta"], (K + 63) // 64
        assert p["sk_dp"] < T
        # space-sliced group: rank group r owns CTAs [r*n_cta, (r+1)*n_cta); tid // 8 = CTA index in the group
        for w in range(nw):
            want = [p["order"][pc[0]] for pc in osch.worker_pieces(T, nw, p["sk_dp"], nkb, w)]
            mine = sorted((e for e in ev if e["pid"] == r and (e["tid"] // 8) // cg == w), key=lambda e: e["ts"])
            got = [int(e["name"].split()[1]) for e in mine]
            assert got == want, (r, w, got, want)
    for c in ctxs:
        c.close()
