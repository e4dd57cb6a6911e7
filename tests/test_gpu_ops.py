"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle, element by element.

Tolerance (BASELINE.json north star): |gpu - oracle| <= 1e-2 * max(1, |oracle|) per element
and relative Frobenius error <= 2e-3.  Integer/provenance and copy results are bit-exact.
Multi-rank cases run in loopback (W ranks of one world on this GPU, one fused launch).
"""
import numpy as np
import pytest
import torch

from oracle import numeric as on
from synthetic import inputs as si

pytestmark = pytest.mark.gpu


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


# ------------------------------------------------------------------------ plain GEMM
@pytest.mark.parametrize("bm", [128, 256])
@pytest.mark.parametrize("M,N,K,bn", [(256, 256, 64, 256), (256, 512, 512, 256), (768, 392, 136, 256),
                                      (512, 520, 1000, 128), (1024, 2048, 4096, 256), (256, 128, 8, 128),
                                      (256, 384, 0, 256), (128, 256, 64, 256)])
def test_gemm_vs_oracle(ao, M, N, K, bn, bm):
    if M % bm:
        pytest.skip("M not a multiple of the tile")
    A, B = si.ag_inputs(1, M, K, N, salt=M + N + K)
    A, B = A[0], B[0]
    C = ao.gemm(A.cuda(), B.cuda(), tile_n=bn, tile_m=bm)
    torch.cuda.synchronize()
    ref = on.gemm(si.to_f64(A), si.to_f64(B))
    _check(C, ref, f"gemm {M}x{N}x{K}")


def test_gemm_large_sampled(ao):
    # full per-rank shape of BASELINE configs[1] at TP=1 (8192 x 14336 x 4096), sampled rows
    M, N, K = 8192, 14336, 4096
    A, B = si.ag_inputs(1, M, K, N)
    C = ao.gemm(A[0].cuda(), B[0].cuda())
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.arange(0, M, 997), [M - 1, 127, 128]]))
    ref = on.gemm_rows(si.to_f64(A[0]), si.to_f64(B[0]), rows)
    _check(C[torch.as_tensor(rows)], ref, "gemm large sampled")


@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("n", [1, 3, 8])
def test_gemm_batched_vs_oracle(ao, n, tile):
    # the GEMM-only leg: n problems in one launch, each on its own workers
    M, N, K = 512, 520, 1000
    A, B = si.ag_inputs(n, n * M, K, N, salt=31)
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    ao.gemm_batched(_dev(A), _dev(B), Cs, tile_m=tile[0], tile_n=tile[1], group_m=4)
    torch.cuda.synchronize()
    for i in range(n):
        _check(Cs[i], on.gemm(si.to_f64(A[i]), si.to_f64(B[i])), f"gemm_batched n={n} #{i}")


# ------------------------------------------------------------------------ AG-GEMM loopback
def _ag_world(ao, W, M, N, K, chunk, backend, **kw):
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=chunk, backend=backend,
                n_cta=max(1, 148 // W), timeout_ns=2_000_000_000)
    desc.update(kw)
    ws = ao.workspace_bytes(desc)
    ctxs = ao.loopback_world(0, W, ws)
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    return ctxs, plans


def _run_ag(ao, ctxs, plans, A, B, gather=False):
    W = len(plans)
    M = sum(a.shape[0] for a in A)
    Cs = [torch.empty(M, B[r].shape[0], dtype=torch.bfloat16, device="cuda") for r in range(W)]
    G = [torch.empty(M, A[0].shape[1], dtype=torch.bfloat16, device="cuda") for _ in range(W)] if gather else None
    ao.ag_gemm_group(plans, A, B, Cs, G)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Cs, G


@pytest.mark.parametrize("tile", [(128, 128), (256, 128), (256, 256)])
@pytest.mark.parametrize("backend", ["ce", "ldst", "tma"])
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_ag_gemm_tiny_vs_oracle(ao, backend, W, tile):
    # BASELINE configs[0]: M=256/rank, K=512, N=512, chunk=64 rows
    M, K, N, C = 256 * W, 512, 512, 64
    A, B = si.ag_inputs(W, M, K, N)
    ctxs, plans = _ag_world(ao, W, M, N, K, C, backend, tile_m=tile[0], tile_n=tile[1], n_slices=2)
    Cs, G = _run_ag(ao, ctxs, plans, _dev(A), _dev(B), gather=True)
    A64 = [si.to_f64(a) for a in A]
    full = torch.cat(A, 0)
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag W={W} {backend} rank {r}")
        assert torch.equal(G[r].cpu(), full), "gathered A must be a bit-exact copy"


@pytest.mark.parametrize("backend", ["ce", "ldst", "tma"])
def test_ag_gemm_provenance_exact(ao, backend):
    W, M, K, N = 4, 1024, 64, 256
    ctxs, plans = _ag_world(ao, W, M, N, K, 64, backend, n_slices=3)
    for it in range(5):  # back-to-back epochs exercise both parities
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=it + 1)
        Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
        for r in range(W):
            c = Cs[r].float().cpu()
            rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
            assert torch.equal(rid, torch.arange(M, dtype=torch.float32)), (backend, it, r)
            assert torch.all(c[:, 3] == (it + 1) % 32)


@pytest.mark.parametrize("W,ragged", [(2, False), (4, True)])
def test_ag_gemm_ragged_and_orders(ao, W, ragged):
    M, K, N = 512 * W, 1000 if ragged else 1024, 1000 if ragged else 768
    for kw in (dict(intra="grouped", group_m=2), dict(intra="col", chunk_order="chunk_major")):
        A, B = si.ag_inputs(W, M, K, N, salt=3)
        ctxs, plans = _ag_world(ao, W, M, N, K, 128, "ce", **kw)
        Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
        A64 = [si.to_f64(a) for a in A]
        for r in range(W):
            _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag ragged W={W} {kw} r{r}")


# ------------------------------------------------------------------------ GEMM-RS loopback
def _rs_world(ao, W, M, N, K, chunk, **kw):
    desc = dict(op="gemm_rs", world_size=W, M=M, N=N, K=K, chunk_rows=chunk,
                n_cta=max(1, 148 // W), timeout_ns=2_000_000_000, **kw)
    ws = ao.workspace_bytes(desc)
    ctxs = ao.loopback_world(0, W, ws)
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    return ctxs, plans


def _run_rs(ao, ctxs, plans, A, B):
    W = len(plans)
    M, N = A[0].shape[0], B[0].shape[0]
    Cs = [torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.gemm_rs_group(plans, A, B, Cs)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Cs


@pytest.mark.parametrize("tile", [(128, 128), (256, 128), (256, 256)])
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_gemm_rs_tiny_vs_oracle(ao, W, tile):
    M, K, N, C = 256 * W, 256, 512, 64
    A, B = si.rs_inputs(W, M, K, N)
    ctxs, plans = _rs_world(ao, W, M, N, K, C, tile_m=tile[0], tile_n=tile[1])
    Cs = _run_rs(ao, ctxs, plans, _dev(A), _dev(B))
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    for r in range(W):
        _check(Cs[r], on.gemm_rs(A64, B64, r), f"rs W={W} rank {r}")


def test_gemm_rs_bitmask_and_determinism(ao):
    W, M, K, N = 4, 1024, 64, 520
    ctxs, plans = _rs_world(ao, W, M, N, K, 128)
    A, B = si.rs_provenance_inputs(W, M, K, N)
    for it in range(4):
        Cs = _run_rs(ao, ctxs, plans, _dev(A), _dev(B))
        for r in range(W):
            assert torch.all(Cs[r].float().cpu() == 2 ** W - 1), (it, r)
    A, B = si.rs_inputs(W, M, K, N, salt=5)
    A, B = _dev(A), _dev(B)
    first = [c.clone() for c in _run_rs(ao, ctxs, plans, A, B)]
    second = _run_rs(ao, ctxs, plans, A, B)
    for r in range(W):
        assert torch.equal(first[r], second[r]), "RS must be bitwise deterministic (ascending-rank sum)"


def test_gemm_rs_ragged(ao):
    W, M, K, N = 2, 1024, 1000, 1000
    A, B = si.rs_inputs(W, M, K, N, salt=8)
    ctxs, plans = _rs_world(ao, W, M, N, K, 128, intra="grouped", group_m=2)
    Cs = _run_rs(ao, ctxs, plans, _dev(A), _dev(B))
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    for r in range(W):
        _check(Cs[r], on.gemm_rs(A64, B64, r), f"rs ragged r{r}")


# ------------------------------------------------------------------------ failure paths
@pytest.mark.parametrize("backend", ["ldst", "tma"])
def test_wait_mutation_is_detected_and_delays_are_safe(ao, backend):
    """Fault injection: random per-transfer delays never break results; skipping
    one chunk wait while transfers are delayed is caught by the provenance decode."""
    W, M, K, N = 2, 512, 64, 256
    # chunk = tile rows: the first remote tile of rank 0 / worker 0 waits on exactly one chunk
    ctxs, plans = _ag_world(ao, W, M, N, K, 128, backend, tile_m=128, tile_n=128, n_cta=4)

    def decode_ok(Cs):
        ok = True
        for r in range(W):
            c = Cs[r].float().cpu()
            rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
            ok &= bool(torch.equal(rid, torch.arange(M, dtype=torch.float32)))
        return ok

    try:
        ao.debug_set("delay_ns", 1_000_000)
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=1)
        Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
        assert decode_ok(Cs), "delayed transfers must not change the result"
        ao.debug_set("skip_wait", 0)  # rank 0, worker 0: its first chunk wait is dropped
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=2)
        Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
        assert not decode_ok(Cs), "a dropped wait must be observable (mutation kill)"
    finally:
        ao.debug_set("skip_wait", -1)
        ao.debug_set("delay_ns", 0)
    A, B = si.ag_provenance_inputs(W, M, K, N, epoch=3)
    Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
    assert decode_ok(Cs), "recovers once the mutation is removed"


def test_device_timeout_is_reported(ao):
    """A rank whose peer never runs must not hang: the bounded spin records the first
    expired wait and ao_ctx_check_async reports AO_ERR_TIMEOUT."""
    W, M, K, N = 2, 512, 64, 256
    ctxs, plans = _ag_world(ao, W, M, N, K, 128, "ce", tile_m=128, tile_n=128, n_cta=2, timeout_ns=20_000_000)
    A, B = si.ag_provenance_inputs(W, M, K, N)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ao.ag_gemm_group(plans[:1], [A[0].cuda()], [B[0].cuda()], [C])  # rank 1 never pushes
    torch.cuda.synchronize()
    with pytest.raises(ao.AOError, match="TIMEOUT"):
        ctxs[0].check_async()
    ctxs[0].check_async()  # the error is reported once


def test_boundary_rejects_bad_calls(ao):
    W, M, K, N = 2, 512, 64, 256
    desc = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=64, n_cta=8)
    ctxs = ao.loopback_world(0, W, 4 * ao.workspace_bytes(desc))
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.Plan(ctxs[0], dict(desc, rank=1))  # desc rank != ctx rank
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.Plan(ctxs[0], dict(desc, rank=0, chunk_rows=96))  # S % chunk_rows
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.Plan(ctxs[0], dict(desc, rank=0, M=8 * M))  # workspace too small
    p0 = ao.Plan(ctxs[0], dict(desc, rank=0))
    p1 = ao.Plan(ctxs[1], dict(desc, rank=1, chunk_rows=128))
    A = [torch.zeros(M // W, K, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    B = [torch.zeros(N, K, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    C = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    with pytest.raises(ao.AOError, match="PEER"):
        ao.ag_gemm_group([p0, p1], A, B, C)  # plans of one world must agree (hash)
    rs = ao.Plan(ctxs[0], dict(desc, rank=0, op="gemm_rs", N=64))
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.ag_gemm(rs, A[0], B[0], C[0])  # op mismatch


def test_empty_problem_is_a_noop(ao):
    W = 2
    desc = dict(op="ag_gemm", world_size=W, M=0, N=256, K=64, chunk_rows=64, n_cta=8)
    ctxs = ao.loopback_world(0, W, 1 << 20)
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    z = [torch.empty(0, 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    B = [torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    C = [torch.empty(0, 256, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.ag_gemm_group(plans, z, B, C)
    torch.cuda.synchronize()


@pytest.mark.parametrize("backend", ["tma", "ldst"])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
def test_ag_gemm_dedicated_comm_ctas(ao, backend, tile):
    """Fig.7(b) realization: chunk pushes issued by dedicated communication CTAs
    ("specialized SMs") instead of co-located warps."""
    W, M, K, N = 2, 1024, 256, 512
    A, B = si.ag_inputs(W, M, K, N, salt=11)
    ctxs, plans = _ag_world(ao, W, M, N, K, 128, backend, tile_m=tile[0], tile_n=tile[1], n_cta=64, comm_ctas=8,
                            n_slices=4)
    Cs, G = _run_ag(ao, ctxs, plans, _dev(A), _dev(B), gather=True)
    A64 = [si.to_f64(a) for a in A]
    full = torch.cat(A, 0)
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag comm_ctas {backend} r{r}")
        assert torch.equal(G[r].cpu(), full)


@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_gemm_rs_atomic_vs_oracle(ao, W, tile):
    """rs_reduce=atomic: peers reduce-add into the owner's accumulator (Q23)."""
    M, K, N, C = 256 * W, 256, 520, 64
    A, B = si.rs_inputs(W, M, K, N, salt=13)
    ctxs, plans = _rs_world(ao, W, M, N, K, C, tile_m=tile[0], tile_n=tile[1], rs_reduce="atomic")
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    dA, dB = _dev(A), _dev(B)
    for it in range(3):  # the accumulator must be re-armed (zero) between calls
        Cs = _run_rs(ao, ctxs, plans, dA, dB)
        for r in range(W):
            _check(Cs[r], on.gemm_rs(A64, B64, r), f"rs atomic W={W} it={it} rank {r}")


def test_gemm_rs_atomic_bitmask_and_mode_mixing(ao):
    """Exact integer sums are order-independent, so the bitmask pattern is bit-exact in
    atomic mode; mixing slots / atomic / AG ops on one ctx keeps the accumulator armed."""
    W, M, K, N = 4, 1024, 64, 256
    desc = dict(op="gemm_rs", world_size=W, M=M, N=N, K=K, chunk_rows=128, n_cta=36, timeout_ns=2_000_000_000)
    ag = dict(op="ag_gemm", world_size=W, M=M, N=N, K=K, chunk_rows=128, n_cta=36, timeout_ns=2_000_000_000)
    ctxs = ao.loopback_world(0, W, max(ao.workspace_bytes(desc), ao.workspace_bytes(ag)))
    p_slots = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    p_atom = [ao.Plan(ctxs[r], dict(desc, rank=r, rs_reduce="atomic")) for r in range(W)]
    p_ag = [ao.Plan(ctxs[r], dict(ag, rank=r)) for r in range(W)]
    A, B = si.rs_provenance_inputs(W, M, K, N)
    A, B = _dev(A), _dev(B)
    Ag, Bg = si.ag_inputs(W, M, K, N)
    Ag, Bg = _dev(Ag), _dev(Bg)
    Cg = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for seq in (["atomic", "slots", "atomic", "ag", "atomic", "ag", "ag", "atomic"]):
        if seq == "ag":
            ao.ag_gemm_group(p_ag, Ag, Bg, Cg)
            torch.cuda.synchronize()
            continue
        Cs = _run_rs(ao, ctxs, p_atom if seq == "atomic" else p_slots, A, B)
        for r in range(W):
            assert torch.all(Cs[r].float().cpu() == 2 ** W - 1), seq


# ------------------------------------------------------------------------ RS bf16 wire
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_gemm_rs_bf16_wire(ao, W, tile):
    """rs_wire=bf16 (non-conforming, Q14): each partial is rounded to bf16 and
    reduce-added into a bf16 accumulator, so every addition rounds (each by up to 2^-9 of
    the running sum, in an order that varies run to run).  Accepted with the status AO_OK
    and flagged in ao_last_error; checked against the oracle within the bound that
    arithmetic allows -- per element W * 2^-8 (+ 1e-2) of max(1, |ref|), Frobenius
    2e-3 * W^0.5 (measured at W = 8: up to 2.9e-2 and 4.0e-3) -- epochs re-arm the
    accumulator, and the bitmask pattern (sums of distinct powers of two < 256, exact in
    bf16) stays bit-exact."""
    M, K, N, C = 256 * W, 256, 520, 64
    A, B = si.rs_inputs(W, M, K, N, salt=23)
    ctxs, plans = _rs_world(ao, W, M, N, K, C, tile_m=tile[0], tile_n=tile[1], rs_reduce="atomic", rs_wire="bf16")
    assert "non-conforming" in ao.N.lib().ao_last_error().decode()
    A64, B64 = [si.to_f64(a) for a in A], [si.to_f64(b) for b in B]
    dA, dB = _dev(A), _dev(B)
    for it in range(3):
        Cs = _run_rs(ao, ctxs, plans, dA, dB)
        for r in range(W):
            ok, e, f = on.check_tolerance(Cs[r].float().cpu().numpy(), on.gemm_rs(A64, B64, r),
                                          elem_rel=1e-2 + W * 2.0 ** -8, frob_rel=2e-3 * W ** 0.5)
            assert ok, f"rs bf16 wire W={W} it={it} rank {r}: {e:.3e} {f:.3e}"
    Ap, Bp = si.rs_provenance_inputs(W, M, 64, N)
    ctxs2, plans2 = _rs_world(ao, W, M, N, 64, C, tile_m=tile[0], tile_n=tile[1], rs_reduce="atomic", rs_wire="bf16")
    Cs = _run_rs(ao, ctxs2, plans2, _dev(Ap), _dev(Bp))
    for r in range(W):
        assert torch.all(Cs[r].float().cpu() == 2 ** W - 1)


# ------------------------------------------------------------------------ AG PULL
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("backend", ["ce", "ldst", "tma"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_ag_gemm_pull_vs_oracle(ao, backend, W, tile):
    """dir=pull (Lst.2 with the consumer as issuer): each rank stages
    its shard, then fetches peer chunks (src - r) mod W = d in plan order."""
    M, K, N, C = 256 * W, 512, 512, 64
    A, B = si.ag_inputs(W, M, K, N, salt=17)
    ctxs, plans = _ag_world(ao, W, M, N, K, C, backend, dir="pull", tile_m=tile[0], tile_n=tile[1], n_slices=2)
    Cs, G = _run_ag(ao, ctxs, plans, _dev(A), _dev(B), gather=True)
    A64 = [si.to_f64(a) for a in A]
    full = torch.cat(A, 0)
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag pull W={W} {backend} rank {r}")
        assert torch.equal(G[r].cpu(), full), "gathered A must be a bit-exact copy"


@pytest.mark.parametrize("backend", ["ce", "ldst", "tma"])
def test_ag_gemm_pull_provenance_epochs_and_delays(ao, backend):
    """Back-to-back epochs (both parities, staged regions reused) with random per-transfer
    delays on the in-kernel backends: every output row decodes to its gathered row id."""
    W, M, K, N = 4, 1024, 64, 256
    ctxs, plans = _ag_world(ao, W, M, N, K, 64, backend, dir="pull", chunk_order="chunk_major", n_slices=3)
    try:
        for it in range(6):
            ao.debug_set("delay_ns", 200_000 if (backend != "ce" and it % 2) else 0)
            A, B = si.ag_provenance_inputs(W, M, K, N, epoch=it + 1)
            Cs, _ = _run_ag(ao, ctxs, plans, _dev(A), _dev(B))
            for r in range(W):
                c = Cs[r].float().cpu()
                rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
                assert torch.equal(rid, torch.arange(M, dtype=torch.float32)), (backend, it, r)
                assert torch.all(c[:, 3] == (it + 1) % 32)
    finally:
        ao.debug_set("delay_ns", 0)


@pytest.mark.parametrize("dir_", ["push", "pull"])
@pytest.mark.parametrize("backend", ["ce", "tma"])
def test_ag_gemm_per_rank_calls_on_separate_streams(ao, backend, dir_):
    """The multi-process protocol in one process: each rank is its own call (n_group = 1)
    on its own stream, as with one process per GPU; CE pull then waits on the source's
    ready flag with cuStreamWaitValue32."""
    W, M, K, N = 2, 1024, 256, 512
    A, B = si.ag_inputs(W, M, K, N, salt=23)
    # two concurrent kernels must be co-resident: 2 x 32 workers x (up to) 2 CTAs <= 148 SMs
    ctxs, plans = _ag_world(ao, W, M, N, K, 128, backend, dir=dir_, n_cta=32)
    dA, dB = _dev(A), _dev(B)
    A64 = [si.to_f64(a) for a in A]
    streams = [torch.cuda.Stream() for _ in range(W)]
    for it in range(3):
        Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
        for r in (1, 0) if it % 2 else (0, 1):
            ao.ag_gemm(plans[r], dA[r], dB[r], Cs[r], stream=streams[r])
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_async()
        for r in range(W):
            _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag per-rank {backend} {dir_} it={it} r{r}")


def test_ag_gemm_pull_dedicated_comm_ctas(ao):
    W, M, K, N = 2, 1024, 256, 512
    A, B = si.ag_inputs(W, M, K, N, salt=29)
    ctxs, plans = _ag_world(ao, W, M, N, K, 128, "tma", dir="pull", tile_m=256, tile_n=256, n_cta=32,
                            comm_ctas=8, n_slices=4)
    Cs, G = _run_ag(ao, ctxs, plans, _dev(A), _dev(B), gather=True)
    A64 = [si.to_f64(a) for a in A]
    for r in range(W):
        _check(Cs[r], on.ag_gemm(A64, si.to_f64(B[r])), f"ag pull comm_ctas r{r}")
        assert torch.equal(G[r].cpu(), torch.cat(A, 0))


# ------------------------------------------------------------------------ GEMM-AR (NEXT-1)
def _ar_world(ao, W, M, N, K, chunk, **kw):
    desc = dict(op="gemm_ar", world_size=W, M=M, N=N, K=K, chunk_rows=chunk, backend="ldst", n_slices=4,
                n_cta=max(1, 148 // W), timeout_ns=2_000_000_000, **kw)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(desc))
    return ctxs, [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]


def _run_ar(ao, ctxs, plans, A, B):
    M, N = A[0].shape[0], B[0].shape[0]
    Cs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in plans]
    ao.gemm_ar_group(plans, A, B, Cs)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return Cs


@pytest.mark.parametrize("rs_reduce", ["atomic", "slots"])
@pytest.mark.parametrize("tile", [(128, 128), (256, 256)])
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_gemm_ar_vs_oracle(ao, W, tile, rs_reduce):
    """GEMM-AR: every rank's full C equals the fp64 sum of the partials (all rows)."""
    M, K, N, C = 256 * W, 256, 520, 64
    A, B = si.rs_inputs(W, M, K, N, salt=41)
    ctxs, plans = _ar_world(ao, W, M, N, K, C, tile_m=tile[0], tile_n=tile[1], rs_reduce=rs_reduce)
    dA, dB = _dev(A), _dev(B)
    ref = on.gemm_ar([si.to_f64(a) for a in A], [si.to_f64(b) for b in B])
    for it in range(2):  # both parities
        Cs = _run_ar(ao, ctxs, plans, dA, dB)
        for r in range(W):
            _check(Cs[r], ref, f"ar W={W} {rs_reduce} it={it} rank {r}")
        for r in range(1, W):  # the gathered rows are copies of the owners' rows: bit-identical
            assert torch.equal(Cs[r].cpu(), Cs[0].cpu())


@pytest.mark.parametrize("rs_reduce", ["atomic", "slots"])
def test_gemm_ar_bitmask_epochs_and_chunk_major(ao, rs_reduce):
    W, M, K, N = 4, 1024, 64, 256
    ctxs, plans = _ar_world(ao, W, M, N, K, 128, chunk_order="chunk_major", rs_reduce=rs_reduce)
    A, B = si.rs_provenance_inputs(W, M, K, N)
    dA, dB = _dev(A), _dev(B)
    for it in range(4):
        Cs = _run_ar(ao, ctxs, plans, dA, dB)
        for r in range(W):
            assert torch.all(Cs[r].float() == 2 ** W - 1), (it, r)


def test_gemm_ar_rejects_wrong_op_and_backend(ao):
    W, M, K, N = 2, 512, 64, 256
    ctxs, plans = _ar_world(ao, W, M, N, K, 64)
    A = [torch.zeros(M, K, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    B = [torch.zeros(N, K, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    C = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.gemm_rs_group(plans, A, B, C)  # an AR plan is not an RS plan
    with pytest.raises(ao.AOError, match="INVALID_ARG"):
        ao.Plan(ctxs[0], dict(plans[0].desc, backend="ce"))  # gather transport is ld/st


@pytest.mark.parametrize("backend", ["ce", "tma", "ldst"])
def test_transfer_bench_backends(ao, backend):
    """E4 microbenchmark entry point: every backend moves a message into a peer's symmetric
    buffer and reports a positive time (the AG tests check the same code's data)."""
    ctxs = ao.loopback_world(0, 2, 8 << 20)
    src = torch.zeros(1 << 21, dtype=torch.bfloat16, device="cuda")
    ms = ao.transfer_bench(ctxs[0], 1, backend, src, 4 << 20, 1 << 18, n_ctas=8, n_streams=2, iters=3)
    assert ms > 0
    for c in ctxs:
        c.close()
