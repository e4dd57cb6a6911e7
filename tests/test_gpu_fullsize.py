"""Full-size parity in the exact launch configuration bench.py times: Llama-3-8B FFN at
TP=8 (8192 tokens, hidden 4096, ffn 14336), 8 loopback ranks, CE backend, chunk = shard,
GROUP_M 4, shard-major RS with the atomic (TMA reduce-add) reduction bench.py uses (and the
deterministic slots mode), heuristic tile (256x256 CTA pairs).  Plus BASELINE config 5's
Llama-3-70B TP=8 AG-GEMM shape (M = 32768, reading Q5) at a mid-sweep chunk size.  The oracle computes sampled
output rows one by one (every chunk-boundary row + seeded random rows of every rank);
tolerance as in BASELINE.json."""
import numpy as np
import pytest
import torch

from oracle import numeric as on
from synthetic import inputs as si

pytestmark = pytest.mark.gpu

W, M, H, F = 8, 8192, 4096, 14336


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _rows(S, chunk, rng, extra=6):
    rows = set()
    for g0 in range(0, S, chunk):
        rows.update((g0, g0 + chunk - 1))
    rows.update(rng.integers(0, S, size=extra).tolist())
    return np.array(sorted(rows))


def _worlds(ao, rs_reduce):
    Fl = F // W
    base = dict(world_size=W, M=M, chunk_rows=1024, intra="grouped", group_m=4, n_cta=148 // W,
                timeout_ns=5_000_000_000)
    ag = dict(base, op="ag_gemm", N=Fl, K=H, backend="ce", n_slices=2)
    rs = dict(base, op="gemm_rs", N=H, K=Fl, chunk_order="shard_major", rs_reduce=rs_reduce)
    ctxs = ao.loopback_world(0, W, max(ao.workspace_bytes(ag), ao.workspace_bytes(rs)))
    pa = [ao.Plan(ctxs[r], dict(ag, rank=r)) for r in range(W)]
    pr = [ao.Plan(ctxs[r], dict(rs, rank=r)) for r in range(W)]
    return ctxs, pa, pr


@pytest.mark.parametrize("rs_reduce", ["atomic", "slots"])
def test_fullsize_ag_and_rs_sampled_vs_oracle(ao, rs_reduce):
    Fl = F // W
    S = M // W
    ctxs, pa, pr = _worlds(ao, rs_reduce)
    assert pa[0].info()["tile_m"] == 256 and pa[0].info()["tile_n"] == 256
    rng = np.random.default_rng(123)

    A, Bu = si.ag_inputs(W, M, H, Fl)
    dA, dBu = [a.cuda() for a in A], [b.cuda() for b in Bu]
    Cu = [torch.empty(M, Fl, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for _ in range(2):  # second call runs on the other epoch parity
        ao.ag_gemm_group(pa, dA, dBu, Cu)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    A64 = [si.to_f64(a) for a in A]
    for r in range(W):
        rows = _rows(M, 1024, rng)
        ref = on.ag_gemm_rows(A64, si.to_f64(Bu[r]), rows)
        ok, e, f = on.check_tolerance(Cu[r][torch.as_tensor(rows)].float().cpu().numpy(), ref)
        assert ok, f"AG rank {r}: elem {e:.3e} frob {f:.3e}"
    del dA, dBu, Cu, A64

    Ar, Bd = si.rs_inputs(W, M, Fl, H)
    dAr, dBd = [a.cuda() for a in Ar], [b.cuda() for b in Bd]
    Cd = [torch.empty(S, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for _ in range(2):
        ao.gemm_rs_group(pr, dAr, dBd, Cd)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    Bd64 = [si.to_f64(b) for b in Bd]
    for r in range(W):
        local = _rows(S, 64, rng, extra=24)
        grows = r * S + local
        A_rows = [si.to_f64(Ar[s][torch.as_tensor(grows)]) for s in range(W)]
        ref = on.gemm_rs_from_rows(A_rows, Bd64)
        ok, e, f = on.check_tolerance(Cd[r][torch.as_tensor(local)].float().cpu().numpy(), ref)
        assert ok, f"RS rank {r}: elem {e:.3e} frob {f:.3e}"


@pytest.mark.parametrize("W2", [3, 5, 6, 7])
def test_non_power_of_two_worlds(ao, W2):
    """W that does not divide the SM count or the tile grid evenly: AG + RS tiny shapes."""
    Ml, K, N = 256 * W2, 192, 264
    A, B = si.ag_inputs(W2, Ml, K, N, salt=W2)
    desc = dict(op="ag_gemm", world_size=W2, M=Ml, N=N, K=K, chunk_rows=64, n_cta=148 // W2,
                backend="tma", n_slices=2, timeout_ns=2_000_000_000)
    rsd = dict(op="gemm_rs", world_size=W2, M=Ml, N=N, K=K, chunk_rows=64, n_cta=148 // W2,
               timeout_ns=2_000_000_000)
    ctxs = ao.loopback_world(0, W2, max(ao.workspace_bytes(desc), ao.workspace_bytes(rsd)))
    pa = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W2)]
    pr = [ao.Plan(ctxs[r], dict(rsd, rank=r)) for r in range(W2)]
    Cs = [torch.empty(Ml, N, dtype=torch.bfloat16, device="cuda") for _ in range(W2)]
    ao.ag_gemm_group(pa, [a.cuda() for a in A], [b.cuda() for b in B], Cs)
    Ar, Br = si.rs_inputs(W2, Ml, K, N, salt=W2)
    Ds = [torch.empty(Ml // W2, N, dtype=torch.bfloat16, device="cuda") for _ in range(W2)]
    ao.gemm_rs_group(pr, [a.cuda() for a in Ar], [b.cuda() for b in Br], Ds)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    A64 = [si.to_f64(a) for a in A]
    Ar64, Br64 = [si.to_f64(a) for a in Ar], [si.to_f64(b) for b in Br]
    for r in range(W2):
        ok, e, f = on.check_tolerance(Cs[r].float().cpu().numpy(), on.ag_gemm(A64, si.to_f64(B[r])))
        assert ok, f"AG W={W2} r{r}: {e:.3e} {f:.3e}"
        ok, e, f = on.check_tolerance(Ds[r].float().cpu().numpy(), on.gemm_rs(Ar64, Br64, r))
        assert ok, f"RS W={W2} r{r}: {e:.3e} {f:.3e}"


@pytest.mark.parametrize("backend", ["tma", "ce"])
def test_config5_70b_ag_sampled_vs_oracle(ao, backend):
    """Llama-3-70B TP=8 up-proj: M = 32768 tokens, K = 8192, N = 28672/8 per rank, 256-row
    chunks (4 MiB), 8 loopback ranks; sampled rows (chunk boundaries + random) of 3 ranks."""
    W5, M5, K5, N5 = 8, 32768, 8192, 28672 // 8
    desc = dict(op="ag_gemm", world_size=W5, M=M5, N=N5, K=K5, chunk_rows=256, backend=backend, n_slices=2,
                intra="grouped", group_m=4, n_cta=148 // W5, timeout_ns=10_000_000_000)
    ctxs = ao.loopback_world(0, W5, ao.workspace_bytes(desc))
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W5)]
    A, B = si.ag_inputs(W5, M5, K5, N5, salt=5)
    dA, dB = [a.cuda() for a in A], [b.cuda() for b in B]
    C = [torch.empty(M5, N5, dtype=torch.bfloat16, device="cuda") for _ in range(W5)]
    ao.ag_gemm_group(plans, dA, dB, C)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    rng = np.random.default_rng(5)
    A64 = [si.to_f64(a) for a in A]
    for r in (0, 3, 7):
        rows = _rows(M5, 4096, rng, extra=8)
        ref = on.ag_gemm_rows(A64, si.to_f64(B[r]), rows)
        ok, e, f = on.check_tolerance(C[r][torch.as_tensor(rows)].float().cpu().numpy(), ref)
        assert ok, f"config5 {backend} rank {r}: elem {e:.3e} frob {f:.3e}"


@pytest.mark.parametrize("sched", ["space", "time"])
def test_fullsize_gemm_ar_sampled_vs_oracle(ao, sched):
    """GEMM-AR (NEXT-1) on the down-proj shape at TP=8: space-sliced (1024-row chunks) and the
    bench's time-sliced configuration (all SMs per rank, 256-row chunks in chunk-major order,
    256x256 tiles, the peer-grouped gather walk); every rank's full [M, hidden] output,
    sampled rows of every owner block on 3 ranks."""
    Fl, S = F // W, M // W
    desc = dict(op="gemm_ar", world_size=W, M=M, N=H, K=Fl, chunk_rows=1024, intra="grouped", group_m=4,
                n_cta=148 // W, backend="ldst", n_slices=8, rs_reduce="atomic", timeout_ns=5_000_000_000)
    if sched == "time":
        desc.update(n_cta=148, chunk_rows=256, chunk_order="chunk_major", tile_m=256, tile_n=256)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(desc))
    plans = [ao.Plan(ctxs[r], dict(desc, rank=r)) for r in range(W)]
    Ar, Bd = si.rs_inputs(W, M, Fl, H)
    dA, dB = [a.cuda() for a in Ar], [b.cuda() for b in Bd]
    C = [torch.empty(M, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for _ in range(2):
        ao.gemm_ar_group(plans, dA, dB, C)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    rng = np.random.default_rng(77)
    Bd64 = [si.to_f64(b) for b in Bd]
    rows = np.concatenate([o * S + _rows(S, 512, rng, extra=2) for o in range(W)])
    A_rows = [si.to_f64(Ar[s][torch.as_tensor(rows)]) for s in range(W)]
    ref = on.gemm_rs_from_rows(A_rows, Bd64)  # sum_s A_s[rows] . B_s^T, ascending s
    for r in (0, 3, 7):
        ok, e, f = on.check_tolerance(C[r][torch.as_tensor(rows)].float().cpu().numpy(), ref)
        assert ok, f"AR rank {r}: elem {e:.3e} frob {f:.3e}"
