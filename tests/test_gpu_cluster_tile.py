"""GPU parity of the 512-row cluster tile (two CTA pairs stacked along M, each CTA TMA-
multicasting a quarter of the tile's B rows to both pairs) vs the fp64
oracle / fp32 reference: plain GEMM, AG-GEMM (copy engine), GEMM-RS and GEMM-AR (atomic
reduction), space- and time-sliced, with the provenance patterns bit-exact."""
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


@pytest.fixture(scope="module")
def n4(ao):
    n = ao.device_query(0, "cluster4_ctas")
    assert n >= 4 and n % 4 == 0 and n <= SMS
    return n


def _dev(ts):
    return [t.cuda() for t in ts]


@pytest.mark.parametrize("M,N,K", [(1024, 256, 64), (2048, 1000, 520), (8192, 1792, 4096)])
def test_gemm_cluster_tile_vs_fp32(ao, M, N, K):
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).bfloat16().cuda()
    B = (torch.randn(N, K, generator=g) / K ** 0.5).bfloat16().cuda()
    C = ao.gemm(A, B, tile_m=512, tile_n=256)
    ref = (A.double() @ B.double().t()).cpu().numpy()
    ok, e, f = on.check_tolerance(C.float().cpu().numpy(), ref)
    assert ok, (e, f)


@pytest.mark.parametrize("ts", [False, True])
@pytest.mark.parametrize("W", [2, 4])
def test_ag_rs_ar_cluster_tile_vs_oracle(ao, n4, W, ts):
    M, K, N, C = 512 * W, 256, 776, 256
    per = n4 if ts else (n4 // W) // 4 * 4
    base = dict(world_size=W, M=M, chunk_rows=C, tile_m=512, tile_n=256, n_cta=per, timeout_ns=2_000_000_000)
    d_ag = dict(base, op="ag_gemm", N=N, K=K, backend="ce")
    d_rs = dict(base, op="gemm_rs", N=N, K=K, rs_reduce="atomic")
    d_ar = dict(base, op="gemm_ar", N=N, K=K, rs_reduce="atomic", backend="ldst", n_slices=2)
    ws = max(ao.workspace_bytes(d) for d in (d_ag, d_rs, d_ar))
    ctxs = ao.loopback_world(0, W, ws)
    pa = [ao.Plan(ctxs[r], dict(d_ag, rank=r)) for r in range(W)]
    pr = [ao.Plan(ctxs[r], dict(d_rs, rank=r)) for r in range(W)]
    pc = [ao.Plan(ctxs[r], dict(d_ar, rank=r)) for r in range(W)]
    assert pa[0].info()["tile_m"] == 512 and pa[0].info()["cta_group"] == 4
    if ts:
        assert '"time_sliced"' in ao.group_schedule_json(pa, SMS)
    A, B = si.ag_inputs(W, M, K, N, salt=81)
    Cs = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.ag_gemm_group(pa, _dev(A), _dev(B), Cs)
    Ar, Br = si.rs_inputs(W, M, K, N, salt=82)
    Ds = [torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.gemm_rs_group(pr, _dev(Ar), _dev(Br), Ds)
    Es = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ao.gemm_ar_group(pc, _dev(Ar), _dev(Br), Es)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    A64 = [si.to_f64(a) for a in A]
    Ar64, Br64 = [si.to_f64(a) for a in Ar], [si.to_f64(b) for b in Br]
    full = on.gemm_ar(Ar64, Br64)
    for r in range(W):
        ok, e, f = on.check_tolerance(Cs[r].float().cpu().numpy(), on.ag_gemm(A64, si.to_f64(B[r])))
        assert ok, f"ag r{r}: {e:.3e} {f:.3e}"
        ok, e, f = on.check_tolerance(Ds[r].float().cpu().numpy(), on.gemm_rs(Ar64, Br64, r))
        assert ok, f"rs r{r}: {e:.3e} {f:.3e}"
        ok, e, f = on.check_tolerance(Es[r].float().cpu().numpy(), full)
        assert ok, f"ar r{r}: {e:.3e} {f:.3e}"
    # provenance over back-to-back epochs: AG row ids / epochs, RS bitmask
    for it in range(3):
        Ap, Bp = si.ag_provenance_inputs(W, M, K, N, epoch=it + 7)
        ao.ag_gemm_group(pa, _dev(Ap), _dev(Bp), Cs)
        torch.cuda.synchronize()
        for r in range(W):
            c = Cs[r].float().cpu()
            rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
            assert torch.equal(rid, torch.arange(M, dtype=torch.float32)) and torch.all(c[:, 3] == (it + 7) % 32)
    Ap, Bp = si.rs_provenance_inputs(W, M, K, N)
    for it in range(3):
        ao.gemm_rs_group(pr, _dev(Ap), _dev(Bp), Ds)
        torch.cuda.synchronize()
        for r in range(W):
            assert torch.all(Ds[r].float().cpu() == 2 ** W - 1), (it, r)
    for c in ctxs:
        c.check_async()
        c.close()
