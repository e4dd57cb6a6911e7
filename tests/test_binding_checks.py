"""The Python binding's operand checks (no GPU): the kernels take every extent from the
plan, so the binding must refuse tensors whose shape disagrees with the plan's desc
before any pointer reaches the C ABI."""
import pytest
import torch

import paper_2601_20595_b200.api as api
from oracle import schedule as osch


def test_shape_mismatch_is_refused_before_the_abi():
    d = osch.default_desc(op="ag_gemm", world_size=2, rank=0, M=512, N=384, K=256, chunk_rows=64)
    p = api.Plan(None, d)
    W, M, N, K = api._op_shapes(p)
    ok = dict(A_shard=(torch.empty(M // W, K), (M // W, K)), B=(torch.empty(N, K), (N, K)),
              C=(torch.empty(M, N), (M, N)))
    api._expect(p, **ok)
    for name, bad in (("A_shard", torch.empty(M // W - 8, K)), ("B", torch.empty(N, K + 8)), ("C", torch.empty(M // W, N))):
        kw = dict(ok)
        kw[name] = (bad, kw[name][1])
        with pytest.raises(api.AOError) as ei:
            api._expect(p, **kw)
        assert ei.value.status == "AO_ERR_INVALID_ARG" and name in str(ei.value)
    p.close()


def test_expected_shapes_per_op():
    rs = api.Plan(None, osch.default_desc(op="gemm_rs", world_size=4, rank=1, M=1024, N=384, K=128, chunk_rows=64))
    assert api._op_shapes(rs) == (4, 1024, 384, 128)
    with pytest.raises(api.AOError):
        api._expect(rs, C_shard=(torch.empty(1024, 384), (1024 // 4, 384)))
    rs.close()
