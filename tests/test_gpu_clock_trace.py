"""The in-kernel clock instrument the bench's peak regime rests on (bench.kernel_clocks):
every MMA span of a traced fused launch emits a TR_CLK event whose id is the SM cycles
(clock64) over the span; cycles / ns must be a plausible SM clock (above the idle floor,
at most sm_max), and there is one clock event per MMA event."""
import json
import os

import pytest
import torch

from synthetic import inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def test_clock_events_per_mma_span(ao, tmp_path):
    W, M, K, N = 2, 1024, 2048, 1024
    d = dict(op="gemm_rs", world_size=W, M=M, N=N, K=K, chunk_rows=256, tile_m=256, tile_n=256, n_cta=32,
             rs_reduce="atomic", timeout_ns=2_000_000_000)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    pr = [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
    Ar, Br = si.rs_inputs(W, M, K, N, salt=5)
    A = [a.cuda() for a in Ar]
    B = [b.cuda() for b in Br]
    Ds = [torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    ctxs[0].trace_enable(1 << 16)
    for _ in range(3):
        ao.gemm_rs_group(pr, A, B, Ds)
    path = str(tmp_path / "t.json")
    ctxs[0].trace_dump(path)
    ctxs[0].trace_enable(0)
    ev = json.load(open(path))["traceEvents"]
    mma = [e for e in ev if e["cat"] == "mma"]
    clk = [e for e in ev if e["cat"] == "clock"]
    assert mma and len(clk) == len(mma)
    max_mhz = torch.cuda.get_device_properties(0).clock_rate / 1000 if hasattr(
        torch.cuda.get_device_properties(0), "clock_rate") else 1965
    for e in clk:
        if e["dur"] > 0.5:  # spans long enough for ns resolution
            mhz = int(e["name"].split()[1]) / e["dur"]
            assert 100 < mhz <= max(max_mhz, 1965) * 1.02, mhz
    for c in ctxs:
        c.check_async()
        c.close()
