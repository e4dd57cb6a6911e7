"""Why the e2e step's compute slows while its PCIe copies run: the bench's loopback TP=8 FFN
step back to back (a) alone, (b) beside 64 MB H2D + 64 MB D2H per step on two copy streams,
(c) beside the same bytes as device-to-device copies (SM copy kernels, same HBM/L2 traffic, no
PCIe), (d) beside H2D only.  Prints the median step span on the compute stream.
usage: python scripts/e2e_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, H, FF = 8, 8192, 4096, 14336
F = FF // W
base = dict(world_size=W, M=M, chunk_rows=1024, timeout_ns=5_000_000_000, intra="grouped", group_m=4,
            n_cta=148, tile_m=256, tile_n=256)
ag = dict(base, op="ag_gemm", N=F, K=H, backend="ce", dir="push", n_slices=2)
rs = dict(base, op="gemm_rs", N=H, K=F, chunk_order="shard_major", rs_reduce="atomic")
ctxs = ao.loopback_world(0, W, max(ao.workspace_bytes(ag), ao.workspace_bytes(rs)))
pa = [ao.Plan(ctxs[r], dict(ag, rank=r)) for r in range(W)]
pr = [ao.Plan(ctxs[r], dict(rs, rank=r)) for r in range(W)]
A_cpu, Bu_cpu = si.ag_inputs(W, M, H, F)
Bd_cpu = si.rs_weights(W, F, H)
A = [a.cuda() for a in A_cpu]
Bu = [b.cuda() for b in Bu_cpu]
Bd = [b.cuda() for b in Bd_cpu]
Cu = [torch.empty(M, F, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
Cd = [torch.empty(M // W, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
stream = torch.cuda.current_stream()
hbuf = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
hbuf2 = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
dbuf = [torch.empty(64 << 20, dtype=torch.uint8, device="cuda") for _ in range(4)]
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def step():
    ao.ag_gemm_group(pa, A, Bu, Cu)
    ao.gemm_rs_group(pr, Cu, Bd, Cd)


def run(mode, n=30):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    for i in range(n):
        if mode in ("pcie", "h2d"):
            with torch.cuda.stream(up):
                dbuf[0].copy_(hbuf, non_blocking=True)
        if mode == "pcie":
            with torch.cuda.stream(down):
                hbuf2.copy_(dbuf[1], non_blocking=True)
        if mode == "d2d":
            with torch.cuda.stream(up):
                dbuf[0].copy_(dbuf[2], non_blocking=True)
            with torch.cuda.stream(down):
                dbuf[1].copy_(dbuf[3], non_blocking=True)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
        # keep the copies in step with the compute (one set per step)
        up.wait_stream(stream)
        down.wait_stream(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs[3:])


def clock(mode):
    """median in-kernel SM clock (TR_CLK events) over 6 steps in this mode"""
    import json
    import tempfile
    ctxs[0].trace_enable(1 << 21)
    run(mode, n=6)
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    ctxs[0].trace_dump(path)
    ctxs[0].trace_enable(0)
    ev = json.load(open(path))["traceEvents"]
    os.unlink(path)
    mhz = [int(e["name"].split()[1]) / e["dur"] for e in ev if e["cat"] == "clock" and e["dur"] > 0]
    return statistics.median(mhz) if mhz else float("nan")


for _ in range(5):
    step()
for rep in range(2):
    for mode in ("alone", "pcie", "d2d", "h2d"):
        print(f"{mode:6s} step span {run(mode):.4f} ms, in-kernel SM clock {clock(mode):.0f} MHz", flush=True)
for c in ctxs:
    c.check_async()
