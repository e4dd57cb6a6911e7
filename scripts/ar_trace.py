"""Trace a time-sliced GEMM-AR launch (Llama-3-8B down-proj, TP=8 loopback) at two chunk
sizes: per-role summaries and the comm (gather) item timeline."""
import sys
import os
import json
import subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, H, F = 8, 8192, 4096, 14336
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ar_trace"
A, B = si.rs_inputs(W, M, F // W, H)
dA, dB = [a.cuda() for a in A], [b.cuda() for b in B]
C = [torch.empty(M, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
base = dict(op="gemm_ar", world_size=W, M=M, N=H, K=F // W, intra="grouped", group_m=4, backend="ldst", n_slices=8,
            rs_reduce="atomic", tile_m=256, tile_n=256, n_cta=148, timeout_ns=5_000_000_000)
for c in (256, 1024):
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(dict(base, chunk_rows=c)))
    plans = [ao.Plan(ctxs[r], dict(base, rank=r, chunk_rows=c, chunk_order="chunk_major")) for r in range(W)]
    for _ in range(3):
        ao.gemm_ar_group(plans, dA, dB, C)
    torch.cuda.synchronize()
    ctxs[0].trace_enable(1 << 21)
    ao.gemm_ar_group(plans, dA, dB, C)
    ctxs[0].trace_dump(f"{out}_{c}.json")
    print(f"=== chunk {c}", flush=True)
    subprocess.run([sys.executable, "scripts/trace_summary.py", f"{out}_{c}.json"])
    ev = json.load(open(f"{out}_{c}.json"))["traceEvents"]
    t0 = min(e["ts"] for e in ev)
    comm = sorted((e["ts"] - t0, e["dur"]) for e in ev if e["cat"] == "comm")
    if comm:
        n = len(comm)
        for q in (0, n // 4, n // 2, 3 * n // 4, n - 1):
            print(f"  comm item #{q}: start {comm[q][0]:.1f} us dur {comm[q][1]:.1f} us")
    for p in plans:
        p.close()
    for x in ctxs:
        x.close()
