"""Trace the per-rank TP=8 AG (rank 0 alone, peers pre-arrived) with and without the
stream-K tail; prints per-role summaries (scripts/trace_summary.py) and the time."""
import sys
import os
import subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, K, N = 8, 8192, 4096, 1792
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sk_trace"
A, B = si.ag_inputs(W, M, K, N)
A0, B0 = A[0].cuda(), B[0].cuda()
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for sk in (0, 1):
    d = dict(op="ag_gemm", world_size=W, rank=0, M=M, N=N, K=K, chunk_rows=1024, backend="ce", tile_m=256,
             tile_n=256, n_cta=148, stream_k=sk, intra="grouped", group_m=4, timeout_ns=5_000_000_000)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    p = ao.Plan(ctxs[0], d)
    ao.debug_set("prearrive", 1)
    for _ in range(5):
        ao.ag_gemm(p, A0, B0, C)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        ao.ag_gemm(p, A0, B0, C)
    e.record()
    torch.cuda.synchronize()
    print(f"stream_k={sk}: {s.elapsed_time(e) / 20:.4f} ms", flush=True)
    ctxs[0].trace_enable(1 << 20)
    for _ in range(2):
        ao.ag_gemm(p, A0, B0, C)
    ctxs[0].trace_dump(f"{out}_{sk}.json")
    ctxs[0].trace_enable(0)
    ao.debug_set("prearrive", 0)
    p.close()
    for c in ctxs:
        c.close()
    subprocess.run([sys.executable, "scripts/trace_summary.py", f"{out}_{sk}.json"])
