"""GEMM-AR (NEXT-1) probe, Llama-3-8B down-proj at TP=8 in loopback: space- vs time-sliced
groups x chunk rows x chunk order (device time per call, CUDA events)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, H, F = 8, 8192, 4096, 14336
Fl = F // W
A, B = si.rs_inputs(W, M, Fl, H)
dA, dB = [a.cuda() for a in A], [b.cuda() for b in B]
C = [torch.empty(M, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
import os as _os
configs = [("space", 256, "chunk_major", 8), ("time", 256, "chunk_major", 8), ("time", 1024, "shard_major", 8),
           ("time", 256, "shard_major", 8), ("space", 1024, "shard_major", 8)]
if _os.environ.get("AR_SLICES"):
    configs = [("time", c, o, int(ns)) for ns in _os.environ["AR_SLICES"].split(",")
               for c, o in ((256, "chunk_major"), (128, "chunk_major"), (512, "chunk_major"))]
base = dict(op="gemm_ar", world_size=W, M=M, N=H, K=Fl, intra="grouped", group_m=4, backend="ldst",
            rs_reduce="atomic", tile_m=256, tile_n=256, timeout_ns=5_000_000_000)
ws = max(ao.workspace_bytes(dict(base, chunk_rows=c, n_slices=ns)) for _, c, _, ns in configs)
ctxs = ao.loopback_world(0, W, ws)
for sched, c, o, ns in configs:
    nc = 148 if sched == "time" else 148 // W // 2 * 2
    plans = [ao.Plan(ctxs[r], dict(base, rank=r, chunk_rows=c, chunk_order=o, n_cta=nc, n_slices=ns))
             for r in range(W)]
    for _ in range(3):
        ao.gemm_ar_group(plans, dA, dB, C)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        ao.gemm_ar_group(plans, dA, dB, C)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{sched:5s} chunk {c:5d} {o:12s} slices {ns:3d}: {ms:.4f} ms  {2 * M * F * H / ms / 1e9:.0f} TF/s",
          flush=True)
    for p in plans:
        p.close()
