"""GEMM-AR (NEXT-1) configuration probe on the 8B down-proj shape, TP=8 loopback."""
import itertools
import sys

import torch

import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, H, F = 8, 8192, 4096, 14336
Fl = F // W
A, B = si.rs_inputs(W, M, Fl, H)
dA, dB = [a.cuda() for a in A], [b.cuda() for b in B]
C = [torch.empty(M, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
configs = [(c, o, ns, red) for c, o, ns, red in itertools.product((256, 512, 1024), ("shard_major", "chunk_major"),
                                                                   (8, 32), ("atomic",))]
base = dict(op="gemm_ar", world_size=W, M=M, N=H, K=Fl, intra="grouped", group_m=4, n_cta=148 // W, backend="ldst",
            timeout_ns=5_000_000_000)
ws = max(ao.workspace_bytes(dict(base, chunk_rows=c, rs_reduce=red)) for c, _, _, red in configs)
ctxs = ao.loopback_world(0, W, ws)
for c, o, ns, red in configs:
    plans = [ao.Plan(ctxs[r], dict(base, rank=r, chunk_rows=c, chunk_order=o, n_slices=ns, rs_reduce=red))
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
    print(f"chunk {c:5d} {o:12s} slices {ns:3d} {red:7s}: {ms:.4f} ms  {2 * M * F * H / ms / 1e9:.0f} TF/s",
          flush=True)
    for p in plans:
        p.close()
