"""Device time of rank 0's per-GPU TP=8 ops alone on the GPU (peers pre-arrived): AG
(8192 x 1792 x 4096, stream-K off / auto) and plain GEMM on the same shape; one JSON line."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, M, K, N = 8, 8192, 4096, 1792
A, B = si.ag_inputs(W, M, K, N)
A0, B0, Af = A[0].cuda(), B[0].cuda(), torch.cat(A, 0).cuda()
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")


def timed(fn, k=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return round(s.elapsed_time(e) / k, 4)


out = {}
for sk in (0, -1):
    d = dict(op="ag_gemm", world_size=W, rank=0, M=M, N=N, K=K, chunk_rows=1024, backend="ce", tile_m=256,
             tile_n=256, n_cta=148, stream_k=sk, intra="grouped", group_m=4, timeout_ns=5_000_000_000)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    p = ao.Plan(ctxs[0], d)
    ao.debug_set("prearrive", 1)
    out[f"ag_sk{sk}"] = timed(lambda: ao.ag_gemm(p, A0, B0, C))
    ao.debug_set("prearrive", 0)
    ao.debug_set("gemm_stream_k", sk)
    out[f"gemm_sk{sk}"] = timed(lambda: ao.gemm(Af, B0, C, tile_m=256, tile_n=256))
    ao.debug_set("gemm_stream_k", 0)
    p.close()
    for c in ctxs:
        c.close()
Bb = torch.cat([B0] * 8, 0)
Cb = torch.empty(M, 8 * N, dtype=torch.bfloat16, device="cuda")
out["gemm_big_8192x14336x4096"] = timed(lambda: ao.gemm(Af, Bb, Cb, tile_m=256, tile_n=256), 10)
print(json.dumps(out))
