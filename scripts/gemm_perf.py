"""Times the plain tcgen05 mainloop (ao.gemm) against cuBLAS (torch.matmul) on the
per-rank GEMM shapes of the benchmark.  Usage: python scripts/gemm_perf.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao


def bench(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


shapes = [(8192, 14336, 4096), (8192, 4096, 14336), (8192, 1792, 4096), (8192, 4096, 1792), (8192, 8192, 8192)]
for M, N, K in shapes:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    res = []
    for bm, bn in ((256, 256), (256, 128), (128, 256)):
        ms = bench(lambda: ao.gemm(A, B, C, tile_n=bn, tile_m=bm))
        res.append(f"ao {bm}x{bn}: {fl / ms / 1e9:7.1f} TF/s")
    ms = bench(lambda: torch.matmul(A, B.t(), out=C))
    res.append(f"cublas: {fl / ms / 1e9:7.1f} TF/s ({ms:.3f} ms)")
    print(f"{M}x{N}x{K}: " + " | ".join(res), flush=True)
