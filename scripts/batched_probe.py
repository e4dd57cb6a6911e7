"""Probe ao_gemm_batched vs ao_gemm: device time per call and host time per call."""
import time

import torch

import paper_2601_20595_b200 as ao


def t(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    s.record()
    for _ in range(k):
        fn()
    e.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k, (h1 - h0) * 1e3 / k


M, H, F = 8192, 4096, 1792
A = [torch.randn(M, H, device="cuda").to(torch.bfloat16) for _ in range(8)]
B = [torch.randn(F, H, device="cuda").to(torch.bfloat16) for _ in range(8)]
C = [torch.empty(M, F, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
print("ao_gemm 256x256: dev %.4f host %.4f ms" % t(lambda: ao.gemm(A[0], B[0], C[0], 256, 256)))
for n, ncta, gm in ((1, 0, 16), (1, 18, 16), (8, 18, 4), (8, 18, 16), (8, 18, 64)):
    print(f"batched n={n} n_cta={ncta} gm={gm}: dev %.4f host %.4f ms" %
          t(lambda: ao.gemm_batched(A[:n], B[:n], C[:n], 256, 256, gm, ncta)), flush=True)
