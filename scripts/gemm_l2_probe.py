"""ao_gemm 8192x14336x4096 under a chosen GROUP_M / L2 policy (for ncu DRAM-byte probes).
usage: python scripts/gemm_l2_probe.py GROUP_M L2_HINT"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao

gm, hint = int(sys.argv[1]), int(sys.argv[2])
ao.debug_set("gemm_group_m", gm)
ao.debug_set("l2_hint", hint)
M, N, K = 8192, 14336, 4096
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ao.gemm(A, B, C)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ao.gemm(A, B, C)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"gm={gm} hint={hint}: {2 * M * N * K / ms / 1e9:.1f} TF/s")
