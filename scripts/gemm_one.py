"""One plain-GEMM configuration through ao.gemm, a few launches (for ncu captures).
usage: python scripts/gemm_one.py M N K BM BN [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao

M, N, K, bm, bn = (int(x) for x in sys.argv[1:6])
it = int(sys.argv[6]) if len(sys.argv) > 6 else 3
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(it):
    ao.gemm(A, B, C, tile_m=bm, tile_n=bn)
torch.cuda.synchronize()
print("ok", M, N, K, bm, bn)
