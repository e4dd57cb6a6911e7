"""Measures the plain-GEMM mainloop throughput of every tile candidate the planner knows
(through ao.gemm, i.e. the fused kernel with no communication) and writes
profiles/tile_eff.json -- the measurement the planner's TILE_EFF table (Q19) is
typed from.  Efficiency of a shape = its TFLOP/s on a problem with ~55 waves of its own
tiles and no ragged edge (M = 16384, N = 64 * BN, K = 4096; wave quantization < 2 %),
relative to the 2-CTA 256 x 256 tile.  Also times every shape on the per-GPU TP shapes
of the benchmark (reported, not used by the planner) and checks each result against
torch.matmul.  Usage: python scripts/measure_tile_eff.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao

SHAPES = [(256, 256), (256, 128), (128, 256), (128, 128), (256, 224), (256, 208), (256, 192), (256, 160),
          (256, 144), (256, 112), (512, 256)]
PER_RANK = {"ag_w8": (8192, 1792, 4096), "ag_w4": (8192, 3584, 4096), "ag_w2": (8192, 7168, 4096),
            "rs_w8": (8192, 4096, 1792)}


def bench(fn, n=20, reps=3):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / n)
    return best


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/tile_eff.json"
    torch.manual_seed(0)
    res = {"how": "ao.gemm TFLOP/s, best of 3 x 20 launches after 3 warm-up (CUDA events); "
                  "eff on M=16384, N=64*BN, K=4096", "tflops": {}, "per_rank": {}}
    for bm, bn in SHAPES:
        M, N, K = 16384 * (2 if bm == 512 else 1), 64 * bn, 4096
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = (torch.randn(N, K, device="cuda") / 64).bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ao.gemm(A, B, C, tile_m=bm, tile_n=bn)
        ref = (A.float() @ B.float().t())
        err = ((C.float() - ref).norm() / ref.norm()).item()
        assert err < 4e-3, (bm, bn, err)
        ms = bench(lambda: ao.gemm(A, B, C, tile_m=bm, tile_n=bn))
        res["tflops"][f"{bm}x{bn}"] = round(2.0 * M * N * K / ms / 1e9, 1)
        print(bm, bn, res["tflops"][f"{bm}x{bn}"], f"frob {err:.2e}", flush=True)
        del A, B, C, ref
    base = res["tflops"]["256x256"]
    res["eff_pct"] = {k: int(round(100 * v / base)) for k, v in res["tflops"].items()}
    for name, (M, N, K) in PER_RANK.items():
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = (torch.randn(N, K, device="cuda") / 64).bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        row = {}
        for bm, bn in SHAPES:
            ms = bench(lambda: ao.gemm(A, B, C, tile_m=bm, tile_n=bn))
            row[f"{bm}x{bn}"] = round(2.0 * M * N * K / ms / 1e9, 1)
        ms = bench(lambda: torch.matmul(A, B.t(), out=C))
        row["cublas"] = round(2.0 * M * N * K / ms / 1e9, 1)
        res["per_rank"][name] = row
        print(name, row, flush=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res["eff_pct"]))


if __name__ == "__main__":
    main()
