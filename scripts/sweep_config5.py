"""BASELINE config 5: chunk-size x backend sweep on Llama-3-70B TP=8 AG-GEMM shapes
(§6 Fig.11a/b ablation, reading Q5: M = 32768
tokens so S = 4096 rows per rank and chunk sizes 64..4096 rows = 1..64 MiB).

Loopback world of W = 8 ranks on one GPU (one fused launch per op), measured through the
tuner's timing path.  Writes one JSON line per point to the given file and a table to stdout.
usage: python scripts/sweep_config5.py OUT.jsonl [--tokens 32768]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2601_20595_b200 import tune  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--tokens", type=int, default=32768)
ap.add_argument("--budget", type=float, default=900.0)
ap.add_argument("--no-e4", action="store_true", help="measure every backend (no E4-seeded pruning)")
a = ap.parse_args()
W, HIDDEN, FFN = 8, 8192, 28672
M, N, K = a.tokens, FFN // W, HIDDEN
S = M // W
chunks = [c for c in (64, 128, 256, 512, 1024, 2048, 4096) if c <= S and S % c == 0]
space = tune.candidate_space("ag_gemm", W, M, N, K, chunks=chunks, backends=["ce", "tma", "ldst"],
                             intras=[("grouped", 4)], tiles=[(256, 256)], dirs=["push"], scheds=["space", "time"],
                             comm_ctas=[0], slices=[2])
rows, pruned = tune.tune_loopback("ag_gemm", W, M, N, K, budget_s=a.budget, warmup=2, iters=10, space=space,
                                  use_e4=not a.no_e4)
with open(a.out, "w") as f:
    for r in rows:
        d = r["desc"]
        f.write(json.dumps({"chunk_rows": d["chunk_rows"], "chunk_mib": d["chunk_rows"] * K * 2 / 2**20,
                            "backend": d["backend"], "sched": d["sched"], "ms": round(r["ms"], 4),
                            "tflops": round(r["tflops"], 1), "tile": r["tile"]}) + "\n")
    for d, why in pruned:
        f.write(json.dumps({"chunk_rows": d["chunk_rows"], "backend": d["backend"], "pruned": why}) + "\n")
by = {(r["desc"]["chunk_rows"], r["desc"]["backend"], r["desc"]["sched"]): r["tflops"] for r in rows}
cols = [("ce", "time"), ("ce", "space"), ("tma", "space"), ("ldst", "space")]
print(f"config 5 loopback W={W} M={M} N={N}/rank K={K}: TFLOP/s (all 8 ranks)")
print("chunk rows  MiB   " + "  ".join(f"{b + '/' + s:>10s}" for b, s in cols))
for c in chunks:
    print(f"{c:10d} {c * K * 2 / 2**20:5.0f}  " + "  ".join(
        f"{by.get((c, b, s), float('nan')):10.0f}" for b, s in cols))
for d, why in pruned:
    print("pruned", d["chunk_rows"], d["backend"], why)
