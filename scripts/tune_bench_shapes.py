"""Auto-tuner (NEXT-2) over the bench's Llama-3-8B TP=8 FFN shapes, both loopback
group schedules (Q24): chunk rows x intra order x RS chunk order x schedule, tile
256x256.  usage: python scripts/tune_bench_shapes.py OUT_PREFIX   (writes OUT_{ag,rs}.jsonl)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20595_b200 import tune  # noqa: E402

pre = sys.argv[1]
W, M, H, F = 8, 8192, 4096, 14336
for op, N, K in (("ag_gemm", F // W, H), ("gemm_rs", H, F // W)):
    space = tune.candidate_space(op, W, M, N, K, chunks=[256, 512, 1024], backends=["ce"],
                                 intras=[("row", 1), ("grouped", 4), ("grouped", 8)], tiles=[(256, 256)],
                                 dirs=["push"], scheds=["space", "time"])
    if op == "gemm_rs":
        for d in space:
            d["rs_reduce"] = "atomic"
    rows, pruned = tune.tune_loopback(op, W, M, N, K, budget_s=600, warmup=3, iters=10, space=space)
    with open(f"{pre}_{'ag' if op == 'ag_gemm' else 'rs'}.jsonl", "w") as f:
        for r in rows:
            d = r["desc"]
            f.write(json.dumps({"ms": round(r["ms"], 4), "tflops": round(r["tflops"], 1), "tile": r["tile"],
                                "cfg": {k: d.get(k) for k in ("chunk_rows", "backend", "intra", "group_m",
                                                              "chunk_order", "sched", "rs_reduce")}}) + "\n")
    print(op, "best:", json.dumps({k: rows[0][k] for k in ("ms", "tflops")} | {"sched": rows[0]["desc"]["sched"],
          "chunk": rows[0]["desc"]["chunk_rows"], "intra": rows[0]["desc"]["intra"], "gm": rows[0]["desc"]["group_m"],
          "order": rows[0]["desc"]["chunk_order"]}), "measured", len(rows), "pruned", len(pruned))
