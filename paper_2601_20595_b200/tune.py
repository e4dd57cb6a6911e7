"""Communication-centric auto-tuning (§5.3).

"AutoOverlap automatically generates all valid implementations, measures their end-to-end
performance, and selects the best-performing backend for each operator and hardware
configuration".  The search space is the paper's:
  * inter-chunk: chunk size (split factor) per logical transfer;
  * intra-chunk: transfer backend, tile configuration, intra-chunk tile order;
  * AG-GEMM: transfer direction, push or pull ("different implementation choices
    during lowering");
  * GEMM-RS: chunk order of the owner rotation.
Candidates are pruned by the planner's validation (hardware constraints: alignment, tile
fit) and by a minimum efficient transfer size for the copy engine ("minimum
efficient transfer size for copy engines"), then timed with CUDA events on the launch
configuration they would run in (loopback world on this GPU, or the caller's world).

Host logic only: every candidate runs through the C ABI like a user call.
"""
from __future__ import annotations

import itertools
import time

from . import api

# a copy-engine launch costs ~2-3 us; below ~1 MiB a transfer cannot amortise it.
CE_MIN_CHUNK_BYTES = 1 << 20


def candidate_space(op: str, W: int, M: int, N: int, K: int, chunks=None, backends=None, intras=None,
                    tiles=None, orders=None, dirs=None, scheds=None):
    """Enumerate descs of one op (dicts with the oracle/planner desc keys).  `scheds`
    (optional) adds the loopback group schedule as key "sched": "space" (SMs/W CTAs per
    rank, ranks concurrent) or "time" (every rank over all SMs, Q24)."""
    S = M // W
    chunks = chunks or [c for c in (128, 256, 512, 1024, 2048, 4096) if c <= S and S % c == 0]
    backends = backends or (["ce", "tma", "ldst"] if op == "ag_gemm" and W > 1 else ["ce"])
    intras = intras or [("row", 1), ("grouped", 2), ("grouped", 4)]
    tiles = tiles or [(0, 0), (128, 256)]
    orders = orders or (["shard_major", "chunk_major"] if op == "gemm_rs" else ["shard_major"])
    dirs = dirs or (["push", "pull"] if op == "ag_gemm" and W > 1 else ["push"])
    out = []
    for c, b, (intra, gm), (tm, tn), o, dr in itertools.product(chunks, backends, intras, tiles, orders, dirs):
        d = dict(op=op, world_size=W, M=M, N=N, K=K, chunk_rows=c, backend=b, intra=intra, group_m=gm,
                 tile_m=tm, tile_n=tn, chunk_order=o, dir=dr, n_slices=2)
        for sc in (scheds or [None]):
            out.append(d if sc is None else dict(d, sched=sc))
    return out


def prune(descs, sm_count: int = 148):
    """(kept, pruned) with reasons: planner validation, CE minimum efficient size."""
    kept, pruned = [], []
    for d in descs:
        v = api.validate(dict(d, rank=0), sm_count)
        if v:
            pruned.append((d, "invalid: " + ";".join(v)))
            continue
        if d.get("sched") == "time" and not (d["op"] == "gemm_rs" or (d["backend"] == "ce" and d["dir"] == "push")):
            pruned.append((d, "invalid: time-sliced groups need copy-engine push (AG) or GEMM-RS"))
            continue
        if d["op"] == "ag_gemm" and d["backend"] == "ce" and d["world_size"] > 1:
            if d["chunk_rows"] * d["K"] * 2 < CE_MIN_CHUNK_BYTES:
                pruned.append((d, "inefficient: CE chunk below %d bytes" % CE_MIN_CHUNK_BYTES))
                continue
        kept.append(d)
    return kept, pruned


def _time_loopback(desc, W, device, A, B, C, warmup, iters, n_cta):
    import torch
    d = dict(desc, n_cta=n_cta, timeout_ns=5_000_000_000)
    ctxs = api.loopback_world(device, W, api.workspace_bytes(d))
    try:
        plans = [api.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
        fn = (lambda: api.ag_gemm_group(plans, A, B, C)) if d["op"] == "ag_gemm" else \
            (lambda: api.gemm_rs_group(plans, A, B, C))
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_async()
        ms = s.elapsed_time(e) / iters
        info = plans[0].info()
        for p in plans:
            p.close()
        return ms, info
    finally:
        for c in ctxs:
            c.close()


def tune_loopback(op: str, W: int, M: int, N: int, K: int, device: int = 0, budget_s: float = 120.0,
                  warmup: int = 2, iters: int = 5, space=None, log=None):
    """Measure every kept candidate of `op` in a W-rank loopback world on `device` and
    return rows sorted by time: [{desc, ms, tflops, tile}] + the pruned list."""
    import torch

    from synthetic import inputs as si
    torch.cuda.set_device(device)
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    descs = space if space is not None else candidate_space(op, W, M, N, K)
    kept, pruned = prune(descs, sms // W)
    if op == "ag_gemm":
        A, B = si.ag_inputs(W, M, K, N)
        A = [a.cuda() for a in A]
        B = [b.cuda() for b in B]
        C = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    else:
        A, B = si.rs_inputs(W, M, K, N)
        A = [a.cuda() for a in A]
        B = [b.cuda() for b in B]
        C = [torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    flops = 2.0 * M * N * K * W
    rows = []
    t0 = time.time()
    for d in kept:
        if time.time() - t0 > budget_s:
            pruned.append((d, "budget exhausted"))
            continue
        try:
            ms, info = _time_loopback(d, W, device, A, B, C, warmup, iters, sms if d.get("sched") == "time" else sms // W)
        except api.AOError as exc:  # e.g. workspace / launch limits on this device
            pruned.append((d, "failed: %s" % exc))
            continue
        rows.append({"desc": d, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                     "tile": [info["tile_m"], info["tile_n"], info["cta_group"]]})
        if log:
            log(rows[-1])
    rows.sort(key=lambda r: r["ms"])
    return rows, pruned


def main():
    import argparse
    import json
    ap = argparse.ArgumentParser(description="AutoOverlap communication-centric tuner (loopback world)")
    ap.add_argument("--op", choices=["ag_gemm", "gemm_rs"], default="ag_gemm")
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--budget", type=float, default=120.0)
    a = ap.parse_args()
    W = a.tp
    if a.op == "ag_gemm":
        M, N, K = a.tokens, a.ffn // W, a.hidden
    else:
        M, N, K = a.tokens, a.hidden, a.ffn // W
    rows, pruned = tune_loopback(a.op, W, M, N, K, budget_s=a.budget,
                                 log=lambda r: print(json.dumps({k: r[k] for k in ("ms", "tflops", "tile")} |
                                                                {"cfg": {k: r["desc"][k] for k in
                                                                         ("chunk_rows", "backend", "intra", "group_m",
                                                                          "tile_m", "tile_n", "chunk_order",
                                                                          "dir")}}),
                                                     flush=True))
    print(json.dumps({"best": rows[0] if rows else None, "n_measured": len(rows), "n_pruned": len(pruned)}))


if __name__ == "__main__":
    main()
