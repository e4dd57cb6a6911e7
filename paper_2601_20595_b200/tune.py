"""Communication-centric auto-tuning (§5.3).

"AutoOverlap automatically generates all valid implementations, measures their end-to-end
performance, and selects the best-performing backend for each operator and hardware
configuration".  The search space is the paper's:
  * inter-chunk: chunk size (split factor) per logical transfer;
  * intra-chunk: transfer backend, tile configuration, intra-chunk tile order;
  * AG-GEMM: transfer direction, push or pull ("different implementation choices
    during lowering");
  * GEMM-RS: chunk order of the owner rotation.
  * in-kernel backends: dedicated communication CTAs vs co-located warps (comm_ctas, the
    "specialized SMs" of Fig.7 / Fig.11c) and slices per chunk (n_slices).
Candidates are pruned by the planner's validation (hardware constraints: alignment, tile
fit), by a minimum efficient transfer size for the copy engine ("minimum efficient
transfer size for copy engines") and -- seeded by the E4 backend microbenchmark
(scripts/e4_microbench.py -> profiles/r02_e4.jsonl) -- by each candidate's estimated
transfer time at its chunk size and SM budget, then timed with CUDA events on the launch
configuration they would run in (loopback world on this GPU, or the caller's world).
save_table / resolve: the winners per (op, W, M, N, K) become a table that plans with
backend "auto" consume (api.Plan).

Host logic only: every candidate runs through the C ABI like a user call.
"""
from __future__ import annotations

import bisect
import itertools
import json
import os
import time

from . import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E4_PATH = os.path.join(ROOT, "profiles", "r02_e4.jsonl")
TABLE_PATH = os.path.join(ROOT, "profiles", "r02_tune_table.json")

# a copy-engine launch costs ~2-3 us; below ~1 MiB a transfer cannot amortise it.
CE_MIN_CHUNK_BYTES = 1 << 20


def candidate_space(op: str, W: int, M: int, N: int, K: int, chunks=None, backends=None, intras=None,
                    tiles=None, orders=None, dirs=None, scheds=None, comm_ctas=None, slices=None, stream_ks=None):
    """Enumerate descs of one op (dicts with the oracle/planner desc keys).  `scheds`
    (optional) adds the loopback group schedule as key "sched": "space" (SMs/W CTAs per
    rank, ranks concurrent) or "time" (every rank over all SMs, Q24).
    `stream_ks` (optional, e.g. [0, -1]): the stream-K tail setting of AG plans with the
    copy engine (Q28); other plans keep 0."""
    S = M // W
    chunks = chunks or [c for c in (128, 256, 512, 1024, 2048, 4096) if c <= S and S % c == 0]
    backends = backends or (["ce", "tma", "ldst"] if op == "ag_gemm" and W > 1 else ["ce"])
    intras = intras or [("row", 1), ("grouped", 2), ("grouped", 4)]
    tiles = tiles or [(0, 0), (128, 256)]
    orders = orders or (["shard_major", "chunk_major"] if op == "gemm_rs" else ["shard_major"])
    dirs = dirs or (["push", "pull"] if op == "ag_gemm" and W > 1 else ["push"])
    comm_ctas = comm_ctas or [0, 8, 16]
    slices = slices or [1, 2, 4]
    out = []
    for c, b, (intra, gm), (tm, tn), o, dr in itertools.product(chunks, backends, intras, tiles, orders, dirs):
        inkernel = op == "ag_gemm" and b in ("tma", "ldst")
        sks = (stream_ks or [0]) if (op == "ag_gemm" and b == "ce" and tm != 512) else [0]
        for cc, ns, sk in itertools.product(comm_ctas if inkernel else [0], slices if inkernel else [1], sks):
            d = dict(op=op, world_size=W, M=M, N=N, K=K, chunk_rows=c, backend=b, intra=intra, group_m=gm,
                     tile_m=tm, tile_n=tn, chunk_order=o, dir=dr, n_slices=ns, comm_ctas=cc)
            if sk:
                d["stream_k"] = sk
            for sc in (scheds or [None]):
                out.append(d if sc is None else dict(d, sched=sc))
    return out


# ---- E4-seeded pruning --------------------------------------------------------------------
def load_e4(path: str = E4_PATH, mode: str = "loopback"):
    """{(backend, ctas_or_streams): sorted [(bytes, GB/s)]} from the E4 microbenchmark."""
    if not os.path.exists(path):
        return None
    curves = {}
    for line in open(path):
        r = json.loads(line)
        if r["mode"] != mode:
            continue
        key = (r["backend"], r.get("ctas", r.get("streams")))
        curves.setdefault(key, []).append((r["bytes"], r["GBps"]))
    return {k: sorted(v) for k, v in curves.items()}


def e4_bandwidth(curves, backend: str, units: int, nbytes: int):
    """GB/s of `backend` moving messages of nbytes with `units` CTAs (TMA/LDST) or streams
    (CE): log-interpolated in message size, nearest measured unit count at or below."""
    keys = sorted(u for b, u in curves if b == backend)
    if not keys:
        return None
    u = max([k for k in keys if k <= units] or [keys[0]])
    pts = curves[(backend, u)]
    xs = [p[0] for p in pts]
    i = bisect.bisect_left(xs, nbytes)
    if i == 0:
        return pts[0][1] * nbytes / xs[0]  # below the smallest size: latency-bound, linear
    if i >= len(pts):
        return pts[-1][1]
    import math
    (x0, y0), (x1, y1) = pts[i - 1], pts[i]
    t = (math.log(nbytes) - math.log(x0)) / (math.log(x1) - math.log(x0))
    return y0 + t * (y1 - y0)


def e4_transfer_ms(desc, curves, sm_count: int = 148):
    """Estimated time to move this rank's outgoing AG bytes ((W-1) shards of M/W rows) at the
    candidate's chunk size and transfer resources: CE -- one copy stream; TMA / LDST --
    comm_ctas dedicated CTAs, or the 2 co-located warps of every GEMM CTA (= n_cta / 4 CTAs
    of 8 warps)."""
    if desc["op"] != "ag_gemm" or desc["world_size"] == 1:
        return 0.0
    W, M, K = desc["world_size"], desc["M"], desc["K"]
    chunk_bytes = desc["chunk_rows"] * K * 2
    total = (W - 1) * (M // W) * K * 2
    if desc["backend"] == "ce":
        bw = e4_bandwidth(curves, "ce", 1, chunk_bytes)
    else:
        units = desc["comm_ctas"] if desc.get("comm_ctas") else max(1, (sm_count // W) // 4)
        bw = e4_bandwidth(curves, desc["backend"], units, max(16, chunk_bytes // max(1, desc.get("n_slices", 1))))
    return None if not bw else total / (bw * 1e9) * 1e3


def prune(descs, sm_count: int = 148, e4=None, slack: float = 1.5):
    """(kept, pruned) with reasons: planner validation, CE minimum efficient size, and with
    E4 curves: candidates whose estimated transfer time exceeds `slack` x the best estimate
    among the candidates of the same chunk size."""
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
    if e4:
        est = {id(d): e4_transfer_ms(d, e4, sm_count) for d in kept}
        best = {}
        for d in kept:
            e = est[id(d)]
            if e is not None:
                best[d["chunk_rows"]] = min(best.get(d["chunk_rows"], e), e)
        k2 = []
        for d in kept:
            e = est[id(d)]
            if e is not None and d["chunk_rows"] in best and e > slack * best[d["chunk_rows"]]:
                pruned.append((d, "e4: est. transfer %.3f ms > %.1f x %.3f ms" % (e, slack, best[d["chunk_rows"]])))
            else:
                k2.append(d)
        kept = k2
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
                  warmup: int = 2, iters: int = 5, space=None, log=None, use_e4: bool = True):
    """Measure every kept candidate of `op` in a W-rank loopback world on `device` and
    return rows sorted by time: [{desc, ms, tflops, tile}] + the pruned list."""
    import torch

    from synthetic import inputs as si
    torch.cuda.set_device(device)
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    descs = space if space is not None else candidate_space(op, W, M, N, K)
    kept, pruned = prune(descs, sms // W, e4=load_e4() if use_e4 else None)
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
            n_cta = sms if d.get("sched") == "time" else sms // W - d.get("comm_ctas", 0)
            ms, info = _time_loopback(d, W, device, A, B, C, warmup, iters, n_cta)
        except api.AOError as exc:  # e.g. workspace / launch limits on this device
            pruned.append((d, "failed: %s" % exc))
            continue
        rows.append({"desc": d, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                     "tile": [info["tile_m"], info["tile_n"], info["cta_group"]]})
        if log:
            log(rows[-1])
    rows.sort(key=lambda r: r["ms"])
    return rows, pruned


# ---- the tuned table and "auto" plans -----------------------------------------------------
TUNED_KEYS = ("chunk_rows", "backend", "dir", "chunk_order", "intra", "group_m", "tile_m", "tile_n", "n_slices",
              "comm_ctas")


def _shape_key(op, W, M, N, K):
    return f"{op}:W{W}:M{M}:N{N}:K{K}"


def save_table(rows, path: str = TABLE_PATH):
    """Merge the winner of a tune (rows sorted by time) into the table file."""
    if not rows:
        return None
    d = rows[0]["desc"]
    table = json.load(open(path)) if os.path.exists(path) else {}
    table[_shape_key(d["op"], d["world_size"], d["M"], d["N"], d["K"])] = {
        "desc": {k: d[k] for k in TUNED_KEYS if k in d}, "ms": rows[0]["ms"], "tflops": rows[0]["tflops"]}
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)
    return table


def resolve(desc: dict, path: str = TABLE_PATH) -> dict:
    """A desc with backend "auto" takes the tuned winner of its (op, W, M, N, K) from the
    table; without an entry, the planner defaults (copy engine, push, 128-row chunks, ROW
    order, tile picked by the planner)."""
    if desc.get("backend") != "auto":
        return desc
    table = json.load(open(path)) if os.path.exists(path) else {}
    hit = table.get(_shape_key(desc.get("op", "ag_gemm"), desc.get("world_size", 1), desc["M"], desc["N"], desc["K"]))
    out = {k: v for k, v in desc.items() if k != "backend"}
    if hit:
        out.update(hit["desc"])
    else:
        out["backend"] = "ce" if out.get("op", "ag_gemm") != "gemm_ar" else "ldst"
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser(description="AutoOverlap communication-centric tuner (loopback world)")
    ap.add_argument("--op", choices=["ag_gemm", "gemm_rs"], default="ag_gemm")
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--budget", type=float, default=120.0)
    ap.add_argument("--save", action="store_true", help="merge the winner into profiles/r02_tune_table.json")
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
    if a.save:
        save_table(rows)


if __name__ == "__main__":
    main()
