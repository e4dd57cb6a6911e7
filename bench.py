#!/usr/bin/env python
"""Benchmark of the AutoOverlap hot path on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one batch: a tensor-parallel Llama-3-8B
FFN pair on 8192 tokens --
  up-proj   ag_gemm : C_up_r[8192, 14336/W] = AllGather(A)[8192, 4096] . B_up_r^T
  down-proj gemm_rs : C_r[8192/W, 4096]     = ReduceScatter_s(C_up_s . B_down_s^T)
(BASELINE.json configs[1] and configs[2]; the down-proj consumes the up-proj output).

  N = 1 (default): W = --tp logical ranks (default 8) run in LOOPBACK on the one GPU:
        every rank has its own symmetric workspace; chunks move HBM->HBM instead of over
        NVLink; both fused ops are single launches covering all W ranks.
  N > 1 (torchrun): one rank per GPU, W = N, peer memory over NVLink (cudaIpc).
Total work is the same FFN layer for every N ("scaling": "strong").

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead (the
tier's reference arm).  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks; inputs > L2 (no flush needed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HIDDEN, FFN, TOKENS = 4096, 14336, 8192
METRIC = "fused AG-GEMM / GEMM-RS TFLOP/s and % roofline at 2/4/8 B200 vs NCCL+GEMM overlap"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tp", type=int, default=8, help="logical TP ranks in loopback (N=1)")
    ap.add_argument("--backend", default="ce", choices=["ce", "tma", "ldst"])
    ap.add_argument("--exp", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--debug", action="append", default=[], help=argparse.SUPPRESS)
    ap.add_argument("--no-ar", action="store_true", help="skip the GEMM-AR (NEXT-1) leg")
    ap.add_argument("--no-a2a", action="store_true", help="skip the A2A-GEMM (NEXT-3, Mixtral) leg")
    ap.add_argument("--no-attn", action="store_true", help="skip the SP-attention (NEXT-4) leg")
    ap.add_argument("--attn-seq", type=int, default=32768, help="SP attention: total sequence length")
    ap.add_argument("--a2a-chunk", type=int, default=64, help="A2A chunk rows")
    ap.add_argument("--a2a-zipf", type=float, default=0.0, help="A2A routing skew (0 = top-2 of N(0,1) logits)")
    ap.add_argument("--a2a-group-m", type=int, default=16,
                    help="A2A GROUP_M (row blocks per group; 16 covers an expert's ~2050 rows: its weight is read once)")
    ap.add_argument("--ar-chunk", type=int, default=256, help="GEMM-AR chunk rows")
    ap.add_argument("--ag-dir", default="push", choices=["push", "pull"], help="AG transfer direction (Lst.2, P:295)")
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--tile", default="256x256", help="time-sliced AG / RS tile BMxBN (512x256: two CTA pairs "
                    "sharing B by multicast)")
    ap.add_argument("--sched", default="time", choices=["time", "space"],
                    help="loopback group schedule: time-sliced (all SMs per rank) or space-sliced (SMs/W per rank)")
    ap.add_argument("--tokens", type=int, default=TOKENS)
    ap.add_argument("--intra", default="grouped", choices=["row", "col", "grouped"])
    ap.add_argument("--group-m", type=int, default=4)
    ap.add_argument("--rs-chunk", type=int, default=0, help="GEMM-RS chunk rows (0 = --chunk)")
    ap.add_argument("--rs-order", default="shard_major", choices=["shard_major", "chunk_major"])
    ap.add_argument("--rs-reduce", default="atomic", choices=["slots", "atomic"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-baseline", action="store_true")
    ap.add_argument("--l2-hint", type=int, default=-1)
    ap.add_argument("--no-check", action="store_true", help="skip the fp32 sanity check (keeps ncu launch lists clean)")
    ap.add_argument("--trace", default="", help="write Chrome traces of one extra step to PREFIX_{ag,rs}.json")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, device):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def nvlink_roofline(W, M, F, loop, ag_ms, rs_ms, peak, flops):
    """SURVEY §8(d) per-rank roofline of the fused ops: T_roof = max(FLOPs_rank / P, wire bytes
    per rank per direction / B_link) with B_link = 900 GB/s nominal (770 measured peer copy):
    AG (W-1)/W*M*K*2, RS (W-1)/W*M*N*4 (fp32 partials).  In loopback (N = 1) the transfers stay
    on the GPU, so the link terms are what TP=W would need, not what was measured."""
    f_rank = flops / (W if loop else 1)
    out = {"link_gbs": 900.0, "link_gbs_measured_peer_copy": 770.0,
           "exercised": not loop}
    for op, wire, ms in (("ag_gemm", (W - 1) / W * M * HIDDEN * 2, ag_ms), ("gemm_rs", (W - 1) / W * M * HIDDEN * 4, rs_ms)):
        t_gemm = f_rank / (peak * 1e12) * 1e3
        t_link = wire / 900e9 * 1e3
        d = {"wire_bytes_per_rank": int(wire), "t_gemm_ms": round(t_gemm, 4), "t_link_ms": round(t_link, 4),
             "bound": "nvlink" if t_link > t_gemm else "tensor", "t_roof_ms": round(max(t_gemm, t_link), 4)}
        if not loop:
            d["frac"] = round(max(t_gemm, t_link) / ms, 4)
        out[op] = d
    return out


def choose_peak(peaks, f_kernel):
    """Roofline denominator by the task's rule -- the burst figure for a kernel timed alone,
    the sustained one for a kernel timed inside a long step -- decided by measurement: the
    sustained figure when the kernel's in-kernel SM clock (MHz) is at most 1.1x the clock the
    sustained cuBLAS figure was measured at.  Returns (peak, sustained?, regime text)."""
    sus_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
    sustained = bool(f_kernel and sus_mhz and "bf16_tflops_sustained" in peaks and f_kernel <= 1.1 * sus_mhz)
    if sustained:
        return peaks["bf16_tflops_sustained"], True, (
            f"sustained: the kernel runs at {f_kernel} MHz (in-kernel clock64/globaltimer median over its MMA "
            f"spans) vs sm_max {peaks.get('sm_max_mhz')} MHz; the sustained cuBLAS figure was measured at "
            f"{sus_mhz} MHz")
    return peaks["bf16_tflops"], False, f"burst: in-kernel clock {f_kernel} MHz, sustained measurement at {sus_mhz} MHz"


def kernel_clocks(ctx, step, steps=3):
    """The SM clock the fused kernels actually run at: clock64 cycles / %globaltimer ns over
    every MMA span (TR_CLK trace events) of `steps` extra back-to-back steps run right after
    the timed region (tracing costs ~3 %, so never inside it).  NVML's clock reading stays at
    sm_max_mhz through these kernels while the in-kernel rate is ~30 % lower: the power limit
    acts below NVML's view (scripts/experiments/clock_probe.cu calibrates the method: an idle
    GPU reads sm_max_mhz).  Launches alternate ag_gemm, rs; the first step is skipped."""
    import tempfile
    ctx.trace_enable(1 << 21)
    for _ in range(steps):
        step()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    try:
        ctx.trace_dump(path)
        with open(path) as f:
            ev = json.load(f)["traceEvents"]
    finally:
        ctx.trace_enable(0)
        os.unlink(path)
    out = {}
    for name, par in (("ag_gemm", 0), ("gemm_rs", 1)):
        mhz = [int(e["name"].split()[1]) / e["dur"] for e in ev
               if e["cat"] == "clock" and e["dur"] > 0 and e["args"]["launch"] >= 2 and e["args"]["launch"] % 2 == par]
        out[name] = round(statistics.median(mhz)) if mhz else None
    return out


# ============================================================================ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2601_20595_b200 import build
    build.build(verbose=False)  # no-op when the in-tree .so is current
    import paper_2601_20595_b200 as ao
    from synthetic import inputs as si

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if args.l2_hint >= 0:
        ao.debug_set("l2_hint", args.l2_hint)
    if args.exp:
        ao.debug_set("exp", args.exp)  # timing experiments: results are NOT valid
    for kv in args.debug:
        k, v = kv.split("=")
        ao.debug_set(k, int(v))
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    if SHARED_GPU and world > 1:
        sms = sms // world // 2 * 2  # the ranks' persistent kernels must co-reside (MPS)
    M = args.tokens
    loop = world == 1
    W = args.tp if loop else world
    F = FFN // W
    base = dict(world_size=W, M=M, chunk_rows=args.chunk, timeout_ns=5_000_000_000, intra=args.intra,
                group_m=args.group_m)
    ag_desc = dict(base, op="ag_gemm", N=F, K=HIDDEN, backend=args.backend, dir=args.ag_dir, n_slices=2)
    rs_desc = dict(base, op="gemm_rs", N=HIDDEN, K=F, chunk_order=args.rs_order,
                   chunk_rows=args.rs_chunk or args.chunk, rs_reduce=args.rs_reduce)
    # NEXT-1 row, measured beside the step: GEMM-AR on the down-proj shape
    # (scripts/ar_probe.py: 256-row chunks in chunk-major order let owners reduce chunk j
    # mid-kernel so the gather overlaps the GEMM; best of chunk x order x slices)
    ar_desc = dict(rs_desc, op="gemm_ar", backend="ldst", n_slices=8, chunk_rows=args.ar_chunk,
                   chunk_order="chunk_major")
    if loop:
        # time-sliced (default): every rank's plan spans all SMs and the group launch runs the
        # ranks' tile lists in one global order; space-sliced: SMs // W CTAs per rank
        # GEMM-AR time-sliced too (0.92 ms vs 1.14 space-sliced, scripts/ar_probe2.py)
        ar_desc["n_cta"] = sms if args.sched == "time" else sms // W
        ar_desc["tile_m"], ar_desc["tile_n"] = 256, 256
        ag_desc["n_cta"] = rs_desc["n_cta"] = sms if args.sched == "time" else sms // W
        if args.sched == "time":
            tm, tn = (int(x) for x in args.tile.split("x"))
            for d in (ag_desc, rs_desc):
                d["tile_m"], d["tile_n"] = tm, tn
                if tm == 512:  # 4-CTA clusters: as many as fit the GPU at once
                    d["n_cta"] = ao.device_query(local_rank, "cluster4_ctas")
    if not loop and SHARED_GPU:
        ag_desc["n_cta"] = rs_desc["n_cta"] = ar_desc["n_cta"] = sms
    ws = max(ao.workspace_bytes(ag_desc), ao.workspace_bytes(rs_desc),
             0 if args.no_ar else ao.workspace_bytes(ar_desc))
    if loop:
        ctxs = ao.loopback_world(local_rank, W, ws)
        my_ranks = list(range(W))
    else:
        ctxs = [ao.dist_world(local_rank, ws)]
        my_ranks = [rank]
    pa = [ao.Plan(c, dict(ag_desc, rank=r)) for c, r in zip(ctxs, my_ranks)]
    pr = [ao.Plan(c, dict(rs_desc, rank=r)) for c, r in zip(ctxs, my_ranks)]

    # inputs (seeded, synthetic; same generator as the tests)
    A_cpu, Bu_cpu = si.ag_inputs(W, M, HIDDEN, F)
    Bd_cpu = si.rs_weights(W, F, HIDDEN)
    A = [A_cpu[r].to(dev) for r in my_ranks]
    Bu = [Bu_cpu[r].to(dev) for r in my_ranks]
    Bd = [Bd_cpu[r].to(dev) for r in my_ranks]
    del Bu_cpu, Bd_cpu
    Cu = [torch.empty(M, F, dtype=torch.bfloat16, device=dev) for _ in my_ranks]
    Cd = [torch.empty(M // W, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in my_ranks]
    stream = torch.cuda.current_stream()

    def step(ev=None, A_in=None, C_out=None):
        A_in = A if A_in is None else A_in
        C_out = Cd if C_out is None else C_out
        if ev is not None:
            ev[0].record(stream)
        if loop:
            ao.ag_gemm_group(pa, A_in, Bu, Cu)
        else:
            ao.ag_gemm(pa[0], A_in[0], Bu[0], Cu[0])
        if ev is not None:
            ev[1].record(stream)
        if loop:
            ao.gemm_rs_group(pr, Cu, Bd, C_out)
        else:
            ao.gemm_rs(pr[0], Cu[0], Bd[0], C_out[0])
        if ev is not None:
            ev[2].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    for c in ctxs:
        c.check_async()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        t0.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t1.record(stream)
        barrier()
    for c in ctxs:
        c.check_async()
    total_ms = t0.elapsed_time(t1)
    ag_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    rs_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    if world > 1:
        t = torch.tensor([total_ms, ag_ms, rs_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, ag_ms, rs_ms = t.tolist()
    ms = total_ms / args.steps
    ms_median = statistics.median(e[0].elapsed_time(e[2]) for e in evs)
    flops_ag = 2.0 * M * FFN * HIDDEN  # whole layer, all ranks
    flops_step = 2 * flops_ag
    value = flops_step / (ms * 1e-3) / 1e12

    if args.trace:
        # three back-to-back steps (launches 0..5: ag, rs, ag, rs, ag, rs) in one trace; every
        # rank steps (collective ops), rank r > 0 writes PREFIX.rank<r>.json
        ctxs[0].trace_enable(1 << 21)
        for _ in range(3):
            step()
        ctxs[0].trace_dump(args.trace + (".json" if rank == 0 else ".rank%d.json" % rank))
        ctxs[0].trace_enable(0)
        barrier()

    # --- the SM clock under load, measured inside the kernels (decides the peak regime) -----
    # every rank runs the traced steps (the ops are collective: a rank stepping alone would
    # wait on its peers' chunks); each reads its own kernels' clock
    clk_kernel = kernel_clocks(ctxs[0], step)
    barrier()

    # --- single-op latency: each op alone, barrier + synchronize before it ---
    def one_op(fn):
        ts = []
        for _ in range(7):
            barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            fn()
            s1.record(stream)
            s1.synchronize()
            ts.append(s0.elapsed_time(s1))
        v = statistics.median(ts[1:])
        if world > 1:
            t = torch.tensor([v], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            v = t.item()
        return round(v, 4)

    if loop:
        latency = {"ag_gemm": one_op(lambda: ao.ag_gemm_group(pa, A, Bu, Cu)),
                   "gemm_rs": one_op(lambda: ao.gemm_rs_group(pr, Cu, Bd, Cd))}
    else:
        latency = {"ag_gemm": one_op(lambda: ao.ag_gemm(pa[0], A[0], Bu[0], Cu[0])),
                   "gemm_rs": one_op(lambda: ao.gemm_rs(pr[0], Cu[0], Bd[0], Cd[0]))}
    latency["what"] = "ms per op launched alone after a barrier + synchronize (median of 6, max over ranks)"

    # --- sanity vs cuBLAS on sampled rows (not the oracle; parity lives in tests/) ------
    check = None
    if rank == 0 and not args.no_check:
        rows = torch.arange(0, M, 509, device=dev)
        A_full = torch.cat(A, 0) if loop else None
        if loop:
            ref_up = (A_full[rows].float() @ Bu[0].float().t())
            err_up = (Cu[0][rows].float() - ref_up).abs().max().item()
            part = sum((Cu[s][: M // W].float() @ Bd[s].float().t()) for s in range(W))
            err_rs = (Cd[0].float() - part).abs().max().item()
            check = {"max_abs_err_up_vs_fp32": err_up, "max_abs_err_down_vs_fp32": err_rs}

    # --- kernel-level baseline on this box (cuBLAS + copies / NCCL, two streams) --------
    baseline = None
    if loop and not args.no_baseline and rank == 0:
        baseline = loopback_baseline(torch, A, Bu, Bd, Cu, W, M, F, args)
    elif not loop and not args.no_baseline and not SHARED_GPU:
        baseline = nccl_baseline(torch, dist, A[0], Bu[0], Bd[0], W, M, F, args, dev)

    # --- GEMM-only leg: the same kernel, tiles and workers with no communication -------
    gemm_only = None
    if not args.no_baseline:
        gemm_only = gemm_only_leg(torch, ao, pa, pr, A, Bu, Bd, W, M, F, args, dev, loop)
        if gemm_only is not None:
            gemm_only["exposed_comm_ms"] = {"ag_gemm": round(ag_ms - gemm_only["ag_gemm_ms"], 4),
                                            "gemm_rs": round(rs_ms - gemm_only["gemm_rs_ms"], 4)}

    # --- the per-GPU TP shapes: one rank alone, peers' chunks pre-arrived ----------------
    per_rank = None
    if loop and not args.no_baseline:
        per_rank = per_rank_leg(torch, ao, ctxs, A, Bu, Cu, Bd, W, M, F, args, dev, sms)

    # --- GEMM-AR (NEXT-1) on the down-proj shape, same ctxs ----------------------------
    ar = None
    if not args.no_ar:
        ar = ar_leg(torch, ao, ctxs, my_ranks, ar_desc, Cu, Bd, M, W, args, dev, loop, world, dist)

    # --- A2A-GEMM (NEXT-3): Mixtral-8x7B MoE dispatch + expert GEMM, BASELINE configs[3] -----
    a2a = None
    if not args.no_a2a:
        a2a = a2a_leg(torch, ao, si, args, dev, loop, world, rank, local_rank, dist, sms)

    # --- SP attention (NEXT-4): Llama-3-8B attention, sequence-parallel over W ranks ---------
    attn = None
    if not args.no_attn:
        attn = attn_leg(torch, ao, si, args, dev, loop, world, rank, local_rank, dist, sms)

    # --- e2e through the public API with host buffers --------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(torch, dist, args, A, Cd, step, barrier, world, flops_step, dev)

    peaks, peaks_src = load_peaks()
    # Peak regime (task rule: burst for a kernel timed alone, sustained for one timed inside
    # a long step), decided by measurement: the dominant kernel's in-kernel SM clock against
    # the clock MEASURED_PEAKS' sustained cuBLAS figure was taken at.
    dom_ms = max(ag_ms, rs_ms)
    f_dom = clk_kernel.get("ag_gemm" if ag_ms >= rs_ms else "gemm_rs")
    peak, sustained, regime = choose_peak(peaks, f_dom)
    dom = "ag_gemm" if ag_ms >= rs_ms else "gemm_rs"
    per_launch_flops = flops_ag / (1 if loop else W)
    achieved = per_launch_flops / (dom_ms * 1e-3) / 1e12
    traffic = load_traffic(dom)
    ag_ach = per_launch_flops / (ag_ms * 1e-3) / 1e12
    rs_ach = per_launch_flops / (rs_ms * 1e-3) / 1e12
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "ms_per_step_median": round(ms_median, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) activations, N(0,1)/sqrt(K) weights)",
        "config": {"workload": f"llama3-8b-tp{W}-ffn-pair-{'loopback' if loop else 'nvlink'}",
                   "tokens": M, "hidden": HIDDEN, "ffn": FFN, "tp": W, "ranks_per_gpu": W if loop else 1,
                   "backend_ag": args.backend, "ag_dir": args.ag_dir, "chunk_rows": args.chunk, "rs_chunk_rows": args.rs_chunk or args.chunk,
                   "intra": args.intra, "group_m": args.group_m, "rs_chunk_order": args.rs_order,
                   "rs_reduce": args.rs_reduce, "group_schedule": (args.sched + "-sliced") if loop else "one rank per GPU",
                   "tile": [pa[0].info()["tile_m"], pa[0].info()["tile_n"]], "cta_group": pa[0].info()["cta_group"],
                   "workers_per_rank": pa[0].info()["n_cta"],
                   "ctas_per_rank": pa[0].info()["n_cta"] * pa[0].info()["cta_group"],
                   "l2": "inputs+weights ~0.7 GB/step > 126 MB L2 (no flush)", "parallelism": f"tp{W}"},
        "gpu_launches": 2 * args.steps * (1 if loop else world),  # fused kernels, all ranks
        "kernels_ms": {"ag_gemm": round(ag_ms, 4), "gemm_rs": round(rs_ms, 4)},
        "single_op_latency_ms": latency,
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "peak_source": f"{peaks_src} bf16_tflops{'_sustained' if sustained else ''} "
                                    f"({'sustained' if sustained else 'burst'})",
                     "peak_regime": regime, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4),
                     "frac_of_burst": round(achieved / peaks["bf16_tflops"], 4),
                     "frac_of_nominal": round(achieved / 2250.0, 4),  # 2.25 PFLOP/s dense bf16
                     # the tensor pipe's own ceiling at the clock the kernel ran: 148 SMs x 8192
                     # dense bf16 flop/clk (tcgen05 kind::f16; 2.25 PFLOP/s nominal = 1.86 GHz)
                     "frac_at_kernel_clock": (round(achieved / (torch.cuda.get_device_properties(dev).multi_processor_count * 8192 * f_dom * 1e-6), 4) if f_dom else None),
                     "frac_of_sustained": round(achieved / peaks.get("bf16_tflops_sustained", peak), 4),
                     "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
                     "flops_per_launch": per_launch_flops,
                     "per_kernel": {"ag_gemm": {"achieved": round(ag_ach, 1), "frac": round(ag_ach / peak, 4)},
                                    "gemm_rs": {"achieved": round(rs_ach, 1), "frac": round(rs_ach / peak, 4)}},
                     "nvlink": nvlink_roofline(W, M, F, loop, ag_ms, rs_ms, peak, per_launch_flops)},
        "clocks": clk.summary(),
        # not the NVML record above: clock64 / globaltimer over the fused kernels' MMA spans
        # (three extra steps after the timed region) -- the power limit's effective SM clock
        "sm_mhz_in_kernel": dict(clk_kernel, method="clock64 cycles / globaltimer ns over every MMA span, "
                                 "median; NVML shows sm_max through the same kernels"),
        "e2e": e2e,
        "check": check,
        "baseline_kernel_level": baseline,
        "gemm_only": gemm_only,
        "per_rank_tp": per_rank,
        "gemm_ar": ar,
        "a2a_gemm": a2a,
        "sp_attn": attn,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(W, M, budget_s=12.0)
    if rank == 0:
        print(json.dumps(out), flush=True)


def load_traffic(kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def loopback_baseline(torch, A, Bu, Bd, Cu, W, M, F, args):
    """SURVEY §8(d)(ii), the kernel-level two-stream overlap baseline with the W
    loopback ranks on this GPU: the op split into s pieces; a comm stream runs the
    collective of piece i+1 (AG: every rank's gathered copy of piece i's rows of all shards;
    RS: the owners' sums of piece i's columns of the W partials) while the compute stream
    runs cuBLAS on piece i.  RS partials in fp32 (cuBLAS bf16 x bf16 -> fp32, precision-
    matched with the fused kernel's fp32 wire) and in bf16 (the usual practice, reported
    beside it).  Best s in {1, 2, 4, 8} per precision; the headline comparison is fp32."""
    dev = A[0].device
    S = M // W
    comm = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    A_st = torch.stack(A, 0)  # [W, S, K]: the W ranks' shards (loopback: all on this GPU)
    Cup = [torch.empty(M, F, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    Out = [torch.empty(S, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    out = {}
    for prec in ("fp32", "bf16"):
        pdt = torch.float32 if prec == "fp32" else torch.bfloat16
        res = {}
        for s in (1, 2, 4, 8):
            rows, cols = S // s, HIDDEN // s
            G = [[torch.empty(W, rows, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in range(s)] for _ in range(W)]
            P = [torch.empty(W, M, cols, dtype=pdt, device=dev) for _ in range(s)]
            ev_ag = [torch.cuda.Event() for _ in range(s)]
            ev_mm = [torch.cuda.Event() for _ in range(s)]
            ev_rs = [torch.cuda.Event() for _ in range(s)]

            def step():
                comm.wait_stream(main)
                with torch.cuda.stream(comm):  # AG of piece i into every rank's gathered buffer
                    for i in range(s):
                        for r in range(W):
                            G[r][i].copy_(A_st[:, i * rows:(i + 1) * rows])
                        ev_ag[i].record(comm)
                for i in range(s):
                    main.wait_event(ev_ag[i])
                    for r in range(W):
                        y = torch.matmul(G[r][i].view(W * rows, HIDDEN), Bu[r].t())
                        Cup[r].view(W, S, F)[:, i * rows:(i + 1) * rows].copy_(y.view(W, rows, F))
                for i in range(s):  # RS: column pieces; partials of every source rank
                    for q in range(W):
                        if prec == "fp32":
                            torch.mm(Cup[q], Bd[q][i * cols:(i + 1) * cols].t(), out_dtype=torch.float32, out=P[i][q])
                        else:
                            torch.matmul(Cup[q], Bd[q][i * cols:(i + 1) * cols].t(), out=P[i][q])
                    ev_mm[i].record(main)
                    comm.wait_event(ev_mm[i])
                    with torch.cuda.stream(comm):  # owners' sums (the ReduceScatter)
                        red = P[i].view(W, W, S, cols).sum(0)
                        for o in range(W):
                            Out[o][:, i * cols:(i + 1) * cols].copy_(red[o])
                        ev_rs[i].record(comm)
                for i in range(s):
                    main.wait_event(ev_rs[i])

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = max(5, args.steps // 2)
            st.record(main)
            for _ in range(n):
                step()
            en.record(main)
            torch.cuda.synchronize()
            res[s] = st.elapsed_time(en) / n
            del G, P
        best = min(res, key=res.get)
        out[prec] = {"ms_per_step": round(res[best], 4), "tflops": round(4.0 * M * FFN * HIDDEN / (res[best] * 1e-3) / 1e12, 2),
                     "best_split": best, "per_split_ms": {str(k): round(v, 4) for k, v in res.items()}}
    return {"what": "kernel-level two-stream split overlap on this GPU (W loopback ranks): comm-stream "
                    "gather copies / owner sums + cuBLAS GEMMs per piece, best split s (SURVEY 8(d)(ii))",
            "ms_per_step": out["fp32"]["ms_per_step"], "tflops": out["fp32"]["tflops"],
            "rs_partials_fp32": out["fp32"], "rs_partials_bf16": out["bf16"]}


def ar_leg(torch, ao, ctxs, my_ranks, ar_desc, Cu, Bd, M, W, args, dev, loop, world, dist):
    """NEXT-1: fused GEMM-AllReduce (RS schedule + pull gather of the reduced chunks) on the
    down-proj shape; every rank ends with the full [M, HIDDEN] output.  Device-timed like
    the step (CUDA events, max over ranks)."""
    plans = [ao.Plan(c, dict(ar_desc, rank=r)) for c, r in zip(ctxs, my_ranks)]
    C = [torch.empty(M, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in my_ranks]

    def run():
        if loop:
            ao.gemm_ar_group(plans, Cu, Bd, C)
        else:
            ao.gemm_ar(plans[0], Cu[0], Bd[0], C[0])

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(5, args.steps // 2)
    if world > 1:
        dist.barrier()
    s.record()
    for _ in range(k):
        run()
    e.record()
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    ms = s.elapsed_time(e) / k
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    flops = 2.0 * M * FFN * HIDDEN / (1 if loop else W)
    info = plans[0].info()
    for p in plans:
        p.close()
    return {"what": "fused GEMM-AllReduce (NEXT-1), down-proj shape, every rank gets [M, hidden]",
            "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
            "rs_reduce": ar_desc["rs_reduce"], "chunk_rows": ar_desc["chunk_rows"],
            "chunk_order": ar_desc["chunk_order"],
            "tile": [info["tile_m"], info["tile_n"]], "launches": k * (1 if loop else 1)}


def a2a_leg(torch, ao, si, args, dev, loop, world, rank, local_rank, dist, sms):
    """NEXT-3 (BASELINE configs[3]): Mixtral-8x7B MoE, 8 experts over 8 ranks, top-2 of 8192
    tokens (1024 per rank), H = 4096, expert w1||w3 (N = 2 * 14336): All-to-All dispatch fused
    with the expert GEMM.  Loopback: the 8 ranks time-sliced over all SMs; N > 1: one rank per
    GPU.  Also the same expert GEMMs on pre-dispatched rows (ao_gemm_batched, no dispatch).
    FLOPs = 2 * (rows received, summed over experts = W*T*k) * N * H."""
    W = 8 if loop else world
    T, H, N, k = 8192 // W, HIDDEN, 2 * FFN, 2
    my = list(range(W)) if loop else [rank]
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k, zipf=args.a2a_zipf)
    desc = dict(op="a2a_gemm", world_size=W, M=T, N=N, K=H, topk=k, chunk_rows=args.a2a_chunk, backend="ldst",
                tile_m=256, tile_n=256, intra="grouped", group_m=args.a2a_group_m, n_cta=sms, timeout_ns=10_000_000_000)
    ctxs = ao.loopback_world(local_rank, W, ao.workspace_bytes(desc)) if loop else \
        [ao.dist_world(local_rank, ao.workspace_bytes(desc))]
    plans = [ao.Plan(c, dict(desc, rank=r)) for c, r in zip(ctxs, my)]
    Xd = [X[r].to(dev) for r in my]
    Id = [idx[r].to(dev) for r in my]
    Bd = [B[r].to(dev) for r in my]
    del B
    Y = [torch.empty(W * T, N, dtype=torch.bfloat16, device=dev) for _ in my]
    rp = [torch.empty(T, k, dtype=torch.int32, device=dev) for _ in my]
    rr = [torch.empty(1, dtype=torch.int32, device=dev) for _ in my]

    def run():
        if loop:
            ao.a2a_gemm_group(plans, Xd, Id, Bd, Y, rp, rr)
        else:
            ao.a2a_gemm(plans[0], Xd[0], Id[0], Bd[0], Y[0], rp[0], rr[0])

    def timed(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    n = max(5, args.steps // 5)
    ms = timed(run, n)
    for c in ctxs:
        c.check_async()
    rows = [int(r.item()) for r in rr]
    flops = 2.0 * W * T * k * N * H / (1 if loop else W)
    # GEMM-only reference: the experts' GEMMs on already-dispatched rows (the mean row count,
    # rounded to the tile), same kernel and workers, no dispatch / waits
    Rm = (W * T * k // W + 255) // 256 * 256
    A_d = [torch.randn(Rm, H, device=dev).to(torch.bfloat16) for _ in my]
    Y_d = [torch.empty(Rm, N, dtype=torch.bfloat16, device=dev) for _ in my]
    g_ms = timed(lambda: ao.gemm_batched(A_d, Bd, Y_d, 256, 256, 8, sms), n)
    g_flops = 2.0 * Rm * N * H * len(my)
    peaks, _ = load_peaks()
    tf = flops / (ms * 1e-3) / 1e12
    for p in plans:
        p.close()
    return {"what": "MoE All-to-All dispatch fused with the expert GEMM (NEXT-3), Mixtral-8x7B 8 experts, top-2",
            "workload": "mixtral-8x7b-moe-ep8-a2a-gemm-" + ("loopback" if loop else "nvlink"),
            "tokens": W * T, "hidden": H, "n_expert_out": N, "topk": k, "zipf": args.a2a_zipf,
            "chunk_rows": args.a2a_chunk, "ms": round(ms, 4), "tflops": round(tf, 1),
            "frac_of_peak": round(tf / peaks["bf16_tflops"], 4),  # burst
            "frac_of_sustained": round(tf / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]), 4),
            "rows_per_expert": rows if loop else rows[0],
            "gemm_only_ms_equal_rows": round(g_ms, 4),
            "gemm_only_tflops": round(g_flops / (g_ms * 1e-3) / 1e12, 1), "launches_per_op": 2}


def attn_leg(torch, ao, si, args, dev, loop, world, rank, local_rank, dist, sms):
    """NEXT-4: sequence-parallel attention with the KV all-gathered in ring order, Llama-3-8B
    attention (32 heads, d = 128), non-causal, --attn-seq tokens split over 8 ranks (loopback,
    time-sliced) or over the N GPUs.  FLOPs = 4 * S_total^2 * d * H (QK^T and PV).  Beside it:
    torch SDPA (library flash attention) on the same gathered K/V, per rank."""
    import torch.nn.functional as Fn
    W = 8 if loop else world
    H, d = 32, 128
    S = args.attn_seq // W
    my = list(range(W)) if loop else [rank]
    Q, K, V = si.attn_inputs(W, H, S, d)
    desc = dict(op="sp_attn", world_size=W, M=S, N=H, K=d, chunk_rows=S, backend="ce", n_cta=sms,
                timeout_ns=10_000_000_000)
    ctxs = ao.loopback_world(local_rank, W, ao.workspace_bytes(desc)) if loop else \
        [ao.dist_world(local_rank, ao.workspace_bytes(desc))]
    plans = [ao.Plan(c, dict(desc, rank=r)) for c, r in zip(ctxs, my)]
    Qd = [Q[r].to(dev) for r in my]
    Kd = [K[r].to(dev) for r in my]
    Vd = [V[r].to(dev) for r in my]
    Od = [torch.empty_like(q) for q in Qd]

    def run():
        if loop:
            ao.sp_attn_group(plans, Qd, Kd, Vd, Od)
        else:
            ao.sp_attn(plans[0], Qd[0], Kd[0], Vd[0], Od[0])

    def timed(fn, n):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    n = max(3, args.steps // 10)
    ms = timed(run, n)
    for c in ctxs:
        c.check_async()
    Stot = S * W
    flops = 4.0 * Stot * Stot * d * H / (1 if loop else W)
    # causal variant (RingAttention for decoders): half the score matrix; same inputs
    cplans = [ao.Plan(c, dict(desc, rank=r, causal=1)) for c, r in zip(ctxs, my)]

    def run_c():
        if loop:
            ao.sp_attn_group(cplans, Qd, Kd, Vd, Od)
        else:
            ao.sp_attn(cplans[0], Qd[0], Kd[0], Vd[0], Od[0])

    ms_c = timed(run_c, n)
    for c in ctxs:
        c.check_async()
    flops_c = 2.0 * Stot * Stot * d * H / (1 if loop else W)
    for p in cplans:
        p.close()
    # head-parallel (Ulysses) variant: Q/K/V all-to-all in, H/W heads per rank over the
    # whole sequence, output tiles returned to their owners (same FLOPs, same result)
    hdesc = dict(desc, op="hp_attn", chunk_rows=(H // W) * S // 4 if (H // W) * S % (4 * 128) == 0 else S)
    hp_res = {}
    if H % W == 0 and S % 256 == 0:
        hctxs = ao.loopback_world(local_rank, W, ao.workspace_bytes(hdesc)) if loop else \
            [ao.dist_world(local_rank, ao.workspace_bytes(hdesc))]
        for cz in (0, 1):
            hplans = [ao.Plan(c, dict(hdesc, rank=r, causal=cz)) for c, r in zip(hctxs, my)]

            def run_h(hplans=hplans):
                if loop:
                    ao.hp_attn_group(hplans, Qd, Kd, Vd, Od)
                else:
                    ao.hp_attn(hplans[0], Qd[0], Kd[0], Vd[0], Od[0])

            ms_h = timed(run_h, n)
            for c in hctxs:
                c.check_async()
            fl = flops_c if cz else flops
            hp_res["causal_ms" if cz else "ms"] = round(ms_h, 4)
            hp_res["causal_tflops" if cz else "tflops"] = round(fl / (ms_h * 1e-3) / 1e12, 1)
            for p in hplans:
                p.close()
        hp_res["chunk_rows"] = hdesc["chunk_rows"]
        for c in hctxs:
            c.close()
    # library reference: SDPA per rank over its gathered K/V (already resident)
    if loop:
        Kf = torch.cat([k.to(dev) for k in K], 1).unsqueeze(0)
        Vf = torch.cat([v.to(dev) for v in V], 1).unsqueeze(0)
        sd = lambda: [Fn.scaled_dot_product_attention(q.unsqueeze(0), Kf, Vf) for q in Qd]
        sd_ms = timed(sd, n)
        del Kf, Vf
    else:
        sd_ms = None
    peaks, _ = load_peaks()
    tf = flops / (ms * 1e-3) / 1e12
    for p in plans:
        p.close()
    return {"what": "sequence-parallel attention over the all-gathered KV in ring order (NEXT-4), non-causal",
            "workload": "llama3-8b-attn-sp%d-%s" % (W, "loopback" if loop else "nvlink"),
            "seq_total": Stot, "heads": H, "head_dim": d, "ms": round(ms, 4), "tflops": round(tf, 1),
            "frac_of_peak": round(tf / peaks["bf16_tflops"], 4),  # burst
            "frac_of_sustained": round(tf / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]), 4),
            "causal_ms": round(ms_c, 4), "causal_tflops": round(flops_c / (ms_c * 1e-3) / 1e12, 1),
            "sdpa_same_gpu_ms": None if sd_ms is None else round(sd_ms, 4),
            "sdpa_tflops": None if sd_ms is None else round(flops / (sd_ms * 1e-3) / 1e12, 1),
            "head_parallel": hp_res}


def per_rank_leg(torch, ao, ctxs, A, Bu, Cu, Bd, W, M, F, args, dev, sms):
    """The per-GPU work of TP=W (the north star's "1 GPU (GEMM only)" point, VERDICT r01 item
    3): rank 0's fused ag_gemm (M x F x HIDDEN) and gemm_rs (M x HIDDEN x F) alone on all
    SMs through the per-rank C ABI call, with every peer chunk flag pre-arrived
    (ao_debug_set prearrive: the waits are satisfied and no copy-engine chain is issued; RS
    still reduce-adds its partials into the peers' accumulators).  Tiles: the planner's
    pick, 256x256 and the 512x256 cluster tile; beside each, the plain GEMM (ao.gemm) on the
    same shape and tile, and cuBLAS."""
    W_ = W
    n4 = ao.device_query(dev.index, "cluster4_ctas")
    res = {"what": "rank 0 of TP=%d alone on the GPU, all SMs, peer chunks pre-arrived" % W_}
    k = max(10, args.steps)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(k):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / k

    flops = 2.0 * M * F * HIDDEN
    base = dict(world_size=W_, rank=0, M=M, chunk_rows=args.chunk, timeout_ns=5_000_000_000, intra=args.intra,
                group_m=args.group_m)
    Cd0 = torch.empty(M // W_, HIDDEN, dtype=torch.bfloat16, device=dev)
    C_up = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
    C_dn = torch.empty(M, HIDDEN, dtype=torch.bfloat16, device=dev)
    A_full = torch.cat(A, 0)
    # its own contexts: only rank 0 launches here, which would put the shared world's
    # epochs and collective plan sequence (AO_ERR_PEER agreement) out of step
    ws = max(ao.workspace_bytes(dict(base, op="ag_gemm", N=F, K=HIDDEN, n_cta=sms)),
             ao.workspace_bytes(dict(base, op="gemm_rs", N=HIDDEN, K=F, n_cta=sms, rs_reduce="atomic")))
    ctxs = ao.loopback_world(dev.index, W_, ws)
    ao.debug_set("prearrive", 1)
    try:
        for op in ("ag_gemm", "gemm_rs"):
            rows = {}
            # (tile, stream_k): the planner's pick with auto stream-K (Q28), 256x256 without
            # and with the stream-K tail, the 512x256 cluster tile
            # gemm_rs "+bf16wire": the non-conforming bf16 partial wire (Q14), half the bytes
            variants = (("auto", -1), ("256x256", 0), ("256x256+sk", 1), ("512x256", 0)) if op == "ag_gemm" else \
                (("auto", 0), ("256x256", 0), ("512x256", 0), ("256x256+bf16wire", 0))
            # two passes over the variants, best of each (the first launches after the main
            # legs run on a GPU still settling its clocks)
            for tile, sk in [v for _ in range(2) for v in variants]:
                d = dict(base, op=op, n_cta=sms)
                if op == "ag_gemm":
                    d.update(N=F, K=HIDDEN, backend="ce", stream_k=sk)
                else:
                    d.update(N=HIDDEN, K=F, rs_reduce="atomic")
                    if tile.endswith("+bf16wire"):
                        d["rs_wire"] = "bf16"
                if tile != "auto":
                    d["tile_m"], d["tile_n"] = (int(x) for x in tile.split("+")[0].split("x"))
                    if d["tile_m"] == 512:
                        d["n_cta"] = n4
                p = ao.Plan(ctxs[0], d)
                info = p.info()
                ao.debug_set("gemm_stream_k", sk if info["tile_m"] != 512 else 0)
                if op == "ag_gemm":
                    ms = timed(lambda: ao.ag_gemm(p, A[0], Bu[0], C_up))
                    g_ms = timed(lambda: ao.gemm(A_full, Bu[0], C_up, tile_m=info["tile_m"], tile_n=info["tile_n"]))
                else:
                    ms = timed(lambda: ao.gemm_rs(p, Cu[0], Bd[0], Cd0))
                    g_ms = timed(lambda: ao.gemm(Cu[0], Bd[0], C_dn, tile_m=info["tile_m"], tile_n=info["tile_n"]))
                ao.debug_set("gemm_stream_k", 0)
                sk_dp = json.loads(p.export_json()).get("sk_dp")
                p.close()
                if tile in rows:
                    ms = min(ms, rows[tile]["ms"])
                    g_ms = min(g_ms, rows[tile]["_g_ms"])
                rows[tile] = {"tile": [info["tile_m"], info["tile_n"], info["cta_group"]], "workers": info["n_cta"],
                              "stream_k_dp": sk_dp, "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
                              "gemm_only_tflops": round(flops / (g_ms * 1e-3) / 1e12, 1), "_g_ms": g_ms}
            for v in rows.values():
                v.pop("_g_ms", None)
            if op == "ag_gemm":
                cb = timed(lambda: torch.matmul(A_full, Bu[0].t(), out=C_up))
            else:
                cb = timed(lambda: torch.matmul(Cu[0], Bd[0].t(), out=C_dn))
            rows["cublas_tflops"] = round(flops / (cb * 1e-3) / 1e12, 1)
            res[op] = rows
    finally:
        ao.debug_set("prearrive", 0)
        for c in ctxs:
            c.close()
    res["shape"] = {"ag_gemm": [M, F, HIDDEN], "gemm_rs": [M, HIDDEN, F]}
    return res


def gemm_only_leg(torch, ao, pa, pr, A, Bu, Bd, W, M, F, args, dev, loop):
    """SURVEY §8(d) baseline (iii): the fused ops' GEMMs through the same kernel (tile shape,
    workers per rank, GROUP_M) with no transfers, flags or reduction -- ao_gemm_batched on
    pre-gathered A (one copy per rank, as the gathered buffers are) and on the RS operands
    into a bf16 scratch.  exposed communication = fused - GEMM-only."""
    ia, ir = pa[0].info(), pr[0].info()
    n = W if loop else 1
    A_full = torch.cat(A, 0) if loop else torch.empty(M, HIDDEN, dtype=torch.bfloat16, device=dev).normal_()
    A_g = [A_full.clone() for _ in range(n)]
    up = [torch.empty(M, F, dtype=torch.bfloat16, device=dev) for _ in range(n)]
    dn = [torch.empty(M, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in range(n)]

    def ag():
        ao.gemm_batched(A_g, Bu[:n], up, ia["tile_m"], ia["tile_n"], args.group_m, ia["n_cta"] * ia["cta_group"])

    def rs():
        ao.gemm_batched(up, Bd[:n], dn, ir["tile_m"], ir["tile_n"], args.group_m, ir["n_cta"] * ir["cta_group"])

    res = {}
    for name, fn in (("ag_gemm_ms", ag), ("gemm_rs_ms", rs)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = max(5, args.steps)  # as many launches per op as the timed region (same power regime)
        s.record()
        for _ in range(k):
            fn()
        e.record()
        torch.cuda.synchronize()
        res[name] = round(s.elapsed_time(e) / k, 4)
    del A_g, up, dn
    res["what"] = ("same tcgen05 kernel, tile and workers per rank, no transfers/flags/reduction "
                   "(ao_gemm_batched over the %d rank problems of one launch)" % n)
    return res


def nccl_baseline(torch, dist, A_shard, Bu, Bd, W, M, F, args, dev):
    """The paper's kernel-level-overlap baseline ("Triton kernels paired with
    NCCL collectives"): NCCL all_gather_into_tensor / reduce_scatter_tensor
    + cuBLAS GEMMs, the op split into s pieces with the collective of piece i+1 on a comm
    stream overlapping the GEMM of piece i.  RS partials in fp32 (cuBLAS bf16 x bf16 -> fp32,
    precision-matched with the fused kernel's fp32 wire) and bf16 (usual practice).  Best s
    in {1, 2, 4, 8} per precision; max over ranks."""
    S = M // W
    comm = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    C_up = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
    C_dn = torch.empty(S, HIDDEN, dtype=torch.bfloat16, device=dev)
    out = {}
    for prec in ("fp32", "bf16"):
        pdt = torch.float32 if prec == "fp32" else torch.bfloat16
        results = {}
        for s in (1, 2, 4, 8):
            if S % s or HIDDEN % s:
                continue
            rows, cols = S // s, HIDDEN // s
            g_bufs = [torch.empty(W * rows, HIDDEN, dtype=torch.bfloat16, device=dev) for _ in range(s)]
            parts = [torch.empty(M, cols, dtype=pdt, device=dev) for _ in range(s)]
            outs = [torch.empty(S, cols, dtype=pdt, device=dev) for _ in range(s)]
            ev_ag = [torch.cuda.Event() for _ in range(s)]
            ev_mm = [torch.cuda.Event() for _ in range(s)]
            ev_rs = [torch.cuda.Event() for _ in range(s)]

            def step():
                comm.wait_stream(main)
                with torch.cuda.stream(comm):  # AG pieces
                    for i in range(s):
                        dist.all_gather_into_tensor(g_bufs[i], A_shard[i * rows:(i + 1) * rows].contiguous())
                        ev_ag[i].record(comm)
                for i in range(s):
                    main.wait_event(ev_ag[i])
                    y = torch.matmul(g_bufs[i], Bu.t())  # [W*rows, F] -> rows p*S + i*rows
                    C_up.view(W, S, F)[:, i * rows:(i + 1) * rows].copy_(y.view(W, rows, F))
                for i in range(s):  # RS pieces (column splits)
                    if prec == "fp32":
                        torch.mm(C_up, Bd[i * cols:(i + 1) * cols].t(), out_dtype=torch.float32, out=parts[i])
                    else:
                        torch.matmul(C_up, Bd[i * cols:(i + 1) * cols].t(), out=parts[i])
                    ev_mm[i].record(main)
                    comm.wait_event(ev_mm[i])
                    with torch.cuda.stream(comm):
                        dist.reduce_scatter_tensor(outs[i], parts[i])
                        ev_rs[i].record(comm)
                for i in range(s):
                    main.wait_event(ev_rs[i])
                    C_dn[:, i * cols:(i + 1) * cols].copy_(outs[i])

            for _ in range(3):
                step()
            torch.cuda.synchronize()
            dist.barrier()
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = max(5, args.steps // 2)
            st.record(main)
            for _ in range(n):
                step()
            en.record(main)
            torch.cuda.synchronize()
            t = torch.tensor([st.elapsed_time(en) / n], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            results[s] = t.item()
        best = min(results, key=results.get)
        out[prec] = {"ms_per_step": round(results[best], 4),
                     "tflops": round(4.0 * M * FFN * HIDDEN / (results[best] * 1e-3) / 1e12, 2),
                     "best_split": best, "per_split_ms": {str(k): round(v, 4) for k, v in results.items()}}
    return {"what": "NCCL all_gather / reduce_scatter + cuBLAS, two-stream split overlap (best s; SURVEY 8(d)(ii))",
            "ms_per_step": out["fp32"]["ms_per_step"], "tflops": out["fp32"]["tflops"],
            "rs_partials_fp32": out["fp32"], "rs_partials_bf16": out["bf16"]}


def e2e_leg(torch, dist, args, A, Cd, step, barrier, world, flops_step, dev):
    """Same step through the public API with this step's activations copied from pinned
    host memory and its output read back to pinned host memory, every step.  Serving-style
    pipelining: inputs/outputs are double-buffered and the copies run on two copy streams,
    so step i+1's upload and step i's download overlap step i's compute (PCIe duplex).  The
    ranks' shards of a step are one contiguous buffer each way (one copy per direction per
    step; the per-rank tensors the ops take are row views of it), so the host issues few
    calls per step."""
    r = len(A)
    S_in, S_out = A[0].shape[0], Cd[0].shape[0]
    hA = torch.cat([a.cpu() for a in A], 0).pin_memory()
    hC = [torch.empty((r * S_out,) + tuple(Cd[0].shape[1:]), dtype=Cd[0].dtype, pin_memory=True) for _ in range(2)]
    dA_all = [torch.empty(hA.shape, dtype=hA.dtype, device=dev) for _ in range(2)]
    dC_all = [torch.empty(hC[0].shape, dtype=hC[0].dtype, device=dev) for _ in range(2)]
    dA = [[t[k * S_in:(k + 1) * S_in] for k in range(r)] for t in dA_all]
    dC = [[t[k * S_out:(k + 1) * S_out] for k in range(r)] for t in dC_all]
    stream = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    computed = [torch.cuda.Event() for _ in range(2)]
    uploaded = [torch.cuda.Event() for _ in range(2)]
    downloaded = [torch.cuda.Event() for _ in range(2)]
    n = max(4, args.steps // 2)
    # per-step diagnosis: the copy and compute spans as they ran inside the pipelined loop
    ev_up = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n + 2)]
    ev_cp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n + 2)]
    ev_dn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n + 2)]

    def upload(i):
        b = i % 2
        up.wait_event(computed[b])  # compute of step i-2 finished reading dA[b]
        ev_up[i][0].record(up)
        with torch.cuda.stream(up):
            dA_all[b].copy_(hA, non_blocking=True)
        ev_up[i][1].record(up)
        uploaded[b].record(up)

    def run(i):
        b = i % 2
        stream.wait_event(uploaded[b])
        stream.wait_event(downloaded[b])  # dC[b] of step i-2 has been read back
        ev_cp[i][0].record(stream)
        step(A_in=dA[b], C_out=dC[b])
        ev_cp[i][1].record(stream)
        computed[b].record(stream)
        down.wait_event(computed[b])
        ev_dn[i][0].record(down)
        with torch.cuda.stream(down):
            hC[b].copy_(dC_all[b], non_blocking=True)
        ev_dn[i][1].record(down)
        downloaded[b].record(down)

    for b in range(2):
        computed[b].record(stream)
        downloaded[b].record(down)
    upload(0)
    run(0)
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    t_host = time.perf_counter()
    upload(1)
    for i in range(1, n + 1):
        if i + 1 <= n:
            upload(i + 1)
        run(i)
    host_ms = (time.perf_counter() - t_host) * 1e3 / n
    stream.wait_event(downloaded[n % 2])
    e.record(stream)
    barrier()
    ms = s.elapsed_time(e) / n
    med = lambda evs: round(statistics.median(a.elapsed_time(b) for a, b in evs[2:n]), 4)
    spans = {"upload_ms": med(ev_up), "compute_ms": med(ev_cp), "download_ms": med(ev_dn),
             "compute_start_gap_ms": round(statistics.median(ev_cp[i][0].elapsed_time(ev_cp[i + 1][0])
                                                             for i in range(2, n - 1)), 4)}
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    h2d = hA.numel() * hA.element_size()
    d2h = hC[0].numel() * hC[0].element_size()
    # the PCIe bound: this step's copies alone, each direction, then both at once
    link = {}
    for name, st, dst, src in (("h2d_gbs_alone", up, dA_all[0], hA), ("d2h_gbs_alone", down, hC[0], dC_all[0])):
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(st)
        with torch.cuda.stream(st):
            for _ in range(3):
                dst.copy_(src, non_blocking=True)
        c1.record(st)
        torch.cuda.synchronize()
        link[name] = round(3 * src.numel() * src.element_size() / (c0.elapsed_time(c1) * 1e-3) / 1e9, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for st, dst, src in ((up, dA_all[0], hA), (down, hC[0], dC_all[0])):
        with torch.cuda.stream(st):
            for _ in range(3):
                dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    link["duplex_gbs_per_direction"] = round(3 * h2d / (time.perf_counter() - t0) / 1e9, 1)
    link["io_bound_ms_per_step"] = round(max(h2d, d2h) / (link["duplex_gbs_per_direction"] * 1e9) * 1e3, 4)
    if world > 1:
        h2d *= world
        d2h *= world
    return {"value": round(flops_step / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "pipelining": "double-buffered; H2D of step i+1 and D2H of step i overlap step i's compute",
            "host_ms_per_step": round(host_ms, 4), "pcie": link, "spans_in_loop": spans}


# ============================================================================ CPU oracle
def _threads():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info if i.get("user_api") == "blas"] or [os.cpu_count()])
    except Exception:
        return os.cpu_count()


def oracle_sample(W, M, i, cache):
    """One bounded sample of the workload on the CPU oracle (oracle/numeric.py as it
    stands): for rank r = i % W and row block j = (i // W) % W, the AG-GEMM output rows
    [j*S, (j+1)*S) of rank r and the GEMM-RS output rows [j*S/W, (j+1)*S/W) of owner r's
    shard.  That is 1/W^2 of one step's FLOPs.  Returns the FLOPs done."""
    from oracle import numeric as on
    from synthetic import inputs as si
    F = FFN // W
    S = M // W
    if "A" not in cache:
        A, Bu = si.ag_inputs(W, M, HIDDEN, F)
        Ars, Bd = si.rs_inputs(W, M, F, HIDDEN)
        cache["A"] = [si.to_f64(a) for a in A]
        cache["Bu"] = [si.to_f64(b) for b in Bu]
        cache["Ars"] = [si.to_f64(a) for a in Ars]
        cache["Bd"] = [si.to_f64(b) for b in Bd]
    r, j = i % W, (i // W) % W
    on.ag_gemm_rows(cache["A"], cache["Bu"][r], list(range(j * S, (j + 1) * S)))
    sub = S // W
    on.gemm_rs_rows(cache["Ars"], cache["Bd"], r, list(range(j * sub, (j + 1) * sub)))
    return 2.0 * S * F * HIDDEN + W * 2.0 * sub * F * HIDDEN


def cpu_baseline(W, M, budget_s=12.0):
    cache = {}
    oracle_sample(W, M, 0, cache)  # input generation + BLAS warm-up, untimed
    t0 = time.time()
    flops, done = 0.0, 0
    while time.time() - t0 < budget_s:
        flops += oracle_sample(W, M, done % (W * W), cache)
        done += 1
    dt = time.time() - t0
    return {"value": round(flops / dt / 1e12, 5), "unit": "TFLOP/s", "cores": _threads(), "kind": "oracle",
            "sample": f"{done} samples (cycling) of 1/{W * W} of a step each (AG-GEMM rows [{M // W}x{FFN // W}] of one rank + "
                      f"GEMM-RS rows [{M // W // W}x{HIDDEN}] of one owner, fp64 numpy), {dt:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    W = args.tp if world == 1 else world
    M = args.tokens
    cache = {}
    oracle_sample(W, M, 0, cache)  # input generation, untimed
    times, flops = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.time()
        f = oracle_sample(W, M, i % W, cache)
        dt = time.time() - t0
        if i >= args.warmup:
            times.append(dt)
            flops.append(f)
    tot = sum(times)
    value = sum(flops) / tot / 1e12
    ms = tot / len(times) * 1e3
    cb = {"value": round(value, 5), "unit": "TFLOP/s", "cores": _threads(), "kind": "oracle",
          "sample": f"each step = 1/{W * W} of the FFN pair (one rank's AG-GEMM row block + one owner's GEMM-RS "
                    f"row block), fp64 numpy"}
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"llama3-8b-tp{W}-ffn-pair-{'loopback' if world == 1 else 'nvlink'}",
                      "tokens": M, "hidden": HIDDEN, "ffn": FFN, "tp": W},
           "cpu_baseline": cb,
           "e2e": {"value": round(value, 5), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# AO_BENCH_SHARED_GPU=1 (scripts/bench_shared_gpu.sh): run the N > 1 code path with every rank
# on GPU 0 under MPS -- gloo process group, each rank's persistent kernels on SMs / N CTAs,
# the NCCL two-stream baseline skipped.  A functional check of the one-rank-per-process bench
# path on a single-GPU box; its numbers are not the multi-GPU measurement.
SHARED_GPU = os.environ.get("AO_BENCH_SHARED_GPU") == "1"


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if SHARED_GPU:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        if SHARED_GPU:  # test harness: every rank on GPU 0 (under MPS); NCCL refuses shared GPUs
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
