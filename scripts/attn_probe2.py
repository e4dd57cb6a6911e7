"""Probe: a small SP-attention world, then a large one in the same process (timeouts 2 s):
reports elapsed time and any device timeout.  usage: python scripts/attn_probe2.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao
from synthetic import inputs as si


def run(W, H, S, n_cta, C=None):
    Q, K, V = si.attn_inputs(W, H, S, 128)
    d = dict(op="sp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=C or S, backend="ce", n_cta=n_cta,
             timeout_ns=2_000_000_000)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    plans = [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
    O = [torch.empty_like(q, device="cuda") for q in Q]
    t = time.time()
    ao.sp_attn_group(plans, [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V], O)
    torch.cuda.synchronize()
    dt = time.time() - t
    err = None
    for c in ctxs:
        try:
            c.check_async()
        except ao.AOError as e:
            err = str(e)
    print(f"W={W} H={H} S={S} n_cta={n_cta} C={C or S}: {dt * 1e3:.1f} ms err={err}", flush=True)
    for p in plans:
        p.close()
    for c in ctxs:
        c.close()


if os.environ.get("EXP"):
    ao.debug_set("exp", int(os.environ["EXP"]))
for cfg in [(8, 8, 2048, 148), (8, 32, 512, 148), (8, 32, 2048, 148), (8, 32, 4096, 148)]:
    run(*cfg)
