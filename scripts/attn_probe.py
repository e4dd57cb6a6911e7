"""Probe: run SP attention at one size (loopback, time-sliced) and compare sampled rows with
the fp64 oracle.  usage: python scripts/attn_probe.py W H S"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_20595_b200 as ao
from oracle import attn as oatt
from synthetic import inputs as si

W, H, S = (int(x) for x in sys.argv[1:4])
Q, K, V = si.attn_inputs(W, H, S, 128)
d = dict(op="sp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=S, backend="ce", n_cta=148, timeout_ns=5_000_000_000)
ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
plans = [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
O = [torch.full_like(q, float("nan"), device="cuda") for q in Q]
t = time.time()
ao.sp_attn_group(plans, [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V], O)
torch.cuda.synchronize()
dt = time.time() - t
for c in ctxs:
    c.check_async()
Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
ref = oatt.sp_attention_rows(Qn, Kn, Vn, 0, 128 ** -0.5, [0, H - 1], np.array([0, S - 1]))
got = O[0][[0, H - 1]][:, [0, S - 1]].float().cpu().numpy()
print(f"W={W} H={H} S={S}: {dt * 1e3:.1f} ms, max abs err {np.abs(got - ref).max():.3e}, nan {np.isnan(got).any()}")
