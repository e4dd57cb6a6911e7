"""Measured SP-attention error vs the fp64 oracle (elementwise / Frobenius) and vs the
bf16-P oracle variant, per test configuration (Q27)."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from oracle import attn as oatt
from oracle import numeric as on
from synthetic import inputs as si
import paper_2601_20595_b200.api as ao

for W, H, S, C, causal in [(1, 2, 256, 128, 0), (2, 2, 256, 256, 0), (4, 2, 128, 128, 0), (8, 1, 256, 128, 0),
                           (4, 2, 512, 128, 0), (4, 2, 512, 128, 1), (8, 2, 1024, 256, 1), (8, 2, 1024, 256, 0)]:
    d = dict(op="sp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=C, backend="ce", n_cta=max(1, 148 // W),
             timeout_ns=2_000_000_000, causal=causal)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    plans = [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=W * 10 + H)
    O = [torch.empty_like(q, device="cuda") for q in Q]
    ao.sp_attn_group(plans, [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V], O)
    torch.cuda.synchronize()
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for r in range(W):
        ref = oatt.sp_attention(Qn, Kn, Vn, r, 128 ** -0.5, causal=bool(causal))
        got = O[r].float().cpu().numpy()
        ok, e, f = on.check_tolerance(got, ref, frob_rel=1.0)
        res = {"W": W, "H": H, "S": S, "causal": causal, "rank": r, "elem": e, "frob": f}
        if hasattr(oatt, "sp_attention_p_bf16"):
            refb = oatt.sp_attention_p_bf16(Qn, Kn, Vn, r, 128 ** -0.5, causal=bool(causal))
            _, eb, fb = on.check_tolerance(got, refb, frob_rel=1.0)
            _, eo, fo = on.check_tolerance(refb, ref, frob_rel=1.0)
            res.update(frob_vs_bf16p=fb, elem_vs_bf16p=eb, bf16p_oracle_frob_vs_exact=fo)
        print(json.dumps(res))
    for c in ctxs:
        c.close()
