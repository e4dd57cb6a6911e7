"""Device trace of the SP attention ping-pong kernel (Llama-3-8B: 32 heads, 32768 tokens over
8 loopback ranks, time-sliced): per role, how long it waits and works per KV block.
TR kinds: load = producer waiting for a free K stage, mma = MMA warp waiting for a tile's P,
wait = softmax waiting for S, epilogue = softmax compute of one block."""
import json
import os
import sys
import collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_20595_b200 as ao
from synthetic import inputs as si

W, H, Stot = 8, 32, int(sys.argv[2]) if len(sys.argv) > 2 else 32768
S = Stot // W
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.json"
Q, K, V = si.attn_inputs(W, H, S, 128)
d = dict(op="sp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=S, backend="ce", n_cta=148, timeout_ns=10_000_000_000)
ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
plans = [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]
dQ, dK, dV = [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V]
O = [torch.empty_like(q) for q in dQ]
for _ in range(3):
    ao.sp_attn_group(plans, dQ, dK, dV, O)
torch.cuda.synchronize()
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record()
for _ in range(5):
    ao.sp_attn_group(plans, dQ, dK, dV, O)
e_.record()
torch.cuda.synchronize()
ms = s_.elapsed_time(e_) / 5
print(f"untraced: {ms:.3f} ms  {4.0 * Stot * Stot * 128 * H / (ms * 1e-3) / 1e12:.0f} TFLOP/s")
ctxs[0].trace_enable(1 << 24)
ao.sp_attn_group(plans, dQ, dK, dV, O)
ctxs[0].trace_dump(out)
ctxs[0].trace_enable(0)
ev = json.load(open(out))["traceEvents"]
t0 = min(e["ts"] for e in ev)
span = max(e["ts"] + e["dur"] for e in ev) - t0
print(f"events {len(ev)}, span {span:.0f} us")
by = collections.defaultdict(list)
for e in ev:
    by[e["cat"]].append(e["dur"])
for k, v in sorted(by.items()):
    v.sort()
    print(f"  {k:9s} n={len(v):8d} mean={sum(v) / len(v):7.3f} us  p50={v[len(v) // 2]:7.3f}  p90={v[int(len(v) * 0.9)]:7.3f}  "
          f"total/CTA={sum(v) / 148:9.1f} us")
