"""Per cluster type (4-CTA cluster vs CTA pair, told apart by the CTA ids the probe showed:
blocks >= 132 were pairs) MMA and epilogue statistics of a hybrid-cluster trace: mean MMA
span per tile pass, MMA-busy fraction, the gaps between a CTA's consecutive MMAs, waits.
usage: python scripts/hyb_trace.py TRACE.json [first_pair_cta] [launch]"""
import collections
import json
import sys

ev = json.load(open(sys.argv[1]))["traceEvents"]
fp = int(sys.argv[2]) if len(sys.argv) > 2 else 132
L = int(sys.argv[3]) if len(sys.argv) > 3 else sorted({e.get("args", {}).get("launch", 0) for e in ev})[-1]
ev = [e for e in ev if e.get("args", {}).get("launch", 0) == L]
t0 = min(e["ts"] for e in ev)
span = max(e["ts"] + e["dur"] for e in ev) - t0
print(f"launch {L}: {len(ev)} events, span {span:.1f} us")
by = collections.defaultdict(lambda: collections.defaultdict(list))
for e in ev:
    by[(e["cat"], e["tid"] // 8 >= fp)][e["tid"]].append((e["ts"] - t0, e["dur"]))
clk = [(int(e["name"].split()[1]), e["dur"]) for e in ev if e["cat"] == "clock" and e["dur"] > 0]
if clk:
    mhz = sorted(c / d for c, d in clk)
    print(f"  SM clock over MMA spans: median {mhz[len(mhz) // 2]:.0f} MHz, p10 {mhz[len(mhz) // 10]:.0f}, "
          f"p90 {mhz[9 * len(mhz) // 10]:.0f}")
for (cat, pair), d in sorted(by.items()):
    if cat == "clock":
        continue
    n = sum(len(v) for v in d.values())
    tot = sum(x[1] for v in d.values() for x in v)
    gaps = []
    for v in d.values():
        v.sort()
        gaps += [v[i + 1][0] - (v[i][0] + v[i][1]) for i in range(len(v) - 1)]
    last = max(x[0] + x[1] for v in d.values() for x in v)
    print(f"  {cat:8s} {'pair' if pair else 'quad'} ctas={len(d):4d} n={n:6d} mean={tot / max(n, 1):7.2f}us "
          f"busy={tot / len(d) / span:6.1%} gap_mean={sum(gaps) / max(len(gaps), 1):6.2f}us last_end={last:8.1f}")
