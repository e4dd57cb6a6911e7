"""Top SASS instructions by warp-stall samples from an ncu report (source page).
usage: python scripts/ncu_hot.py REPORT LAUNCH_INDEX [N]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = hdr.index("Warp Stall Sampling (All Samples)")
si = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = []
tot = 0
for r in rows[2:]:
    try:
        v = float(r[ci])
    except (ValueError, IndexError):
        continue
    tot += v
    reasons = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:3]
    data.append((v, r[0][-5:], r[si].strip(), reasons))
data.sort(reverse=True)
print(f"total samples {tot:.0f}")
for v, a, s, rs in data[:n]:
    print(f"{100 * v / tot:5.1f}% {a} {s[:60]:60s} " + " ".join(f"{h[6:]}={x:.0f}" for x, h in rs if x > 0))
