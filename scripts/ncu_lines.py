"""Top CUDA source lines by warp-stall samples (ncu source page, cuda+sass view).
usage: python scripts/ncu_lines.py REPORT LAUNCH_INDEX [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ci = hdr.index("Warp Stall Sampling (All Samples)")
line_samples = collections.Counter()
line_src = {}
cur = None
for r in rows:
    if not r or r[0] in ("Line No", "File Path", "Function Name"):
        continue
    if r[0]:
        cur = r[0]
        line_src[cur] = r[1].strip()
    try:
        line_samples[cur] += float(r[ci])
    except (ValueError, IndexError):
        pass
tot = sum(line_samples.values())
print(f"total samples {tot:.0f}")
for ln, v in line_samples.most_common(n):
    print(f"{100 * v / tot:5.1f}% L{ln:>5s} {line_src.get(ln, '')[:100]}")
