"""Copy a round's GPU evidence from gpurun_out/ into profiles/ (tracked):
bench line, launch list (+ kernel share), ncu full summary/raw CSV, hot SASS lines,
trace summary, traffic.json.  usage: python scripts/update_profiles.py r01"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout


os.makedirs(P, exist_ok=True)
for src, dst in (("bench_%s.json" % tag, "%s_bench.json" % tag), ("bench_ref_%s.json" % tag, "%s_bench_reference.json" % tag),
                 ("launches_%s.csv" % tag, "%s_launches.csv" % tag), ("gemm_perf_%s.txt" % tag, "%s_gemm_perf.txt" % tag)):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))

# launch-list shares
lp = os.path.join(G, "launches_%s.csv" % tag)
if os.path.exists(lp):
    rows = list(csv.reader(open(lp)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    tot, n = {}, {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        k = d["Kernel Name"][:70]
        tot[k] = tot.get(k, 0) + float(d["Metric Value"])
        n[k] = n.get(k, 0) + 1
    s = sum(tot.values())
    with open(os.path.join(P, "%s_launch_shares.txt" % tag), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised) over\n"
                "`python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-baseline`\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{v / 1e3:10.1f} us  {n[k]:3d} launches  {100 * v / s:5.1f}%  {k}\n")

rep = os.path.join(G, "prof_%s_final.ncu-rep" % tag)
if os.path.exists(rep):
    raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
    open(os.path.join(P, "%s_ncu_full_raw.csv" % tag), "w").write(raw)
    summ = run([sys.executable, "scripts/ncu_summary.py", rep, "--json", os.path.join(P, "%s_ncu_full_summary.json" % tag)])
    open(os.path.join(P, "%s_ncu_full_summary.txt" % tag), "w").write(summ)
    for i, name in ((0, "ag"), (1, "rs")):
        hot = run([sys.executable, "scripts/ncu_hot.py", rep, str(i), "20"]).splitlines()
        open(os.path.join(P, "%s_ncu_hot_%s.txt" % (tag, name)), "w").write("\n".join(hot[::2]) + "\n")
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    tr = {"_source": "profiles/%s_ncu_full_raw.csv: ncu --set full --clock-control none, one launch each of the "
                     "bench's fused kernels (loopback TP=8, default config); dram__bytes_read.sum + "
                     "dram__bytes_write.sum per launch" % tag}
    for r, name in zip(rows[2:4], ("ag_gemm", "gemm_rs")):
        tot = 0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            j = hdr.index(m)
            tot += float(r[j]) * scale[units[j]]
        tr[name] = int(tot)
    json.dump(tr, open(os.path.join(P, "traffic.json"), "w"), indent=1)
rep = os.path.join(G, "prof_%s_a2a.ncu-rep" % tag)
if os.path.exists(rep):  # A2A-GEMM (NEXT-3) kernel, one launch
    raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
    open(os.path.join(P, "%s_ncu_a2a_raw.csv" % tag), "w").write(raw)
    summ = run([sys.executable, "scripts/ncu_summary.py", rep])
    open(os.path.join(P, "%s_ncu_a2a_summary.txt" % tag), "w").write(summ)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    tot = 0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        j = hdr.index(m)
        tot += float(rows[2][j]) * scale[units[j]]
    tp_ = os.path.join(P, "traffic.json")
    tr = json.load(open(tp_)) if os.path.exists(tp_) else {}
    tr["a2a_gemm"] = int(tot)
    json.dump(tr, open(tp_, "w"), indent=1)
rep = os.path.join(G, "prof_%s_attn.ncu-rep" % tag)
if os.path.exists(rep):  # SP attention (NEXT-4) kernel, one launch
    open(os.path.join(P, "%s_ncu_attn_summary.txt" % tag), "w").write(run([sys.executable, "scripts/ncu_summary.py", rep]))
    open(os.path.join(P, "%s_ncu_attn_lines.txt" % tag), "w").write(run([sys.executable, "scripts/ncu_lines.py", rep, "0", "30"]))
tp = os.path.join(G, "trace_%s.json" % tag)
if os.path.exists(tp):
    open(os.path.join(P, "%s_trace_summary.txt" % tag), "w").write(run([sys.executable, "scripts/trace_summary.py", tp]))
print("updated profiles/ for", tag)
