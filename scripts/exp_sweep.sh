#!/bin/bash
# Timing sweep of bench.py variants (kernel ms only; experiment knobs make results invalid).
# usage: scripts/exp_sweep.sh OUT "args1" "args2" ...
out=$1; shift
: > "$out"
for a in "$@"; do
  r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-check $a 2>&1 | tail -1)
  k=$(echo "$r" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d["kernels_ms"], d["value"])
except Exception as e: print("ERR", e)')
  echo "$a => $k" >> "$out"
done
