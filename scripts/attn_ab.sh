#!/bin/bash
# A/B of SP-attention timings across prebuilt libraries in ONE GPU session.
# usage: scripts/attn_ab.sh OUT lib1.so lib2.so ...   (each lib twice, interleaved)
out=$1; shift
lib=paper_2601_20595_b200/libautooverlap.so
cp $lib build/lib_keep.so
: > "$out"
for rep in 1 2; do
  for l in "$@"; do
    cp "$l" $lib
    r=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-a2a --no-check 2>&1 | tail -1)
    echo "$l $(echo "$r" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read())["sp_attn"]; print(d["tflops"], d["causal_tflops"], d["sdpa_tflops"])
except Exception as e: print("ERR", e)')" >> "$out"
  done
done
cp build/lib_keep.so $lib
cat "$out"
