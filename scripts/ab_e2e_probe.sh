#!/bin/bash
# A/B of scripts/e2e_probe.py across prebuilt libraries in ONE GPU session.
# usage: scripts/ab_e2e_probe.sh lib1.so lib2.so ...
lib=paper_2601_20595_b200/libautooverlap.so
cp $lib build/lib_keep_e2e.so
for rep in 1 2; do
  for l in "$@"; do
    cp "$l" $lib
    echo "== $l"; timeout 300 python scripts/e2e_probe.py 2>&1 | tail -8
  done
done
cp build/lib_keep_e2e.so $lib
