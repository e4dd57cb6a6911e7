#!/bin/bash
# A/B timing of the in-tree libautooverlap.so against another build in ONE GPU session
# (boxes differ by a few percent, so compare only within a call).
# usage: scripts/ab_lib.sh OTHER_LIB.so OUT_PREFIX "bench args" ...   (runs new, other, new, other)
other=$1; pre=$2; shift 2
lib=paper_2601_20595_b200/libautooverlap.so
cp $lib build/lib_new.so
for rep in 1 2; do
  cp build/lib_new.so $lib; scripts/exp_sweep.sh ${pre}_new$rep.txt "$@"
  cp "$other" $lib; scripts/exp_sweep.sh ${pre}_other$rep.txt "$@"
done
cp build/lib_new.so $lib
head ${pre}_*.txt
