#!/bin/bash
# GPU evidence for profiles/ (run under gpurun; then `python scripts/update_profiles.py TAG` here).
tag=${1:-r01}
G=gpurun_out
python bench.py > $G/bench_$tag.log 2>&1; tail -1 $G/bench_$tag.log > $G/bench_$tag.json
python bench.py --impl reference --steps 3 --warmup 3 > $G/bench_ref_$tag.log 2>&1; tail -1 $G/bench_ref_$tag.log > $G/bench_ref_$tag.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-a2a --no-attn --no-check --trace $G/trace_$tag > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $G/launches_$tag.csv \
  python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-baseline --no-a2a --no-attn > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -f \
  -o $G/prof_${tag}_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-a2a --no-attn --no-check > $G/ncu_full_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'fused_kernel<.int.256, .int.3' -s 1 -c 1 -f \
  -o $G/prof_${tag}_a2a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-attn --no-check > $G/ncu_a2a_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn -s 1 -c 1 -f \
  -o $G/prof_${tag}_attn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-baseline --no-ar --no-a2a --no-check --attn-seq 16384 > $G/ncu_attn_$tag.log 2>&1
python scripts/gemm_perf.py > $G/gemm_perf_$tag.txt 2>&1
tail -1 $G/bench_$tag.json | cut -c1-400
