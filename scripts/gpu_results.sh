#!/bin/bash
# Bench lines for every headline config (profiles/r1_bench_c*.json) + trace of C4.
mkdir -p gpurun_out
for c in C1 C2 C3 C4 C5; do
  lc=$(echo $c | tr A-Z a-z)
  timeout 600 python bench.py --config $c > gpurun_out/bench_$lc.json 2> gpurun_out/bench_$lc.err
done
timeout 300 python scripts/trace_perf.py C4 > gpurun_out/trace_c4.txt 2>&1
