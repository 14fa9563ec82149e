#!/bin/bash
# Round-2 evidence run on one B200: GPU tests, bench lines of every config
# (C3 also with every hidden layer streamed from L2, as BASELINE.json labels
# it), the ncu launch list of the default bench command, the C4 timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gputest.log
timeout 600 python bench.py > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
for c in C1 C2 C3 C5; do
  lc=$(echo $c | tr A-Z a-z)
  timeout 600 python bench.py --config $c --cpu-seconds 4 > gpurun_out/r2_bench_$lc.json 2> gpurun_out/r2_bench_$lc.err
done
timeout 600 python bench.py --config C3 --residency l2 --cpu-seconds 4 > gpurun_out/r2_bench_c3_l2.json 2> gpurun_out/r2_bench_c3_l2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 0 \
  > gpurun_out/r2_launches_bench.log 2>&1
timeout 300 python scripts/trace_perf.py C4 > gpurun_out/r2_trace_c4.txt 2>&1
