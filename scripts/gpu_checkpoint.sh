#!/bin/bash
# One GPU round trip: tests, bench line, launch list, ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --samples 4000 \
  --deform-images 20000 --cpu-seconds 0 > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train -s 1 -c 1 \
  -o gpurun_out/train_c4 python scripts/ncu_train.py C4 2000 auto > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train -s 1 -c 1 \
  -o gpurun_out/train_c1 python scripts/ncu_train.py C1 2000 auto > gpurun_out/ncu_c1.log 2>&1
tail -3 gpurun_out/gputests.log; cat gpurun_out/bench.json
