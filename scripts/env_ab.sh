#!/bin/bash
# A/B one build under two environment settings: ENV_A / ENV_B (e.g. "DMLP_YFLAT=0")
# needs a library built with the plan-override knobs: DMLP_NVCC_FLAGS=-DDMLP_EXPERIMENT_KNOBS python -m paper_1003_0358_b200.build --force
for round in 1 2; do
for v in A B; do
  e=ENV_$v
  echo "== $v (${!e})"; env ${!e} timeout 300 python scripts/quick_perf.py ${N:-20000} auto ${CFGS:-C1,C4,C5} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
done; done
