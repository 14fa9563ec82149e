#!/bin/bash
# A/B the per-layer row-group mapping (DMLP_GS, capi.cu choose_mapping) on one box.
# needs a library built with the plan-override knobs: DMLP_NVCC_FLAGS=-DDMLP_EXPERIMENT_KNOBS python -m paper_1003_0358_b200.build --force
# usage: CFG=C4 GS_LIST="auto 2 3" bash scripts/gs_ab.sh
for round in 1 2; do
for g in ${GS_LIST:-auto}; do
  if [ "$g" = auto ]; then unset DMLP_GS; else export DMLP_GS=$g; fi
  echo "== ${CFG:-C4} gs=$g"; timeout 300 python scripts/quick_perf.py ${N:-20000} auto ${CFG:-C4} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
done; done
unset DMLP_GS
