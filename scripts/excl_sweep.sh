#!/bin/bash
# Residency A/B with the knob build (scripts/libs_ab/knobs, -DDMLP_EXPERIMENT_KNOBS):
# DMLP_SMEM_EXCLUDE=m keeps the hidden layers in bitmask m out of shared memory
# (C4: m=1 streams layer 0 instead of layer 3).
cd scripts/libs_ab/knobs
for round in 1 2; do
  for ex in ${EXCL:-0 1}; do
    echo "== smem exclude $ex (round $round)"
    DMLP_SMEM_EXCLUDE=$ex timeout 300 python ../../quick_perf.py 20000 auto ${CFGS:-C4} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
  done
done
