#!/bin/bash
# Layer-0 row-group sweep with the knob build (scripts/libs_ab/knobs, -DDMLP_EXPERIMENT_KNOBS).
cd scripts/libs_ab/knobs
for round in 1 2; do
  for g in auto 0 1 2 3; do
    if [ $g = auto ]; then unset DMLP_GS; else export DMLP_GS="$g"; fi
    echo "== L0 gs=$g (round $round)"
    timeout 300 python ../../quick_perf.py 20000 auto ${CFGS:-C2,C3,C4} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
  done
done
