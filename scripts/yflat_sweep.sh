#!/bin/bash
# y-word layout A/B with the knob build: DMLP_YFLAT unset (auto: flat when R % 4 != 0) vs 0 (slots)
cd scripts/libs_ab/knobs
for round in 1 2; do
  for y in auto 0; do
    if [ $y = auto ]; then unset DMLP_YFLAT; else export DMLP_YFLAT=$y; fi
    echo "== yflat=$y (round $round)"
    timeout 300 python ../../quick_perf.py 20000 auto ${CFGS:-C4} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
  done
done
