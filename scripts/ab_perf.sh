#!/bin/bash
# A/B two builds of libdmlp.so on the same box: scripts/libs_ab/{a,b}.so
for round in 1 2; do
for v in ${VARS:-a b}; do
  cp scripts/libs_ab/$v.so paper_1003_0358_b200/libdmlp.so
  echo "== $v"; timeout 300 python scripts/quick_perf.py 20000 auto ${CFGS:-C1,C4,C5} 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])"
done; done
