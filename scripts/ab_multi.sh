#!/bin/bash
# A/B/n: package copies under scripts/libs_ab/<name> (each with its own python +
# libdmlp.so) and the working tree ("work"), alternating, two rounds, same box.
CFGS=${CFGS:-C1,C2,C3,C4,C5}
N=${N:-20000}
VARS=${VARS:-head work}
for round in 1 2; do
  for v in $VARS; do
    echo "== $v (round $round)"
    if [ "$v" = work ]; then
      timeout 300 python scripts/quick_perf.py $N auto $CFGS 2>&1 | grep cfg
    else
      (cd scripts/libs_ab/$v && timeout 300 python ../../quick_perf.py $N auto $CFGS 2>&1 | grep cfg)
    fi
  done
done | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('=='):
        print(l.strip()); continue
    try:
        d = json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])
    except Exception:
        print(l.strip()[:200])
"
