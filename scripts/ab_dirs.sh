#!/bin/bash
# A/B the working tree against a baseline package copy (scripts/libs_ab/head,
# its own python + libdmlp.so) on the same box, alternating, two rounds.
CFGS=${CFGS:-C1,C2,C3,C4,C5}
N=${N:-20000}
for round in 1 2; do
  echo "== head (round $round)"
  (cd scripts/libs_ab/head && timeout 300 python ../../quick_perf.py $N auto $CFGS 2>&1 | grep cfg)
  echo "== work (round $round)"
  timeout 300 python scripts/quick_perf.py $N auto $CFGS 2>&1 | grep cfg
done
