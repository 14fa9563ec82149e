for round in 1 2; do for v in head work; do
  if [ $v = work ]; then d=.; else d=scripts/libs_ab/$v; fi
  echo "== $v C3 all-L2 (round $round)"; (cd $d && timeout 200 python $OLDPWD/scripts/quick_perf.py 20000 l2 C3 2>&1 | grep cfg | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['where'], d['us_per_sample'], d['samples_s'])")
done; done
