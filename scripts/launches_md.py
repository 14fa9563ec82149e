"""ncu gpu__time_duration launch list csv -> markdown summary.

    python scripts/launches_md.py [csv] [out.md] [round tag] [command]
"""
import collections
import csv
import sys

CSV = sys.argv[1] if len(sys.argv) > 1 else "profiles/r1_launches.csv"
OUT = sys.argv[2] if len(sys.argv) > 2 else "profiles/r1_launches.md"
TAG = sys.argv[3] if len(sys.argv) > 3 else "Round 1"
CMD = sys.argv[4] if len(sys.argv) > 4 else None

rows = [r for r in csv.reader(open(CSV)) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split('(')[0].replace('void ', '')
    scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1, 'msecond': 1}
    ms = scale.get(r[ui], 1e-6) * float(r[vi].replace(',', ''))
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(a[1] for a in agg.values())
CMD = CMD or ("ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python "
              "bench.py --steps 2 --warmup 3 --samples 4000 --deform-images 20000 --cpu-seconds 0")
out = [f"# {TAG} launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
       f"Command (one B200, gpurun): `{CMD}`", "",
       "Cold-cache, serialised per-launch times: compare SHARES, not absolutes. Raw CSV: "
       f"`{CSV}`.", "",
       "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, (n, ms) in agg.items():
    out.append(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
out += ["", "`k_train<NRL, RR, RC, RS, FEAT, PROF>` is the persistent on-line BP kernel (register "
        "plan; FEAT = residency paths compiled in, 1 smem + 2 L2 + 4 L1-cached streamed rows; PROF = 1 is the profiling "
        "instance the bench launches once for the per-phase profile); one launch trains a whole step of samples. `k_gemm_tanh` + "
        "`k_out_rank` are the validation/evaluation forward; `k_deform` the per-epoch "
        "deformation; `k_pack`/`k_unpack` the reference-layout conversions."]
open(OUT, 'w').write("\n".join(out) + "\n")
print("\n".join(out))
