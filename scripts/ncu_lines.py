"""Warp-stall samples of one ncu capture aggregated per source line.

    python scripts/ncu_lines.py capture.ncu-rep object.o kernel_mangled_substring [top]

ncu's CLI source page carries metrics only for SASS; this joins it with the
line table of the same cubin (nvdisasm -gi) to attribute stalls to lines,
innermost location plus the kernel-level call site.
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.splitlines()
addr_line = {}
inside = False
cur, site = "?", "?"
chain = []
for ln in dis:
    if ln.startswith(".text."):
        inside = kname in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        chain.append(os.path.basename(m.group(1)) + ":" + m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        if chain:  # innermost first, the kernel-level line last
            cur = chain[0]
            site = next((c for c in reversed(chain) if c.startswith("train_kernel")), chain[-1])
            chain = []
        addr_line[int(m.group(1), 16)] = (cur, site)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
per_line = collections.defaultdict(lambda: [0, collections.Counter()])
per_site = collections.Counter()
total = 0
base = None
for r in rows[hdr + 1:]:
    if len(r) <= si or not r[0].startswith("0x"):
        continue
    if base is None:
        base = int(r[0], 16)
    a = int(r[0], 16) - base
    s = float(r[si] or 0)
    total += s
    key = addr_line.get(a, ("?", "?"))
    e = per_line[key]
    e[0] += s
    for i in stall_cols:
        v = float(r[i] or 0)
        if v:
            e[1][h[i][6:]] += v
    per_site[key[1]] += s
print(f"total samples {total:.0f}")
print("== per kernel-level site (train_kernel.cuh line)")
for k, v in per_site.most_common(25):
    print(f"{v / total:6.1%}  {k}")
print("== per innermost line")
for (f, site), (s, c) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    why = ", ".join(f"{n} {x / s:.0%}" for n, x in c.most_common(3))
    print(f"{s / total:6.1%}  {f:28s} @ {site:22s} {why}")
