"""Instructions executed per source line of one ncu capture (SASS source page
joined with the cubin's line table, like ncu_lines.py for stalls).

    python scripts/ncu_inst_lines.py capture.ncu-rep object.o kernel_substring [top]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.splitlines()
addr_line, inside, cur, chain = {}, False, "?", []
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
            cur = chain[0] + (" @ " + chain[-1] if len(chain) > 1 else "")
            chain = []
        addr_line[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ia, ii, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
per_line, per_op, tot = collections.Counter(), collections.Counter(), 0
base = int(rows[2][ia], 16)  # the page lists absolute addresses; the cubin's start at 0
for r in rows[2:]:
    if len(r) <= ii or not r[ii].strip():
        continue
    n = float(r[ii].replace(",", ""))
    a = int(r[ia], 16) - base
    per_line[addr_line.get(a, "?")] += n
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    per_op[op.split(".")[0]] += n
    tot += n
print(f"warp instructions executed: {tot:.0f}")
print("== per source line")
for k, v in per_line.most_common(top):
    print(f"{100 * v / tot:5.1f}%  {k}")
print("== per opcode")
for k, v in per_op.most_common(20):
    print(f"{100 * v / tot:5.1f}%  {k}")
