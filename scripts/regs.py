"""ptxas spill summary per k_train instance: python scripts/regs.py train_inst_f3 [...]"""
import os, re, subprocess, sys

CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1003_0358_b200", "csrc")
for unit in sys.argv[1:]:
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                        "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas",
                        "-v", *os.environ.get("DMLP_NVCC_FLAGS", "").split(), "-c", f"{unit}.cu", "-o", f"/tmp/{unit}.o"],
                       cwd=CSRC, capture_output=True, text=True)
    name = None
    for line in r.stderr.splitlines():
        m = re.search(r"Compiling entry function '([^']+)'", line) or re.search(r"Function properties for (\S+)", line)
        if m:
            name = m.group(1)
        m2 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m2 and name and "k_train" in name:
            p = re.search(r"k_trainILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb([01])", name)
            print(f"{unit} <{','.join(p.groups()[:4])}> F{p.group(5)} P{p.group(6)}: "
                  f"spill st={m2.group(1)} ld={m2.group(2)}")
