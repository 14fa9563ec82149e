"""Which CTAs are the slowest producers of each exchange (one-sample traces)?

    python scripts/trace_slowest.py C4

For each exchange and traced sample, the 3 latest publishers (CTA id, ns
behind the median) and how often each CTA is among the 5 latest overall.
"""
import collections
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet  # noqa: E402
from paper_1003_0358_b200.rng import substream  # noqa: E402

CONFIGS = {"C4": (841, 2500, 2000, 1500, 1000, 500, 10), "C3": (841, 2000, 1500, 1000, 500, 10)}
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
sizes = CONFIGS[name]
L = len(sizes) - 1
H = L - 1
n = 600
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
rng = substream(0, 1)
layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
          for i, o in zip(sizes[:-1], sizes[1:])]
dn = DeviceNet(sizes)
dn.set_layers(layers)
nct = dn.n_ctas
R = [-(-sizes[l + 1] // nct) for l in range(H)]
P = [-(-sizes[l + 1] // R[l]) for l in range(H)]
wrong = torch.zeros((), dtype=torch.int64, device="cuda")
dn.train_epoch(x, lab, None, 1e-3, wrong)
marks = []
for smp in range(100, 500, 40):
    dn.trace(smp)
    dn.train_epoch(x, lab, None, 1e-3, wrong)
    marks.append(dn.trace(-1).astype(np.int64))
names = [f"fwd y{l}" for l in range(H - 1)] + ["out"] + [f"bwd p{l}" for l in range(H - 1, 0, -1)]
prods = [P[l] for l in range(H - 1)] + [P[H - 1]] + [P[l] for l in range(H - 1, 0, -1)]
late = collections.Counter()
for e, (nm, npro) in enumerate(zip(names, prods)):
    tops = []
    for m in marks:
        pub = m[:npro, 1 + 2 * e]
        med = np.median(pub)
        order = np.argsort(-pub)
        tops.append([(int(c), int(pub[c] - med)) for c in order[:3]])
        for c in order[:5]:
            late[int(c)] += 1
    print(nm, tops[:4])
print("most often among the 5 latest:", late.most_common(12))
dn.close()
