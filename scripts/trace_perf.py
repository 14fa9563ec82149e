"""Timeline of one sample: per exchange, producer skew and gather latency (ns).

    python scripts/trace_perf.py C4[,C5] [residency]

Every CTA records %globaltimer at CTA-synchronised marks of one sample
(dmlp_net_trace): mark 0 = sample start, for exchange e: 1+2e = its
contribution published, 2+2e = its gather done; 63 = sample end.  Only the
CTAs that take part in an exchange (producers / consumers) are counted.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet  # noqa: E402
from paper_1003_0358_b200.rng import substream  # noqa: E402

CONFIGS = {"C1": (841, 1000, 500, 10), "C2": (841, 1500, 1000, 500, 10),
           "C3": (841, 2000, 1500, 1000, 500, 10), "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
           "C5": (841,) + (1000,) * 9 + (10,)}
names = sys.argv[1].split(",")
res = sys.argv[2] if len(sys.argv) > 2 else "auto"
n = 600
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
for name in names:
    sizes = CONFIGS[name]
    L = len(sizes) - 1
    H = L - 1
    rng = substream(0, 1)
    layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
              for i, o in zip(sizes[:-1], sizes[1:])]
    dn = DeviceNet(sizes, residency=res)
    dn.set_layers(layers)
    nct = dn.n_ctas
    R = [-(-sizes[l + 1] // nct) for l in range(H)]
    P = [-(-sizes[l + 1] // R[l]) for l in range(H)]
    wrong = torch.zeros((), dtype=torch.int64, device="cuda")
    dn.train_epoch(x, lab, None, 1e-3, wrong)
    samples = []
    for smp in (300, 400, 500):
        dn.trace(smp)
        dn.train_epoch(x, lab, None, 1e-3, wrong)
        samples.append(dn.trace(-1).astype(np.int64))
    # exchanges: forward y of layers 0..H-2 (producers P[l], consumers P[l+1]),
    # output partials (producers P[H-1], consumers P[H-1] and CTA 0),
    # backward partials of layers H-1..1 (producers P[l], consumers P[l-1])
    ex = []
    for l in range(H - 1):
        ex.append((f"fwd y{l}", P[l], P[l + 1]))
    ex.append(("out partials", P[H - 1], P[H - 1]))
    for l in range(H - 1, 0, -1):
        ex.append((f"bwd p{l}", P[l], P[l - 1]))
    rows = []
    for e, (nm, npro, ncon) in enumerate(ex):
        comp, skew, lat, wait = [], [], [], []
        for m in samples:
            prev = m[:, 0] if e == 0 else m[:, 2 * e]
            pub, got = m[:npro, 1 + 2 * e], m[:ncon, 2 + 2 * e]
            comp.append(np.median(pub - prev[:npro]))
            skew.append(pub.max() - np.median(pub))
            lat.append(got.max() - pub.max())
            wait.append(np.median(got - m[:ncon, 1 + 2 * e]))
        rows.append({"e": e, "what": nm, "producers": npro, "compute_med_ns": int(np.mean(comp)),
                     "slowest_producer_behind_median_ns": int(np.mean(skew)),
                     "last_publish_to_all_gathered_ns": int(np.mean(lat)),
                     "consumer_wait_med_ns": int(np.mean(wait))})
    tot = int(np.mean([m[:, 63].max() - m[:, 0].min() for m in samples]))
    print(json.dumps({"cfg": name, "where": "".join(w[0] for w in dn.layer_residency),
                      "sample_ns": tot}))
    for r in rows:
        print("   ", json.dumps(r))
    dn.close()
