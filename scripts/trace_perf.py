"""Timeline of one sample: per exchange, producer skew and gather latency (ns)."""
import sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet
from paper_1003_0358_b200.rng import substream
CONFIGS = {"C1": (841, 1000, 500, 10), "C2": (841, 1500, 1000, 500, 10),
           "C3": (841, 2000, 1500, 1000, 500, 10), "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
           "C5": (841,) + (1000,) * 9 + (10,)}
names = sys.argv[1].split(",")
res = sys.argv[2] if len(sys.argv) > 2 else "auto"
n = 600
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
for name in names:
    sizes = CONFIGS[name]; L = len(sizes) - 1
    rng = substream(0, 1)
    layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32) for i, o in zip(sizes[:-1], sizes[1:])]
    dn = DeviceNet(sizes, residency=res); dn.set_layers(layers)
    wrong = torch.zeros((), dtype=torch.int64, device="cuda")
    dn.train_epoch(x, lab, None, 1e-3, wrong)
    dn.trace(500)
    dn.train_epoch(x, lab, None, 1e-3, wrong)
    m = dn.trace(-1).astype(np.int64)
    t0 = m[:, 0].min()
    ne = 2 * L - 3
    out = {"cfg": name, "res": dn.residency, "sample_ns": int(m[:, 63].max() - t0)}
    rows = []
    prev_done = m[:, 0]
    for e in range(ne):
        pub = m[:, 1 + 2 * e]; got = m[:, 2 + 2 * e]
        valid = pub > 0
        rows.append({"e": e, "compute_ns(max-prev)": int((pub - prev_done).max()),
                     "compute_ns(median)": int(np.median(pub - prev_done)),
                     "pub_skew_ns": int(pub[valid].max() - pub[valid].min()),
                     "latency_after_last_pub_ns": int(got.max() - pub.max()),
                     "gather_done_spread_ns": int(got.max() - got.min())})
        prev_done = got
    out["tail_ns"] = int((m[:, 63] - prev_done).max())
    print(json.dumps(out))
    for r in rows: print("   ", json.dumps(r))
    dn.close()
