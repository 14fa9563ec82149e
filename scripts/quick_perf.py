"""Quick device timing of the persistent training kernel per config."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet
from paper_1003_0358_b200.rng import substream
CONFIGS = {
    "C1": (841, 1000, 500, 10), "C2": (841, 1500, 1000, 500, 10),
    "C3": (841, 2000, 1500, 1000, 500, 10), "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
    "C5": (841,) + (1000,) * 9 + (10,)}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
res = sys.argv[2] if len(sys.argv) > 2 else "auto"
names = sys.argv[3].split(",") if len(sys.argv) > 3 else list(CONFIGS)
LDX = int(__import__("os").environ.get("LDX", "841"))  # row stride of the inputs
x = (torch.rand((n, LDX), device="cuda") * 2 - 1)[:, :841]
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
for name in names:
    sizes = CONFIGS[name]
    rng = substream(0, 1)
    layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32) for i, o in zip(sizes[:-1], sizes[1:])]
    try:
        dn = DeviceNet(sizes, residency=res, n_ctas=int(__import__("os").environ.get("NCT", "0")))
    except Exception as e:
        print(name, "create failed", e); continue
    dn.set_layers(layers)
    prof = len(sys.argv) > 4
    wrong = torch.zeros((), dtype=torch.int64, device="cuda")
    dn.train_epoch(x[:2000], lab[:2000], None, 1e-3, wrong)
    torch.cuda.synchronize()
    if prof: dn.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dn.train_epoch(x, lab, None, 1e-3, wrong); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    pr = dn.read_profile() if prof else {}
    W = sum((i + 1) * o for i, o in zip(sizes[:-1], sizes[1:]))
    sps = n / (ms / 1e3)
    print(json.dumps({"cfg": name, "res": dn.residency, "where": "".join(w[0] for w in dn.layer_residency), "nct": dn.n_ctas, "smem": dn.smem_bytes,
                      "us_per_sample": round(ms * 1e3 / n, 3), "samples_s": round(sps),
                      "GBs_12B": round(12 * W * sps / 1e9, 1), **({"xchg_frac": round(pr["exchange_fraction"], 3), "phases_per_sample": {k: v // dn.n_ctas // n for k, v in pr.items() if k not in ("exchange_fraction", "layers") and v}, "per_layer": [[v // dn.n_ctas // n for v in lay.values()] for lay in pr["layers"]]} if prof else {})}))
    dn.close()
