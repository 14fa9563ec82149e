"""Per-SM skew of the training kernel: which SMs are the late producers?

    python scripts/sm_skew.py [C4] [launches] [samples]

Each profiled launch records, per CTA, the SM it ran on and its cycles in
the exchange waits.  A CTA that is waited on (a late producer) waits least
itself, so low exchange-wait = late.  Prints, per launch, the CTA -> SM
mapping's stability and the 12 latest CTAs with their SM / TPC, and the
correlation of per-SM lateness across launches.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet  # noqa: E402
from paper_1003_0358_b200.rng import substream  # noqa: E402

CONFIGS = {"C4": (841, 2500, 2000, 1500, 1000, 500, 10), "C3": (841, 2000, 1500, 1000, 500, 10),
           "C2": (841, 1500, 1000, 500, 10)}
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
sizes = CONFIGS[name]
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
rng = substream(0, 1)
layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
          for i, o in zip(sizes[:-1], sizes[1:])]
dn = DeviceNet(sizes)
dn.set_layers(layers)
wrong = torch.zeros((), dtype=torch.int64, device="cuda")
dn.train_epoch(x[:2000], lab[:2000], None, 1e-3, wrong)
dn.profile(True)
dn.read_profile_cta()
sms, waits = [], []
for k in range(launches):
    dn.train_epoch(x, lab, None, 1e-3, wrong)
    sm, slots = dn.read_profile_cta()
    wait = slots[:, 1] / n  # exchange-wait cycles per sample
    sms.append(sm)
    waits.append(wait)
    last_slots = slots
    order = np.argsort(wait)
    print(json.dumps({"launch": k, "same_mapping_as_first": bool((sm == sms[0]).all()),
                      "wait_median": float(np.median(wait)),
                      "latest": [[int(c), int(sm[c]), int(sm[c]) // 2, round(float(wait[c]))]
                                 for c in order[:12]]}))
# per-SM lateness (median wait - wait), correlated across launches
per_sm = []
for sm, wait in zip(sms, waits):
    v = np.zeros(int(sm.max()) + 1)
    v[sm] = np.median(wait) - wait
    per_sm.append(v)
per_sm = np.array(per_sm)
cc = np.corrcoef(per_sm)
print("per-SM lateness correlation across launches:", np.round(cc[0], 2).tolist())
mean = per_sm.mean(0)
top = np.argsort(-mean)[:16]
print("latest SMs on average (sm, tpc, cycles behind the median wait):",
      [[int(s), int(s) // 2, round(float(mean[s]))] for s in top])
per_cta = np.array(waits)
print("per-CTA lateness correlation across launches:",
      np.round(np.corrcoef(np.median(per_cta, 1)[:, None] - per_cta)[0], 2).tolist())
dn.close()
# which phases make the latest CTAs late: per-phase / per-layer cycles per sample of the
# 6 latest CTAs minus the median over CTAs (last launch)
per = last_slots / n
med = np.median(per[:125], 0)
late6 = np.argsort(waits[-1])[:6]
names = DeviceNet.PROFILE_SLOTS
kinds = DeviceNet.LAYER_KINDS
for c in late6:
    d = per[c] - med
    ph = {names[i]: round(float(d[i])) for i in range(16) if names[i] != "smid" and abs(d[i]) > 40}
    lay = {f"L{l}.{kinds[k]}": round(float(d[16 + 5 * l + k]))
           for l in range(len(sizes) - 1) for k in range(5) if abs(d[16 + 5 * l + k]) > 40}
    print(json.dumps({"cta": int(c), "sm": int(sms[-1][c]), "phases": ph, "layers": lay}))
