"""Run the training kernel once on a config (for ncu capture)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet
from paper_1003_0358_b200.rng import substream
CONFIGS = {"C1": (841, 1000, 500, 10), "C2": (841, 1500, 1000, 500, 10),
           "C3": (841, 2000, 1500, 1000, 500, 10), "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
           "C5": (841,) + (1000,) * 9 + (10,)}
name, n, res = sys.argv[1], int(sys.argv[2]), sys.argv[3]
sizes = CONFIGS[name]
rng = substream(0, 1)
layers = [rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32) for i, o in zip(sizes[:-1], sizes[1:])]
dn = DeviceNet(sizes, residency=res)
dn.set_layers(layers)
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
wrong = torch.zeros((), dtype=torch.int64, device="cuda")
for _ in range(2):
    dn.train_epoch(x, lab, None, 1e-3, wrong)
torch.cuda.synchronize()
print("done", name, res)
