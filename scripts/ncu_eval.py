"""Run the evaluation forward once on C4 (for an ncu capture of k_gemm_tanh)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet

sizes = (841, 2500, 2000, 1500, 1000, 500, 10)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
dn = DeviceNet(sizes)
rng = np.random.default_rng(0)
dn.set_layers([rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
               for i, o in zip(sizes[:-1], sizes[1:])])
for _ in range(2):
    dn.eval_counts(x, lab)
torch.cuda.synchronize()
print("done")
