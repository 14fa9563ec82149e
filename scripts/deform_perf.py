"""Device time of one 60k-image deformation epoch (k_deform)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.deform import DeformParams, deform_device
from paper_1003_0358_b200.synthetic import make_digits

imgs, labs = make_digits(2000, seed=3)
n = 60000
raw = torch.from_numpy(np.resize(imgs, (n, 28, 28))).cuda()
lab = torch.from_numpy(np.resize(labs, n)).cuda()
out = torch.empty((n, 841), dtype=torch.float32, device='cuda')
for e in range(3):
    deform_device(raw, lab, DeformParams(), 0, e, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for e in range(10):
    deform_device(raw, lab, DeformParams(), 0, 3 + e, out=out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"deform: {ms:.3f} ms per 60k epoch, {n / ms * 1e3 / 1e6:.2f} M imgs/s")
