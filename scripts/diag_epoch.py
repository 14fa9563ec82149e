"""GPU train_epoch(n) vs n GPU train_step calls: first divergence (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet

g = np.load('tests/golden/train.npz')
x = g['deformed'].reshape(64, -1)
lab = g['labels']
sizes = tuple(int(v) for v in sys.argv[1].split('-'))
nct = int(sys.argv[2]) if len(sys.argv) > 2 else 0
base = [(w * min(1.0, 841.0 / (w.shape[1] - 1)) ** 0.5).astype(np.float32)
        for w in O.init_layers(4, sizes)]
for n in (1, 2, 3, 5, 8):
    a = DeviceNet(sizes, n_ctas=nct); a.set_layers([w.copy() for w in base])
    b = DeviceNet(sizes, n_ctas=nct); b.set_layers([w.copy() for w in base])
    wrong = torch.zeros((), dtype=torch.int64, device="cuda")
    a.train_epoch(torch.from_numpy(x[:n]).cuda(), torch.from_numpy(lab[:n]).cuda(), None, 1e-3, wrong)
    for s in range(n):
        b.train_step(x[s], int(lab[s]), 1e-3)
    la, lb = a.get_layers(), b.get_layers()
    d = [float(np.abs(p - q).max()) for p, q in zip(la, lb)]
    print("n", n, "max|epoch - steps| per layer", d)
    a.close(); b.close()
