"""Per-step GPU vs oracle diagnostics for a layer-size tuple (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet

g = np.load('tests/golden/train.npz')
x = g['deformed'].reshape(64, -1)
lab = g['labels']
for spec in sys.argv[1:]:
    sizes = tuple(int(v) for v in spec.split('-'))
    ref = O.init_layers(4, sizes)
    dn = DeviceNet(sizes)
    dn.set_layers([w.copy() for w in ref])
    O.set_threads(8)
    worst = 0.0
    for s in range(6):
        y = dn.train_step(x[s], int(lab[s]), 1e-3)
        yr = O.train_step(ref, x[s], int(lab[s]), 1e-3)
        worst = max(worst, float(np.abs(y - yr).max()))
    gl = dn.get_layers()
    rel = [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(gl, ref)]
    print(spec, "res", dn.layer_residency, "max|dy|", worst, "rel dW per layer", rel)
    dn.close()
