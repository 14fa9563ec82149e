"""Step-by-step argmax / margin comparison GPU vs oracle (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet

g = np.load('tests/golden/train.npz')
x = g['deformed'].reshape(64, -1)
lab = g['labels']
sizes = tuple(int(v) for v in sys.argv[1].split('-'))
ref = [(w * min(1.0, 841.0 / (w.shape[1] - 1)) ** 0.5).astype(np.float32)
       for w in O.init_layers(4, sizes)]
dn = DeviceNet(sizes)
dn.set_layers([w.copy() for w in ref])
O.set_threads(8)
for s in range(48):
    i = s % 64
    y = dn.train_step(x[i], int(lab[i]), 1e-3)
    yr = O.train_step(ref, x[i], int(lab[i]), 1e-3)
    srt = np.sort(yr)
    print(s, int(np.argmax(y)), int(np.argmax(yr)), "dy %.2e" % np.abs(y - yr).max(),
          "margin %.2e" % (srt[-1] - srt[-2]), "wrong", int(np.argmax(yr)) != int(lab[i]))
