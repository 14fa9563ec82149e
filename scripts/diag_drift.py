import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet
g = np.load('tests/golden/train.npz'); x = g['deformed'].reshape(64, -1); lab = g['labels']
sizes = tuple(int(v) for v in sys.argv[1].split('-'))
ref = [(w * min(1.0, 841.0 / (w.shape[1] - 1)) ** 0.5).astype(np.float32) for w in O.init_layers(4, sizes)]
w0 = [w.copy() for w in ref]
st = DeviceNet(sizes); st.set_layers([w.copy() for w in ref])
O.set_threads(8)
for s in range(48):
    y = st.train_step(x[s], int(lab[s]), 1e-3)
    yr = O.train_step(ref, x[s], int(lab[s]), 1e-3)
    if s % 6 == 5 or s < 3:
        gl = st.get_layers()
        dW = [float(np.abs(a - b).max()) for a, b in zip(gl, ref)]
        upd = [float(np.abs(b - a).max()) for a, b in zip(w0, ref)]
        col = np.abs(gl[-1] - ref[-1]).max(axis=0)
        print(s, "dy %.1e" % np.abs(y - yr).max(), "max|dW|", ["%.1e" % v for v in dW], "max|update|", ["%.1e" % v for v in upd], "worst out col", int(col.argmax()))
