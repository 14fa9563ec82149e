import sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet
g = np.load('tests/golden/train.npz'); x = g['deformed'].reshape(64, -1); lab = g['labels']
sizes = (841, 5000, 10)
ref = [(w * min(1.0, 841.0 / (w.shape[1] - 1)) ** 0.5).astype(np.float32) for w in O.init_layers(4, sizes)]
order = np.arange(48) % 64
dn = DeviceNet(sizes); dn.set_layers([w.copy() for w in ref])
st = DeviceNet(sizes); st.set_layers([w.copy() for w in ref])
ref2 = [w.copy() for w in ref]
O.set_threads(8)
wrong_ref = O.train_epoch(ref, g["deformed"], lab, 1e-3, order=order)
wrong = torch.zeros((), dtype=torch.int64, device="cuda")
dn.train_epoch(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda(), torch.from_numpy(order.astype(np.int32)).cuda(), 1e-3, wrong)
torch.cuda.synchronize()
ws = 0; wr2 = 0
for s in order:
    y = st.train_step(x[s], int(lab[s]), 1e-3); ws += int(np.argmax(y) != lab[s])
    yr = O.train_step(ref2, x[s], int(lab[s]), 1e-3); wr2 += int(np.argmax(yr) != lab[s])
print("gpu epoch", int(wrong.item()), "oracle epoch", wrong_ref, "gpu steps", ws, "oracle steps", wr2)
print("epoch vs steps W diff", [float(np.abs(a - b).max()) for a, b in zip(dn.get_layers(), st.get_layers())])
print("oracle epoch vs steps W diff", [float(np.abs(a - b).max()) for a, b in zip(ref, ref2)])
