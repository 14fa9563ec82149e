import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet
from oracle import oracle as O
g = np.load('tests/golden/train.npz')
x, lab = g['deformed'].reshape(64, -1), g['labels']
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for sizes in [(841, 300, 120, 10), (841, 70, 33, 10)]:
  for res in ["smem", "l2"]:
    for nct in [0, 8, 100]:
        base = O.init_layers(7, sizes)
        outs = []
        for _ in range(3):
            dn = DeviceNet(sizes, residency=res, n_ctas=nct); dn.set_layers([w.copy() for w in base])
            wrong = torch.zeros((), dtype=torch.int64, device="cuda")
            xd = torch.from_numpy(np.tile(x, (n // 64, 1))).cuda(); ld = torch.from_numpy(np.tile(lab, n // 64)).cuda()
            dn.train_epoch(xd, ld, None, 1e-3, wrong); torch.cuda.synchronize()
            outs.append(np.concatenate([w.ravel() for w in dn.get_layers()]))
        print(sizes, res, nct, "same12", np.array_equal(outs[0], outs[1]), "same13", np.array_equal(outs[0], outs[2]), "maxdiff", float(np.abs(outs[0]-outs[1]).max()))
