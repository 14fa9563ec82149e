import sys, time, numpy as np, torch
sys.path.insert(0, '.')
n = 40000
x = torch.rand((n, 841)).pin_memory()
lab = torch.randint(0, 10, (n,), dtype=torch.uint8).pin_memory()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); xd = x.to('cuda'); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"H2D {x.numel()*4/1e6:.0f} MB pinned: {1e3*(t1-t0):.2f} ms = {x.numel()*4/(t1-t0)/1e9:.1f} GB/s")
t0 = time.perf_counter(); o = np.random.default_rng(0).permutation(n); od = torch.from_numpy(o.astype(np.int32)).to('cuda'); torch.cuda.synchronize(); print(f"perm+H2D {1e3*(time.perf_counter()-t0):.2f} ms")
from paper_1003_0358_b200 import trainer
from paper_1003_0358_b200.network import Architecture, init_mlp
from paper_1003_0358_b200.rng import substream
mlp = init_mlp(substream(0, 1), Architecture((841, 2500, 2000, 1500, 1000, 500, 10)))
dn = mlp.device_net(0)
w = torch.zeros((), dtype=torch.int64, device='cuda')
for k in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dn.train_epoch(xd, lab.to('cuda'), od, 1e-3, w); torch.cuda.synchronize(); t1 = time.perf_counter()
    trainer.train_epoch(mlp, x, lab, 1e-3, rng=substream(0, 3, k)); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"device-resident epoch {1e3*(t1-t0):.1f} ms; trainer.train_epoch from pinned host {1e3*(t2-t1):.1f} ms")
