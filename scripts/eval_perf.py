"""Device time of the evaluation forward (k_gemm_tanh + k_out_rank) per config."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.device import DeviceNet

CONFIGS = {"C1": (841, 1000, 500, 10), "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
           "C5": (841,) + (1000,) * 9 + (10,)}
n = 60000
x = torch.rand((n, 841), device="cuda") * 2 - 1
lab = torch.randint(0, 10, (n,), device="cuda", dtype=torch.uint8)
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else CONFIGS):
    sizes = CONFIGS[name]
    dn = DeviceNet(sizes)
    rng = np.random.default_rng(0)
    dn.set_layers([rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
                   for i, o in zip(sizes[:-1], sizes[1:])])
    for _ in range(2):
        dn.eval_counts(x, lab)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        dn.eval_counts(x, lab)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    fl = 2 * sum(i * o for i, o in zip(sizes[:-1], sizes[1:])) * n
    print(f"{name}: {ms:.3f} ms per {n}, {n / ms * 1e3 / 1e6:.3f} M imgs/s, {fl / ms / 1e9:.1f} TFLOP/s")
    dn.close()
