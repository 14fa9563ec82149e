"""Small deformation / upscale / eval calls for compute-sanitizer memcheck:
ragged image batches (n = 13), a byte-offset (unaligned) raw pointer, other
kernel sizes, the padded-input eval path."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1003_0358_b200.deform import DeformParams, deform_device, upscale_device
from paper_1003_0358_b200.device import DeviceNet
from paper_1003_0358_b200.synthetic import make_digits

imgs, labs = make_digits(14, seed=3)
raw = torch.from_numpy(imgs).cuda()
lab = torch.from_numpy(labs).cuda()
a = deform_device(raw[:13], lab[:13], DeformParams(), 1, 2)
flat = raw.reshape(-1)
off = flat[1:1 + 13 * 784].reshape(13, 28, 28)  # 1-byte offset: the unaligned staging path
b = deform_device(off, lab[:13], DeformParams(), 1, 2)
c = deform_device(raw[:5], lab[:5], DeformParams(kernel_size=7), 1, 2)
u = upscale_device(raw[:13])
dn = DeviceNet((841, 300, 120, 10))
rng = np.random.default_rng(0)
dn.set_layers([rng.uniform(-0.05, 0.05, size=(o, i + 1)).astype(np.float32)
               for i, o in zip((841, 300, 120), (300, 120, 10))])
cnt = dn.eval_counts(u, lab[:13])
out = dn.forward_batch(u[:7].contiguous())
torch.cuda.synchronize()
print("ok", float(a.sum()), float(b.sum()), float(c.sum()), int(cnt[0]), float(out.sum()))
