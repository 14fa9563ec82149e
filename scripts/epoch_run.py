"""Whole-epoch run of the drop-in trainer on one GPU.

    python scripts/epoch_run.py [epochs] [n_train]

trainer.train on the headline net (C4) with the synthetic digit set: every
epoch deforms all images on the device (a side stream, overlapped with the
previous epoch's training), trains on-line over the shuffled epoch in one
persistent launch, then validates on the undeformed training set.  Prints one
JSON line per epoch (seconds, on-line samples/s of the whole epoch, the
deformation's share, errors) and a summary line.
"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1003_0358_b200.mnist_io import Dataset  # noqa: E402
from paper_1003_0358_b200.network import Architecture  # noqa: E402
from paper_1003_0358_b200.synthetic import make_digits  # noqa: E402
from paper_1003_0358_b200.trainer import TrainConfig, train  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
t0 = time.time()
imgs, labs = make_digits(n, seed=12345)
t_data = time.time() - t0
ds = Dataset(imgs, labs, "train")
cfg = TrainConfig(arch=Architecture((841, 2500, 2000, 1500, 1000, 500, 10)), max_epochs=epochs,
                  seed=0)
t1 = time.time()
res = train(cfg, ds)
wall = time.time() - t1
for h in res.history:
    print(json.dumps({"epoch": h.epoch, "eta": h.eta, "seconds": round(h.seconds, 4),
                      "samples_per_s": round(n / h.seconds, 1),
                      "deform_share": round(h.deform_share, 4),
                      "train_error_pct": round(h.train_error, 3),
                      "val_error_pct": round(h.val_error, 3)}))
print(json.dumps({"net": "C4 841-2500-2000-1500-1000-500-10", "images": n, "epochs": epochs,
                  "train_wall_s": round(wall, 2), "synthetic_data_s": round(t_data, 1),
                  "best_epoch": res.best_epoch, "best_val_error_pct": round(res.best_val_error, 3)}))
