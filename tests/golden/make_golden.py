"""Generate golden fixtures by running the REFERENCE itself (run here only).

    python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only) with
NUMBA_CACHE_DIR redirected and bytecode writing disabled so nothing is
written into the reference tree.  The fixtures pin oracle/ (checked
bit-for-bit by tests/test_oracle_golden.py), which in turn is the checker
for the CUDA path on the GPU box where /root/reference does not exist.
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from deepmlp import deform, eval_report, kernels, network, rng, trainer  # noqa: E402
from deepmlp.mnist_io import Dataset  # noqa: E402

from paper_1003_0358_b200.synthetic import make_digits  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {
    "C1": (841, 1000, 500, 10),
    "C2": (841, 1500, 1000, 500, 10),
    "C3": (841, 2000, 1500, 1000, 500, 10),
    "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
    "C5": (841,) + (1000,) * 9 + (10,),
}


def sha1(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_rng():
    paths = [(0, 2, 0, 0), (3, 2, 5, 17), (12345, 1), (0, 3, 7), (2**63 + 5, 2, 1, 59999)]
    keys = np.array([rng.stream_key(p[0], *p[1:]) for p in paths], dtype=np.uint64)
    g = rng.substream(0, 2, 0, 0)
    words = g.bit_generator.random_raw(16)
    g = rng.substream(0, 2, 0, 0)
    u = g.uniform(5, 6)
    plen = np.array([len(p) for p in paths])
    flat = np.array([x & 0xFFFFFFFFFFFFFFFF for p in paths for x in p], dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), keys=keys, path_len=plen, path_flat=flat,
                        words=words, first_uniform=np.float64(u))


def gen_deform():
    images, labels = make_digits(96, seed=777)
    ds = Dataset(images, labels, "train")
    params = deform.DeformParams()
    out, _ = deform.deform_epoch(ds, params, seed=3, epoch=5)
    ident, _ = deform.deform_epoch(ds, deform.DeformParams.identity(), seed=3, epoch=5)
    up = deform.upscale_dataset(ds)
    # raw draws for the injected-field parity mode (first 16 images)
    k = 16
    ndx = np.zeros((k, 29, 29))
    ndy = np.zeros((k, 29, 29))
    scal = np.zeros((k, 6))  # sigma alpha mode angle sx sy
    for i in range(k):
        g = rng.substream(3, rng.STREAM_DEFORM, 5, i)
        sigma = g.uniform(*params.sigma_range)
        alpha = g.uniform(*params.alpha_range)
        ndx[i] = g.uniform(-1.0, 1.0, size=(29, 29))
        ndy[i] = g.uniform(-1.0, 1.0, size=(29, 29))
        mode = 0 if g.integers(0, 2) == 0 else 1
        beta = params.beta_reduced if int(labels[i]) in (1, 7) else params.beta_default
        angle = g.uniform(-beta, beta)
        gamma = g.uniform(*params.gamma_range)
        sx = g.uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0)
        sy = g.uniform(1.0 - gamma / 100.0, 1.0 + gamma / 100.0)
        scal[i] = (sigma, alpha, mode, angle, sx, sy)
    # larger fingerprint: 2048 images, seed 11, epoch 2
    big_i, big_l = make_digits(2048, seed=99)
    big, _ = deform.deform_epoch(Dataset(big_i, big_l, "train"), params, seed=11, epoch=2)
    np.savez_compressed(os.path.join(OUT, "deform.npz"), images=images, labels=labels,
                        deformed=out, identity=ident, upscaled=up, inj_noise_dx=ndx,
                        inj_noise_dy=ndy, inj_scalars=scal, big_sha1=sha1(big),
                        big_first=big[:4])


def gen_train():
    images, labels = make_digits(64, seed=4242)
    ds = Dataset(images, labels, "train")
    deformed, _ = deform.deform_epoch(ds, deform.DeformParams(), seed=0, epoch=0)
    x = deformed.reshape(64, -1)
    res = {}
    # small net: full weights after 40 steps
    arch = network.Architecture((841, 70, 33, 10))
    mlp = network.init_mlp(rng.substream(0, rng.STREAM_INIT), arch)
    res["small_init"] = np.concatenate([w.ravel() for w in mlp.layers])
    outs = []
    for s in range(40):
        i = s % 64
        outs.append(kernels.train_step(mlp, x[i], int(labels[i]), 1e-3))
    res["small_outputs"] = np.array(outs)
    res["small_final"] = np.concatenate([w.ravel() for w in mlp.layers])
    # C1: 25 steps, outputs + weight sha1 (bit-exact pin without committing 5 MB)
    arch = network.Architecture(CONFIGS["C1"])
    mlp = network.init_mlp(rng.substream(0, rng.STREAM_INIT), arch)
    outs = []
    for s in range(25):
        outs.append(kernels.train_step(mlp, x[s], int(labels[s]), 1e-3))
    res["c1_outputs"] = np.array(outs)
    res["c1_sha1"] = np.array([sha1(w) for w in mlp.layers])
    # train_epoch with the reference shuffle (substream(0,3,0)) on the small net
    arch = network.Architecture((841, 70, 33, 10))
    mlp = network.init_mlp(rng.substream(0, rng.STREAM_INIT), arch)
    err = trainer.train_epoch(mlp, deformed, labels, 1e-3, rng=rng.substream(0, 3, 0))
    res["epoch_err"] = np.float64(err)
    res["epoch_sha1"] = np.array([sha1(w) for w in mlp.layers])
    res["perm"] = rng.substream(0, 3, 0).permutation(64)
    res["images"] = images
    res["labels"] = labels
    res["deformed"] = deformed
    np.savez_compressed(os.path.join(OUT, "train.npz"), **res)


def gen_naive():
    """The reference's naive variant (kernels.py:58-94) on the train fixture's
    inputs: the yardstick for how far two summation orders of the same
    arithmetic drift apart (tests/test_gpu_parity_deep.py)."""
    g = np.load(os.path.join(OUT, "train.npz"))
    x, labels = g["deformed"].reshape(64, -1), g["labels"]
    arch = network.Architecture((841, 70, 33, 10))
    mlp = network.init_mlp(rng.substream(0, rng.STREAM_INIT), arch)
    outs = []
    for s in range(40):
        i = s % 64
        outs.append(kernels.train_step(mlp, x[i], int(labels[i]), 1e-3, variant="naive"))
    res = {"small_outputs": np.array(outs),
           "small_final": np.concatenate([w.ravel() for w in mlp.layers])}
    arch = network.Architecture(CONFIGS["C1"])
    mlp = network.init_mlp(rng.substream(0, rng.STREAM_INIT), arch)
    outs = []
    for s in range(25):
        outs.append(kernels.train_step(mlp, x[s], int(labels[s]), 1e-3, variant="naive"))
    res["c1_outputs"] = np.array(outs)
    res["c1_sha1"] = np.array([sha1(w) for w in mlp.layers])
    np.savez_compressed(os.path.join(OUT, "naive.npz"), **res)


def gen_eval_and_known():
    images, labels = make_digits(300, seed=31337)
    ds = Dataset(images, labels, "test")
    arch = network.Architecture((841, 70, 33, 10))
    mlp = network.init_mlp(rng.substream(5, rng.STREAM_INIT), arch)
    # make it less trivial: a few on-line steps on the deformed set
    deformed, _ = deform.deform_epoch(ds, deform.DeformParams(), seed=5, epoch=0)
    trainer.train_epoch(mlp, deformed, labels, 5e-3, rng=rng.substream(5, 3, 0))
    x = deform.upscale_dataset(ds)
    out = network.forward_batch(mlp, x)
    rep = eval_report.evaluate(mlp, ds)
    cfg = trainer.TrainConfig(arch=arch)
    np.savez_compressed(
        os.path.join(OUT, "eval.npz"), images=images, labels=labels,
        weights=np.concatenate([w.ravel() for w in mlp.layers]), outputs=out,
        error_percent=np.float64(rep.error_percent), confusion=rep.confusion,
        second_guess_correct=np.int64(rep.second_guess_correct),
        miss_index=np.array([m.index for m in rep.misclassified], dtype=np.int64),
        miss_guess2=np.array([m.guess2 for m in rep.misclassified], dtype=np.int64),
        val_error=np.float64(trainer.error_percent(mlp, x, labels)),
        count_weights=np.array([network.count_weights(network.Architecture(v))
                                for v in CONFIGS.values()], dtype=np.int64),
        scaled_tanh_1p5=np.float64(network.scaled_tanh(1.5)),
        deriv_0=np.float64(network.scaled_tanh_derivative(0.0)),
        lr=np.array([trainer.lr_schedule(e, cfg) for e in (0, 1, 10, 100, 982, 983, 2000)]),
    )


def gen_gradcheck():
    """kernels.backprop_gradients / gradient_check on a tiny float64 net."""
    arch = network.Architecture((24, 9, 7, 10))
    mlp = network.init_mlp(rng.substream(9, rng.STREAM_INIT), arch).astype(np.float64)
    mlp.layers = [w * 4.0 for w in mlp.layers]  # away from the linear regime
    x = rng.substream(9, 4).uniform(-1.0, 1.0, size=24)
    digit = 3
    grads = kernels.backprop_gradients(mlp, x, digit)
    worst = kernels.gradient_check(mlp, x, digit, step=1e-5)
    np.savez_compressed(os.path.join(OUT, "gradcheck.npz"), sizes=np.array(arch.layer_sizes),
                        weights=np.concatenate([w.ravel() for w in mlp.layers]), x=x,
                        digit=np.int64(digit), grads=np.concatenate([g.ravel() for g in grads]),
                        worst=np.float64(worst))


GENERATORS = {"rng": gen_rng, "deform": gen_deform, "train": gen_train, "naive": gen_naive,
              "eval": gen_eval_and_known, "gradcheck": gen_gradcheck}

if __name__ == "__main__":
    # python tests/golden/make_golden.py [name ...]   (default: every fixture)
    for name in (sys.argv[1:] or list(GENERATORS)):
        GENERATORS[name]()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
