"""GPU end-to-end: the drop-in API (trainer.train / train_step / evaluate /
deform_epoch) against an oracle replay of the reference protocol
(trainer.py:130-207) on identical inputs."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle_train(deformed_epochs, images, labels, sizes, seed=0):
    """trainer.train restated with the oracle (trainer.py:130-207): shuffled
    on-line pass over each epoch's deformed set -> validation on the
    un-deformed train set (counts); weights snapshotted after every epoch."""
    layers = O.init_layers(seed, sizes)
    x_val = O.upscale_dataset(images)
    hist, snaps = [], []
    for e, deformed in enumerate(deformed_epochs):
        eta = max(1e-6, 1e-3 * 0.993 ** e)
        perm = O.substream(seed, 3, e).permutation(len(labels))
        wrong = O.train_epoch(layers, deformed, labels, eta, order=perm)
        vwrong = O.eval_counts(O.forward_batch(layers, x_val), labels)[0]
        hist.append((wrong, vwrong))
        snaps.append([w.copy() for w in layers])
    return hist, snaps


def test_train_two_epochs_matches_oracle(tmp_path):
    """trainer.train (C1, 3,000 images, 2 epochs) vs the oracle replay of the
    reference protocol on the same deformed inputs: train and validation
    error counts exact, the best epoch's weights within 1e-5 relative per
    layer.  The deformed inputs are the device kernel's (a pure function of
    seed, epoch and image; checked against the oracle's deformation within
    1e-5 here, and bit-pinned in test_gpu_deform_eval)."""
    import torch

    from paper_1003_0358_b200.deform import DeformParams, deform_device
    from paper_1003_0358_b200.mnist_io import Dataset
    from paper_1003_0358_b200.network import Architecture, load_checkpoint
    from paper_1003_0358_b200.synthetic import make_digits
    from paper_1003_0358_b200.trainer import TrainConfig, train

    imgs, labs = make_digits(3000, seed=21)
    sizes = (841, 1000, 500, 10)
    O.set_threads(16)
    raw, lab = torch.from_numpy(imgs).cuda(), torch.from_numpy(labs).cuda()
    epochs = []
    for e in range(2):
        d = deform_device(raw, lab, DeformParams(), 0, e).cpu().numpy()
        od = O.deform_epoch(imgs[:256], labs[:256], O.DeformParams(), seed=0, epoch=e)
        assert np.abs(d[:256].reshape(-1, 29, 29) - od).max() <= 1e-5
        epochs.append(d)
    ref_hist, snaps = _oracle_train(epochs, imgs, labs, sizes)
    res = train(TrainConfig(arch=Architecture(sizes), max_epochs=2), Dataset(imgs, labs, "train"),
                out_dir=tmp_path)
    n = len(labs)
    for (w, vw), st in zip(ref_hist, res.history):
        assert st.train_error == 100.0 * w / n, (st.epoch, st.train_error, 100.0 * w / n)
        assert st.val_error == 100.0 * vw / n, (st.epoch, st.val_error, 100.0 * vw / n)
    assert res.best_epoch in (0, 1)
    ck = load_checkpoint((tmp_path / "best.dmlp").read_bytes())
    assert ck.epoch == res.best_epoch
    for li, (g, b, r) in enumerate(zip(ck.mlp.layers, res.best_mlp.layers,
                                       snaps[res.best_epoch])):
        assert np.array_equal(g, b)
        rel = np.abs(g.astype(np.float64) - r).max() / np.abs(r).max()
        assert rel <= 1e-5, f"layer {li}: max|dW|/max|W| = {rel:.2e}"
    assert (tmp_path / "run_history.jsonl").read_text().count("\n") == 2


def test_train_step_api_syncs_weights(golden):
    from paper_1003_0358_b200 import kernels
    from paper_1003_0358_b200.network import Architecture, init_mlp
    from paper_1003_0358_b200.rng import substream

    g = golden("train")
    x = g["deformed"].reshape(64, -1)
    sizes = (841, 70, 33, 10)
    mlp = init_mlp(substream(0, 1), Architecture(sizes))
    held = mlp.layers[0]  # the reference mutates layers in place: identity must survive
    for s in range(40):
        kernels.train_step(mlp, x[s % 64], int(g["labels"][s % 64]), 1e-3, variant="tiled")
    flat = np.concatenate([w.ravel() for w in mlp.layers])
    assert mlp.layers[0] is held
    d = np.abs(flat - g["small_final"])
    assert d.max() <= 1e-5 * np.abs(g["small_final"]).max()


def test_deform_epoch_and_upscale_api(golden):
    from paper_1003_0358_b200.deform import DeformParams, deform_epoch, upscale_dataset
    from paper_1003_0358_b200.mnist_io import Dataset

    g = golden("deform")
    ds = Dataset(g["images"], g["labels"], "train")
    out, lab = deform_epoch(ds, DeformParams(), seed=3, epoch=5, lanes=4)
    assert out.shape == (96, 29, 29) and out.dtype == np.float32
    assert np.abs(out - g["deformed"]).max() <= 1e-5
    assert np.array_equal(upscale_dataset(ds), g["upscaled"])


def test_evaluate_api(golden):
    from paper_1003_0358_b200.eval_report import evaluate, format_summary
    from paper_1003_0358_b200.mnist_io import Dataset
    from paper_1003_0358_b200.network import Architecture, Mlp

    g = golden("eval")
    sizes = (841, 70, 33, 10)
    layers, pos = [], 0
    for s in O.layer_shapes(sizes):
        layers.append(g["weights"][pos:pos + s[0] * s[1]].reshape(s).astype(np.float32).copy())
        pos += s[0] * s[1]
    rep = evaluate(Mlp(Architecture(sizes), layers), Dataset(g["images"], g["labels"], "test"))
    assert rep.error_percent == float(g["error_percent"])
    assert np.array_equal(rep.confusion, g["confusion"])
    assert rep.second_guess_correct == int(g["second_guess_correct"])
    assert [m.index for m in rep.misclassified] == list(g["miss_index"])
    assert [m.guess2 for m in rep.misclassified] == list(g["miss_guess2"])
    assert "test error" in format_summary(rep)


def test_distributed_helpers_single_rank():
    import torch

    from paper_1003_0358_b200.deform import DeformParams
    from paper_1003_0358_b200.device import DeviceNet
    from paper_1003_0358_b200.distributed import (deform_sharded, eval_counts_sharded,
                                                  gather_deformed)
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(300, seed=2)
    raw, lab = torch.from_numpy(imgs).cuda(), torch.from_numpy(labs).cuda()
    shard, lo, hi = deform_sharded(raw, lab, DeformParams(), 1, 0)
    full = gather_deformed(shard, 300)
    ref = O.deform_epoch(imgs, labs, O.DeformParams(), seed=1, epoch=0).reshape(300, -1)
    assert (lo, hi) == (0, 300) and np.abs(full.cpu().numpy() - ref).max() <= 1e-5
    dn = DeviceNet((841, 50, 10))
    layers = O.init_layers(9, (841, 50, 10))
    dn.set_layers(layers)
    counts = eval_counts_sharded(dn, full, lab).cpu().numpy()
    w, conf, sec, _ = O.eval_counts(O.forward_batch(layers, ref), labs)
    assert counts[0] == w and counts[101] == sec


def test_train_resume_replays_the_uninterrupted_run(tmp_path):
    """SPEC.md:517 resume path: 1 epoch + checkpoint + resume for epoch 2 gives
    the same weights and history as 2 uninterrupted epochs."""
    from paper_1003_0358_b200.mnist_io import Dataset
    from paper_1003_0358_b200.network import Architecture, save_checkpoint
    from paper_1003_0358_b200.trainer import TrainConfig, train
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(400, seed=5)
    sizes = (841, 90, 40, 10)
    ds = Dataset(imgs, labs, "train")
    full = train(TrainConfig(arch=Architecture(sizes), max_epochs=2), ds)
    first = train(TrainConfig(arch=Architecture(sizes), max_epochs=1), ds)
    # the state after epoch 0 (the last, not necessarily the best, weights)
    ck = save_checkpoint(first.best_mlp if first.best_epoch == 0 else None, 0,
                         first.history[0].val_error)
    rest = train(TrainConfig(arch=Architecture(sizes), max_epochs=2), ds, resume=ck)
    assert [h.epoch for h in rest.history] == [1]
    assert rest.history[0].train_error == full.history[1].train_error
    assert rest.history[0].val_error == full.history[1].val_error
    if full.best_epoch == 1 and rest.best_epoch == 1:
        for a, b in zip(full.best_mlp.layers, rest.best_mlp.layers):
            assert np.array_equal(a, b)


def test_resume_from_interrupt_checkpoint(tmp_path, monkeypatch):
    """KeyboardInterrupt -> interrupt.dmlp stores the epoch that was running
    (trainer.py:203-205); resuming from it continues at that epoch and
    replays the uninterrupted run."""
    from paper_1003_0358_b200 import trainer as T
    from paper_1003_0358_b200.mnist_io import Dataset
    from paper_1003_0358_b200.network import Architecture, load_checkpoint
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(400, seed=6)
    sizes = (841, 90, 40, 10)
    ds = Dataset(imgs, labs, "train")
    cfg = T.TrainConfig(arch=Architecture(sizes), max_epochs=3)
    full = T.train(cfg, ds)
    real = T.lr_schedule

    def stop_at_epoch_1(epoch, c):
        if epoch == 1:
            raise KeyboardInterrupt
        return real(epoch, c)

    monkeypatch.setattr(T, "lr_schedule", stop_at_epoch_1)
    with pytest.raises(T.InterruptCheckpoint) as ei:
        T.train(cfg, ds, out_dir=tmp_path)
    monkeypatch.setattr(T, "lr_schedule", real)
    ck = load_checkpoint(ei.value.path.read_bytes())
    assert ck.epoch == 1 and np.isnan(ck.validation_error)
    rest = T.train(cfg, ds, resume=ei.value.path)
    assert [h.epoch for h in rest.history] == [1, 2]
    for a, b in zip(rest.history, full.history[1:]):
        assert (a.train_error, a.val_error) == (b.train_error, b.val_error)


def test_load_dataset_device_matches_host(tmp_path):
    """IDX ingestion straight into HBM (mnist_io.load_dataset_device) holds the
    same bytes as the host parser, and raises the same errors."""
    import gzip

    from paper_1003_0358_b200 import mnist_io
    from paper_1003_0358_b200.synthetic import make_digits, write_idx_images, write_idx_labels

    imgs, labs = make_digits(300, seed=4)
    (tmp_path / "i.gz").write_bytes(gzip.compress(write_idx_images(imgs)))
    (tmp_path / "l").write_bytes(write_idx_labels(labs))
    di, dl = mnist_io.load_dataset_device(tmp_path / "i.gz", tmp_path / "l")
    assert di.is_cuda and np.array_equal(di.cpu().numpy(), imgs)
    assert np.array_equal(dl.cpu().numpy(), labs)
    bad = labs.copy()
    bad[7] = 11
    (tmp_path / "b").write_bytes(write_idx_labels(bad))
    with pytest.raises(mnist_io.LabelOutOfRange):
        mnist_io.load_dataset_device(tmp_path / "i.gz", tmp_path / "b")
    (tmp_path / "s").write_bytes(write_idx_labels(labs[:10]))
    with pytest.raises(mnist_io.CountMismatch):
        mnist_io.load_dataset_device(tmp_path / "i.gz", tmp_path / "s")


def test_bench_line_smoke():
    """bench.py end to end at a small size: one JSON line with the contract's
    keys, the L2 roofline and the hybrid fraction, the deformation and eval
    extras."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--config", "C1", "--samples", "3000",
                          "--steps", "2", "--warmup", "3", "--cpu-seconds", "0",
                          "--deform-images", "4096"], cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "e2e", "gpu_launches", "roofline",
              "clocks", "deform", "eval"):
        assert k in line, k
    assert line["roofline"]["bound"] == "l2" and 0 < line["roofline"]["frac"] < 1
    assert 0 < line["roofline"]["hybrid"]["frac_hybrid"] < 1
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["deform"]["imgs_per_s"] > 0
