"""GPU end-to-end: the drop-in API (trainer.train / train_step / evaluate /
deform_epoch) against an oracle replay of the reference protocol
(trainer.py:130-207) on identical inputs."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle_train(images, labels, sizes, epochs, seed=0):
    """trainer.train restated with the oracle: deform -> shuffled on-line pass
    -> validation on the un-deformed train set (counts)."""
    layers = O.init_layers(seed, sizes)
    x_val = O.upscale_dataset(images)
    hist = []
    for e in range(epochs):
        deformed = O.deform_epoch(images, labels, O.DeformParams(), seed=seed, epoch=e)
        eta = max(1e-6, 1e-3 * 0.993 ** e)
        perm = O.substream(seed, 3, e).permutation(len(labels))
        wrong = O.train_epoch(layers, deformed, labels, eta, order=perm)
        vwrong = O.eval_counts(O.forward_batch(layers, x_val), labels)[0]
        hist.append((wrong, vwrong))
    return layers, hist


def test_train_two_epochs_matches_oracle(tmp_path):
    from paper_1003_0358_b200.mnist_io import Dataset
    from paper_1003_0358_b200.network import Architecture, load_checkpoint
    from paper_1003_0358_b200.synthetic import make_digits
    from paper_1003_0358_b200.trainer import TrainConfig, train

    imgs, labs = make_digits(600, seed=21)
    sizes = (841, 120, 60, 10)
    O.set_threads(8)
    ref_layers, ref_hist = _oracle_train(imgs, labs, sizes, 2)
    res = train(TrainConfig(arch=Architecture(sizes), max_epochs=2), Dataset(imgs, labs, "train"),
                out_dir=tmp_path)
    n = len(labs)
    for (w, vw), st in zip(ref_hist, res.history):
        assert abs(st.train_error - 100.0 * w / n) <= 100.0 / n + 1e-9
        assert abs(st.val_error - 100.0 * vw / n) <= 100.0 / n + 1e-9
    # weights of the last epoch (best_mlp may be earlier): compare the final net
    # through the checkpoint of the best epoch when it is the last one
    if res.best_epoch == 1:
        ck = load_checkpoint((tmp_path / "best.dmlp").read_bytes())
        for g, r in zip(ck.mlp.layers, ref_layers):
            assert np.abs(g - r).max() <= 1e-5 * np.abs(r).max()
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
