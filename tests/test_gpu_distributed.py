"""World-size-2 tests of the multi-GPU path on ONE GPU.

Two processes share cuda:0 over a gloo process group (NCCL refuses two
ranks on one device; gloo moves CUDA tensors through host memory).  What
runs is the real device path of paper_1003_0358_b200.distributed and of the
sharded entry points -- deform_sharded / gather_deformed, deform_to_lead
(peer-GPU deformation), eval_counts_sharded, broadcast_layers,
evaluate_sharded and trainer.train(group=...) -- and the oracle only checks
the results (reference: deform.py:217-247, eval_report.py:36-67,
trainer.py:130-207)."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIZES = (841, 60, 10)
N_IMG = 301  # odd: ragged shards


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1003_0358_b200.deform import DeformParams, deform_device, upscale_device
        from paper_1003_0358_b200.device import DeviceNet
        from paper_1003_0358_b200.distributed import (broadcast_layers, deform_sharded,
                                                      deform_to_lead, eval_counts_sharded,
                                                      gather_deformed)
        from paper_1003_0358_b200.eval_report import evaluate, evaluate_sharded
        from paper_1003_0358_b200.mnist_io import Dataset
        from paper_1003_0358_b200.network import Architecture, Mlp
        from paper_1003_0358_b200.synthetic import make_digits
        from paper_1003_0358_b200.trainer import TrainConfig, train

        res = {}
        imgs, labs = make_digits(N_IMG, seed=17)
        raw = torch.from_numpy(imgs).cuda()
        lab = torch.from_numpy(labs).cuda()

        # 1. broadcast_layers: rank 1 starts from different weights
        ref = O.init_layers(5, SIZES)
        net = DeviceNet(SIZES)
        net.set_layers(ref if rank == 0 else O.init_layers(6, SIZES))
        broadcast_layers(net, src=0)
        for i, w in enumerate(net.get_layers()):
            res[f"bcast{i}"] = w

        # 2. deformation sharded by image index, assembled with one all-gather
        shard, lo, hi = deform_sharded(raw, lab, DeformParams(), seed=3, epoch=2)
        res["deform_full"] = gather_deformed(shard, N_IMG).cpu().numpy()
        res["deform_lohi"] = np.array([lo, hi])

        # 3. peer deformation to the lead (rank 1 deforms everything here)
        out = torch.full((N_IMG, 841), float("nan"), device="cuda")
        for r in deform_to_lead(raw, lab, DeformParams(), 3, 2, out):
            r.wait()
        torch.cuda.synchronize()
        res["lead_out"] = out.cpu().numpy()

        # 4. sharded evaluation counts (+ one all-reduce)
        x = upscale_device(raw)
        res["counts"] = eval_counts_sharded(net, x, lab).cpu().numpy()

        # 5. evaluate_sharded == evaluate on one GPU
        mlp = Mlp(Architecture(SIZES), [w.copy() for w in (ref if rank == 0 else
                                                           O.init_layers(7, SIZES))])
        rep = evaluate_sharded(mlp, Dataset(imgs, labs, "test"))
        res["ev_err"] = np.array(rep.error_percent)
        res["ev_conf"] = rep.confusion
        res["ev_second"] = np.array(rep.second_guess_correct)
        res["ev_mis"] = np.array([(m.index, m.true, m.guess1, m.guess2)
                                  for m in rep.misclassified], dtype=np.int64).reshape(-1, 4)
        if rank == 0:
            one = evaluate(Mlp(Architecture(SIZES), [w.copy() for w in ref]),
                           Dataset(imgs, labs, "test"))
            res["ev1_err"] = np.array(one.error_percent)
            res["ev1_conf"] = one.confusion
            res["ev1_mis"] = np.array([(m.index, m.true, m.guess1, m.guess2)
                                       for m in one.misclassified], dtype=np.int64).reshape(-1, 4)

        # 6. trainer.train over the group == the single-GPU run, bit for bit
        cfg = TrainConfig(arch=Architecture(SIZES), max_epochs=3, seed=2)
        ds = Dataset(imgs, labs, "train")
        r2 = train(cfg, ds, group=dist.group.WORLD)
        res["tr_hist"] = np.array([(h.train_error, h.val_error) for h in r2.history])
        res["tr_best"] = np.array([r2.best_epoch, r2.best_val_error])
        for i, w in enumerate(r2.best_mlp.layers):
            res[f"tr_w{i}"] = w
        if rank == 0:
            r1 = train(cfg, ds)
            res["tr1_hist"] = np.array([(h.train_error, h.val_error) for h in r1.history])
            res["tr1_best"] = np.array([r1.best_epoch, r1.best_val_error])
            for i, w in enumerate(r1.best_mlp.layers):
                res[f"tr1_w{i}"] = w
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def ws2(tmp_path_factory):
    import torch.multiprocessing as mp

    d = tmp_path_factory.mktemp("ws2")
    mp.spawn(_worker, args=(2, _free_port(), str(d)), nprocs=2, join=True)
    return [dict(np.load(d / f"r{r}.npz")) for r in range(2)]


def test_broadcast_layers_ws2(ws2):
    ref = O.init_layers(5, SIZES)
    for r in ws2:
        for i, w in enumerate(ref):
            assert np.array_equal(r[f"bcast{i}"], w)


def test_deform_sharded_and_to_lead_ws2(ws2):
    import torch

    from paper_1003_0358_b200.deform import DeformParams, deform_device
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(N_IMG, seed=17)
    full = deform_device(torch.from_numpy(imgs).cuda(), torch.from_numpy(labs).cuda(),
                         DeformParams(), 3, 2).cpu().numpy()
    assert [tuple(r["deform_lohi"]) for r in ws2] == [(0, 150), (150, 301)]
    for r in ws2:  # all-gathered shards are byte-identical to the one-GPU epoch
        assert np.array_equal(r["deform_full"], full)
    assert np.array_equal(ws2[0]["lead_out"], full)  # the lead received the peer's epoch
    od = O.deform_epoch(imgs[:64], labs[:64], O.DeformParams(), seed=3, epoch=2)
    assert np.abs(full[:64].reshape(-1, 29, 29) - od).max() <= 1e-5


def test_eval_counts_sharded_ws2(ws2):
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(N_IMG, seed=17)
    out = O.forward_batch(O.init_layers(5, SIZES), O.upscale_dataset(imgs))
    wrong, conf, second, _ = O.eval_counts(out, labs)
    for r in ws2:
        c = r["counts"]
        assert int(c[0]) == wrong and int(c[101]) == second
        assert np.array_equal(c[1:101].reshape(10, 10), conf)


def test_evaluate_sharded_equals_one_gpu_ws2(ws2):
    r0 = ws2[0]
    for r in ws2:  # every rank reports rank 0's weights, equal to the 1-GPU report
        assert float(r["ev_err"]) == float(r0["ev1_err"])
        assert np.array_equal(r["ev_conf"], r0["ev1_conf"])
        assert np.array_equal(r["ev_mis"], r0["ev1_mis"])


def test_train_group_equals_one_gpu_ws2(ws2):
    r0 = ws2[0]
    for r in ws2:
        assert np.array_equal(r["tr_hist"], r0["tr1_hist"])
        assert np.array_equal(r["tr_best"], r0["tr1_best"])
        for i in range(len(SIZES) - 1):
            assert np.array_equal(r[f"tr_w{i}"], r0[f"tr1_w{i}"]), i
