"""World-size-2 gloo tests of the multi-process logic (run on CPU).

The device kernels are replaced by the oracle ONLY as the per-shard checker
here: what is under test is the sharding + all-reduce plumbing of
paper_1003_0358_b200.distributed (shard ranges, count all-reduce, the
deformation shard invariance that lets ranks skip any collective)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1003_0358_b200.distributed import (allreduce_counts, shard_range,
                                                      counts_to_report)
        from paper_1003_0358_b200.synthetic import make_digits

        imgs, labs = make_digits(257, seed=11)
        sizes = (841, 40, 10)
        layers = O.init_layers(3, sizes)
        x = O.upscale_dataset(imgs)
        lo, hi = shard_range(len(labs), rank, world)
        wrong, conf, second, _ = O.eval_counts(O.forward_batch(layers, x[lo:hi]), labs[lo:hi])
        counts = torch.zeros(102, dtype=torch.int64)
        counts[0] = wrong
        counts[1:101] = torch.from_numpy(conf.reshape(-1))
        counts[101] = second
        allreduce_counts(counts)
        rep = counts_to_report(counts)
        # deformation shard: this rank's slice with the global index offset
        shard = O.deform_epoch(imgs[lo:hi], labs[lo:hi], O.DeformParams(), seed=4, epoch=1,
                               first=lo)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), wrong=rep["wrong"],
                 confusion=rep["confusion"], second=rep["second_guess_correct"], shard=shard,
                 lo=lo, hi=hi)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_eval_and_deform(tmp_path, world):
    from oracle import oracle as O
    from paper_1003_0358_b200.synthetic import make_digits

    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    imgs, labs = make_digits(257, seed=11)
    layers = O.init_layers(3, (841, 40, 10))
    wrong, conf, second, _ = O.eval_counts(O.forward_batch(layers, O.upscale_dataset(imgs)), labs)
    for r in res:  # every rank holds the global counts after the all-reduce
        assert int(r["wrong"]) == wrong
        assert np.array_equal(r["confusion"], conf)
        assert int(r["second"]) == second
    full = O.deform_epoch(imgs, labs, O.DeformParams(), seed=4, epoch=1)
    assert np.array_equal(np.concatenate([r["shard"] for r in res]), full)
    assert [(int(r["lo"]), int(r["hi"])) for r in res] == [(0, 128), (128, 257)]


def test_peer_shard_covers_split_without_lead():
    """deform_to_lead's split: the non-lead ranks cover [0, n) in rank order,
    disjoint; the lead deforms nothing (it trains)."""
    from paper_1003_0358_b200.distributed import peer_shard

    for n in (0, 1, 7, 301, 60000):
        for world in (1, 2, 3, 8):
            for lead in {0, world - 1}:
                spans = [peer_shard(n, r, world, lead) for r in range(world)]
                if world == 1:
                    assert spans == [(0, n)]
                    continue
                assert spans[lead] == (0, 0)
                cov = [s for r, s in enumerate(spans) if r != lead]
                assert cov[0][0] == 0 and cov[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(cov, cov[1:]))
