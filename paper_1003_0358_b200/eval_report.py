"""Test-set evaluation (reference eval_report.py:36-84 interface).

The forward pass, stable top-2 ranking and the {wrong, confusion,
second-guess} counters run in libdmlp (csrc/eval_kernel.cu); only the
misclassified list is assembled on the host.  `evaluate_sharded` splits the
samples across torch.distributed ranks and all-reduces the count vector
(one NCCL all-reduce of int64[102]).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .deform import GRID, upscale_device
from .mnist_io import Dataset
from .network import Mlp

N_CLASSES = 10


@dataclass
class Misclassified:
    index: int
    true: int
    guess1: int
    guess2: int
    image: np.ndarray  # the 29x29 network input


@dataclass
class EvalReport:
    error_percent: float
    misclassified: list[Misclassified]
    confusion: np.ndarray  # (10, 10), rows = true digit
    second_guess_correct: int
    n_samples: int


def _device_eval(mlp: Mlp, images: np.ndarray, labels: np.ndarray, want_guess: bool):
    import torch

    dev = mlp.device_net()
    d = f"cuda:{dev.device}"
    raw = torch.from_numpy(np.ascontiguousarray(images, dtype=np.uint8)).to(d)
    lab = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint8)).to(d)
    x = upscale_device(raw)
    guess = torch.empty((len(labels), 2), dtype=torch.int32, device=d) if want_guess else None
    counts = dev.eval_counts(x, lab, guess=guess)
    return x, counts, guess


def evaluate(mlp: Mlp, test: Dataset, group=None) -> EvalReport:
    """eval_report.py:36-67.  With a torch.distributed `group` (e.g.
    torch.distributed.group.WORLD) this is evaluate_sharded: every rank of the
    group must call it.  group None: this GPU alone."""
    if group is not None:
        return evaluate_sharded(mlp, test, group)
    n = len(test)
    if n == 0:
        return EvalReport(0.0, [], np.zeros((10, 10), dtype=np.int64), 0, 0)
    x, counts, guess = _device_eval(mlp, test.images, test.labels, True)
    return _report(x, counts.cpu().numpy(), guess.cpu().numpy(), test)


def evaluate_sharded(mlp: Mlp, test: Dataset, group=None) -> EvalReport:
    """evaluate() over the ranks of `group` (one process per GPU; every rank
    calls it with the same split): rank 0's weights are broadcast, rank r
    ranks the samples [r*n/G, (r+1)*n/G), ONE all-reduce sums the int64[102]
    count vector, and an all-gather of the (n, 2) top-2 guesses lets every
    rank list the misclassified samples.  Returns the same report on every
    rank, equal to evaluate() on one GPU."""
    import torch

    from .distributed import (_dist, allreduce_counts, broadcast_layers, shard_range,
                              world_info)

    rank, world = world_info(group)
    n = len(test)
    if n == 0:
        return EvalReport(0.0, [], np.zeros((10, 10), dtype=np.int64), 0, 0)
    dev = mlp.device_net()
    broadcast_layers(dev, src=0, group=group)
    if rank != 0:
        mlp.mark_device_updated()
    d = f"cuda:{dev.device}"
    raw = torch.from_numpy(np.ascontiguousarray(test.images, dtype=np.uint8)).to(d)
    lab = torch.from_numpy(np.ascontiguousarray(test.labels, dtype=np.uint8)).to(d)
    x = upscale_device(raw)
    lo, hi = shard_range(n, rank, world)
    width = max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))
    guess = torch.zeros((width, 2), dtype=torch.int32, device=d)
    counts = dev.eval_counts(x[lo:hi], lab[lo:hi], guess=guess[: hi - lo])
    allreduce_counts(counts, group)
    parts = [torch.empty_like(guess) for _ in range(world)]
    _dist().all_gather(parts, guess, group=group)
    g = torch.cat([p[: shard_range(n, r, world)[1] - shard_range(n, r, world)[0]]
                   for r, p in enumerate(parts)]).cpu().numpy()
    return _report(x, counts.cpu().numpy(), g, test)


def _report(x, c: np.ndarray, g: np.ndarray, test: Dataset) -> EvalReport:
    n = len(test)
    truth = np.asarray(test.labels).astype(np.int64)
    wrong = np.nonzero(g[:, 0] != truth)[0]
    xs = x[wrong].cpu().numpy() if len(wrong) else np.empty((0, GRID * GRID), np.float32)
    mis = [Misclassified(int(i), int(truth[i]), int(g[i, 0]), int(g[i, 1]),
                         xs[k].reshape(GRID, GRID)) for k, i in enumerate(wrong)]
    return EvalReport(error_percent=100.0 * int(c[0]) / n, misclassified=mis,
                      confusion=c[1:101].reshape(10, 10).copy(),
                      second_guess_correct=int(c[101]), n_samples=n)


def format_summary(report: EvalReport) -> str:
    lines = [f"test error: {report.error_percent:.2f}% ({len(report.misclassified)} of "
             f"{report.n_samples})",
             f"second guess correct for {report.second_guess_correct} of "
             f"{len(report.misclassified)} misclassified",
             "confusion matrix (rows = true digit):",
             "     " + " ".join(f"{d:>5d}" for d in range(N_CLASSES))]
    for d in range(N_CLASSES):
        lines.append(f"  {d}: " + " ".join(f"{int(v):>5d}" for v in report.confusion[d]))
    return "\n".join(lines)
