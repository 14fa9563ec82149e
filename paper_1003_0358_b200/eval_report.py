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


def evaluate(mlp: Mlp, test: Dataset) -> EvalReport:
    n = len(test)
    if n == 0:
        return EvalReport(0.0, [], np.zeros((10, 10), dtype=np.int64), 0, 0)
    x, counts, guess = _device_eval(mlp, test.images, test.labels, True)
    c = counts.cpu().numpy()
    g = guess.cpu().numpy()
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
