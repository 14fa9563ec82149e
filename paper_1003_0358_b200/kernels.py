"""On-line back-propagation operators (reference kernels.py:329-361 interface).

`train_step` keeps the reference signature.  The arithmetic runs in
libdmlp's persistent sm_100a kernel (csrc/train_kernel.cu) launched for one
sample: full forward, output delta, backward of the deltas through the OLD
weights, and the rank-1 updates, fused per layer.  `variant` is the
reference's operator-selection seam (kernels.py:315, trainer.py:43):
"cuda" is this implementation; the reference names "tiled" and "naive" are
accepted as aliases so reference configurations run unchanged -- both
select the same CUDA kernel (results agree with the reference's tiled
arithmetic within the tolerance documented in DESIGN.md §5).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .network import Mlp

VARIANTS = ("cuda", "tiled", "naive")


@dataclass(frozen=True)
class TileScheme:
    """Accepted for signature compatibility (kernels.py:27-40); the CUDA
    kernel's partitioning is fixed by its row-ownership design."""

    segment: int = 32
    tile: int = 32
    staged_stride: int = 33
    update_width: int = 16

    def __post_init__(self):
        if min(self.segment, self.tile, self.update_width) < 1:
            raise ValueError("tile constants must be positive")
        if self.staged_stride < self.tile:
            raise ValueError("staged_stride must cover a full tile row")


DEFAULT_SCHEME = TileScheme()


def check_variant(variant: str) -> None:
    if variant not in VARIANTS:
        raise ValueError(f"variant must be one of {VARIANTS}, got {variant!r}")


def train_step(mlp: Mlp, inputs, digit: int, eta: float, variant: str = "cuda",
               scheme: TileScheme = DEFAULT_SCHEME) -> np.ndarray:
    """One on-line update of `mlp` (in place); returns the output activations
    computed before the update."""
    check_variant(variant)
    dev = mlp.device_net()
    y = dev.train_step(inputs, int(digit), eta)
    mlp.mark_device_updated()
    return y
