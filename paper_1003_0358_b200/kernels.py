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


# --- gradient oracle (kernels.py:364-418), fp64 on the GPU -------------------


def _gradient_check_raw(mlp: Mlp, inputs, digit: int, step: float):
    import ctypes

    from . import _lib

    sizes = tuple(int(s) for s in mlp.arch.layer_sizes)
    w = np.concatenate([np.asarray(l, dtype=np.float64).ravel() for l in mlp.layers])
    x = np.ascontiguousarray(np.asarray(inputs, dtype=np.float64).ravel())
    if x.shape[0] != sizes[0]:
        from .errors import SizeMismatch

        raise SizeMismatch(f"input length {x.shape[0]}, layer fan_in {sizes[0]}")
    gbp = np.empty_like(w)
    gfd = np.empty_like(w)
    worst = ctypes.c_double()
    _lib.check(_lib.lib().dmlp_gradient_check(
        (ctypes.c_int32 * len(sizes))(*sizes), len(sizes), w.ctypes.data, x.ctypes.data,
        int(digit), float(step), gbp.ctypes.data, gfd.ctypes.data, ctypes.byref(worst)),
        "dmlp_gradient_check")
    out_bp, out_fd, pos = [], [], 0
    for fo, fi1 in mlp.arch.layer_shapes():
        out_bp.append(gbp[pos:pos + fo * fi1].reshape(fo, fi1))
        out_fd.append(gfd[pos:pos + fo * fi1].reshape(fo, fi1))
        pos += fo * fi1
    return out_bp, out_fd, float(worst.value)


def backprop_gradients(mlp: Mlp, inputs, digit: int) -> list[np.ndarray]:
    """Analytic dE/dw per layer in float64 (kernels.py:374-389), on the GPU."""
    return _gradient_check_raw(mlp, inputs, digit, 1e-5)[0]


def gradient_check(mlp: Mlp, inputs, digit: int, step: float = 1e-5) -> float:
    """Max relative error of the BP gradient vs central finite differences
    (kernels.py:392-418): float64 whatever the model dtype, denominator
    max(|g_bp|, |g_fd|, 1e-8); every weight's two perturbed forwards run as
    one CTA each (csrc/gradcheck_kernel.cu).  Intended for small nets."""
    return _gradient_check_raw(mlp, inputs, digit, step)[2]
