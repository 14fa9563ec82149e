"""Training-set deformation on the device (reference deform.py interface).

`deform_epoch` / `upscale_dataset` keep the reference signatures and return
host arrays; `deform_device` / `upscale_device` are the device-resident
entry points the trainer uses (torch CUDA tensors in and out).  All of them
call libdmlp's deformation kernel (csrc/deform_kernel.cu), which re-derives
every image's Philox substream (seed, 2, epoch, index) on the device, so an
epoch is a pure function of (seed, epoch, image, params) for any sharding.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EvenSize, InvalidSigma  # noqa: F401
from .mnist_io import Dataset

GRID = 29
CENTER = (GRID - 1) / 2.0
BACKGROUND = -1.0


def _check_range(name, pair):
    lo, hi = pair
    if not (np.isfinite(lo) and np.isfinite(hi)) or lo > hi:
        raise ValueError(f"{name} must be a finite (lo, hi) with lo <= hi, got {pair}")


@dataclass(frozen=True)
class DeformParams:
    """deform.py:40-68 (angles in degrees, scales in %)."""

    sigma_range: tuple[float, float] = (5.0, 6.0)
    alpha_range: tuple[float, float] = (36.0, 38.0)
    beta_default: float = 15.0
    beta_reduced: float = 7.5
    gamma_range: tuple[float, float] = (15.0, 20.0)
    kernel_size: int = 21

    def __post_init__(self):
        for name in ("sigma_range", "alpha_range", "gamma_range"):
            _check_range(name, getattr(self, name))
        if self.sigma_range[0] <= 0:
            raise InvalidSigma(f"sigma must be positive, got {self.sigma_range}")
        if self.alpha_range[0] < 0 or self.gamma_range[0] < 0:
            raise ValueError("alpha and gamma ranges must be non-negative")
        if self.beta_default < 0 or self.beta_reduced < 0:
            raise ValueError("beta angles must be non-negative")
        if self.kernel_size < 3 or self.kernel_size % 2 == 0:
            raise EvenSize(f"kernel_size must be odd and >= 3, got {self.kernel_size}")

    @classmethod
    def identity(cls) -> "DeformParams":
        return cls(alpha_range=(0.0, 0.0), beta_default=0.0, beta_reduced=0.0,
                   gamma_range=(0.0, 0.0))

    def to_c(self) -> _lib.DeformParamsC:
        return _lib.DeformParamsC(self.sigma_range[0], self.sigma_range[1], self.alpha_range[0],
                                  self.alpha_range[1], self.beta_default, self.beta_reduced,
                                  self.gamma_range[0], self.gamma_range[1], self.kernel_size)


def _torch():
    from .device import _torch as t

    return t()


def _stream(device):
    from .device import current_stream_handle

    return current_stream_handle(device)


def deform_device(raw, labels, params: DeformParams, seed: int, epoch: int, first: int = 0,
                  out=None):
    """raw (n,28,28) u8 CUDA tensor, labels (n,) u8 -> (n,841) f32 CUDA tensor.
    Image k uses substream(seed, 2, epoch, first + k)."""
    torch = _torch()
    n = int(raw.shape[0])
    if out is None:
        out = torch.empty((n, GRID * GRID), dtype=torch.float32, device=raw.device)
    pc = params.to_c()
    with torch.cuda.device(raw.device):  # the kernel launches on the current device
        _lib.check(_lib.lib().dmlp_deform(ctypes.c_void_p(raw.data_ptr()),
                                          ctypes.c_void_p(labels.data_ptr()), int(first), n,
                                          int(seed) & 0xFFFFFFFFFFFFFFFF,
                                          int(epoch) & 0xFFFFFFFFFFFFFFFF, ctypes.byref(pc),
                                          ctypes.c_void_p(out.data_ptr()),
                                          _stream(raw.device.index)), "dmlp_deform")
    return out


def deform_injected_device(raw, noise_dx, noise_dy, scalars, kernel_size: int = 21, out=None):
    """Parity mode: the random draws (noise fields, sigma, alpha, mode,
    angle, sx, sy) are supplied instead of drawn."""
    torch = _torch()
    n = int(raw.shape[0])
    if out is None:
        out = torch.empty((n, GRID * GRID), dtype=torch.float32, device=raw.device)
    with torch.cuda.device(raw.device):
        _lib.check(_lib.lib().dmlp_deform_injected(
            ctypes.c_void_p(raw.data_ptr()), n, ctypes.c_void_p(noise_dx.data_ptr()),
            ctypes.c_void_p(noise_dy.data_ptr()), ctypes.c_void_p(scalars.data_ptr()),
            int(kernel_size), ctypes.c_void_p(out.data_ptr()), _stream(raw.device.index)),
            "dmlp_deform_injected")
    return out


def upscale_device(raw, out=None):
    torch = _torch()
    n = int(raw.shape[0])
    if out is None:
        out = torch.empty((n, GRID * GRID), dtype=torch.float32, device=raw.device)
    with torch.cuda.device(raw.device):
        _lib.check(_lib.lib().dmlp_upscale(ctypes.c_void_p(raw.data_ptr()), n,
                                           ctypes.c_void_p(out.data_ptr()),
                                           _stream(raw.device.index)), "dmlp_upscale")
    return out


def _to_device(arr, device: int = 0):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{device}")


def deform_epoch(train: Dataset, params: DeformParams, seed: int, epoch: int,
                 lanes: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """deform.py:217-247: (deformed (n,29,29) float32, labels).  `lanes` is
    accepted for compatibility; the output is identical for any sharding."""
    n = len(train)
    if n == 0:
        return np.empty((0, GRID, GRID), dtype=np.float32), train.labels
    raw = _to_device(np.asarray(train.images, dtype=np.uint8))
    lab = _to_device(np.asarray(train.labels, dtype=np.uint8))
    out = deform_device(raw, lab, params, seed, epoch)
    return out.cpu().numpy().reshape(n, GRID, GRID), train.labels


def upscale_dataset(ds: Dataset) -> np.ndarray:
    """deform.py:250-257: un-deformed (n, 841) float32 network inputs."""
    n = len(ds)
    if n == 0:
        return np.empty((0, GRID * GRID), dtype=np.float32)
    return upscale_device(_to_device(np.asarray(ds.images, dtype=np.uint8))).cpu().numpy()
