"""DeviceNet: the device-resident network state behind the C-ABI.

Owns one `dmlp_net` (include/dmlp.h).  Device buffers passed in and out are
torch CUDA tensors (PyTorch is the plumbing: allocation, streams,
torch.distributed); all arithmetic runs in libdmlp's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import SizeMismatch


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1003_0358_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def current_stream_handle(device: int = 0) -> ctypes.c_void_p:
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class DeviceNet:
    """Padded, device-resident copy of an Mlp plus the persistent-kernel state."""

    def __init__(self, layer_sizes, device: int = 0, residency: str = "auto", n_ctas: int = 0,
                 all_paths: bool = False):
        _torch()
        self.layer_sizes = tuple(int(s) for s in layer_sizes)
        self.device = int(device)
        sizes = (ctypes.c_int32 * len(self.layer_sizes))(*self.layer_sizes)
        h = ctypes.c_void_p()
        if isinstance(residency, int):  # explicit resident-layer bitmask
            code = 0x10000 | residency
        else:
            code = (_lib.RES_AUTO | 0x20000) if residency == "auto-noreg" else _lib.RESIDENCY[residency]
        if all_paths:  # kernel instance with every residency path (sanitizer coverage)
            code |= 0x40000
        _lib.check(_lib.lib().dmlp_net_create(self.device, sizes, len(self.layer_sizes), code,
                                              int(n_ctas), ctypes.byref(h)), "dmlp_net_create")
        self._h = h
        r, c, t, s = (ctypes.c_int32() for _ in range(4))
        _lib.check(_lib.lib().dmlp_net_info(self._h, ctypes.byref(r), ctypes.byref(c),
                                            ctypes.byref(t), ctypes.byref(s)), "dmlp_net_info")
        self.residency = {v: k for k, v in _lib.RESIDENCY.items()}[r.value]
        self.n_ctas, self.threads, self.smem_bytes = c.value, t.value, s.value
        where = (ctypes.c_int32 * len(self.layer_sizes))()
        _lib.check(_lib.lib().dmlp_net_layer_residency(self._h, where), "dmlp_net_layer_residency")
        #: per weight layer: "l2" (streamed every sample), "smem" or "reg" (register file)
        self.layer_residency = [("l2", "smem", "reg")[where[i]]
                                for i in range(len(self.layer_sizes) - 1)]
        rc = (ctypes.c_int32 * len(self.layer_sizes))()
        tc = (ctypes.c_int32 * len(self.layer_sizes))()
        _lib.check(_lib.lib().dmlp_net_layer_regcols(self._h, rc, tc), "dmlp_net_layer_regcols")
        #: per weight layer: columns of every owned row held in registers / in
        #: the register plan's shared-memory tail (0 unless "reg")
        self.layer_reg_cols = [int(rc[i]) for i in range(len(self.layer_sizes) - 1)]
        self.layer_tail_cols = [int(tc[i]) for i in range(len(self.layer_sizes) - 1)]
        l1 = (ctypes.c_int32 * (len(self.layer_sizes) - 1))()
        _lib.check(_lib.lib().dmlp_net_layer_l1rows(self._h, l1), "dmlp_net_layer_l1rows")
        # rows per CTA of a streamed layer served from L1 (0: none)
        self.layer_l1_rows = [int(l1[i]) for i in range(len(self.layer_sizes) - 1)]

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().dmlp_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def shapes(self):
        s = self.layer_sizes
        return [(o, i + 1) for i, o in zip(s[:-1], s[1:])]

    # -- weights (K5 pack / unpack) ---------------------------------------------
    def set_layers(self, layers) -> None:
        if len(layers) != len(self.shapes):
            raise SizeMismatch(f"{len(layers)} layers for a {len(self.shapes)}-layer net")
        for li, (w, shape) in enumerate(zip(layers, self.shapes)):
            if tuple(w.shape) != shape:
                raise SizeMismatch(f"layer {li} shape {tuple(w.shape)}, want {shape}")
            if isinstance(w, np.ndarray):
                w = np.ascontiguousarray(w, dtype=np.float32)
                p = w.ctypes.data_as(ctypes.c_void_p)
            else:  # torch tensor (host or device)
                w = w.contiguous().float()
                if w.is_cuda:  # the copy/conversion (or a broadcast) runs on torch's
                    # stream; dmlp_net_set_layer reads on the net's own stream
                    _torch().cuda.current_stream(w.device).synchronize()
                p = _ptr(w)
            _lib.check(_lib.lib().dmlp_net_set_layer(self._h, li, p, w.size if isinstance(
                w, np.ndarray) else w.numel()), "dmlp_net_set_layer")

    def get_layers(self) -> list[np.ndarray]:
        out = []
        for li, shape in enumerate(self.shapes):
            w = np.empty(shape, dtype=np.float32)
            _lib.check(_lib.lib().dmlp_net_get_layer(self._h, li, w.ctypes.data_as(ctypes.c_void_p),
                                                     w.size), "dmlp_net_get_layer")
            out.append(w)
        return out

    # -- in-kernel profile ----------------------------------------------------------
    def profile(self, enable: bool = True) -> None:
        _lib.check(_lib.lib().dmlp_net_profile(self._h, int(bool(enable))), "dmlp_net_profile")

    PROFILE_SLOTS = ("loop", "exchange", "head", "fwd", "fwd_xchg", "out_part", "out_xchg",
                     "out_stage", "bwd_part", "bwd_upd", "bwd_xchg", "upd0", "smid", "s13", "s14",
                     "s15")

    LAYER_KINDS = ("fwd", "fwd_gather", "bwd_part", "bwd_upd", "bwd_gather")

    def read_profile(self) -> dict:
        """Per-phase cycles summed over CTAs since the last read (thread 0's
        view), the exchange ("grid-sync stall") fraction, and under "layers"
        the per-layer split (LAYER_KINDS) of the layer phases."""
        n = 16 + 5 * 16
        buf = (ctypes.c_int64 * n)()
        _lib.check(_lib.lib().dmlp_net_read_profile_all(self._h, buf, n),
                   "dmlp_net_read_profile_all")
        d = {k: buf[i] for i, k in enumerate(self.PROFILE_SLOTS) if k != "smid"}
        d["exchange_fraction"] = (d["exchange"] / d["loop"]) if d["loop"] else 0.0
        L = len(self.layer_sizes) - 1
        d["layers"] = [{k: buf[16 + 5 * l + j] for j, k in enumerate(self.LAYER_KINDS)}
                       for l in range(L)]
        return d

    def read_profile_cta(self):
        """Per-CTA profile since the last read: (sm, slots) -- the SM id each
        CTA ran on (valid when one launch was profiled) and the raw
        (n_ctas, 96) cycle slots (layout as read_profile)."""
        buf = np.zeros((self.n_ctas, 96), dtype=np.int64)
        _lib.check(_lib.lib().dmlp_net_read_profile_cta(self._h,
                                                        buf.ctypes.data_as(ctypes.c_void_p)),
                   "dmlp_net_read_profile_cta")
        return buf[:, 12] - 1, buf

    def trace(self, sample: int = -1):
        """Arm a one-sample %globaltimer trace for the next launches (sample
        >= 0) and return the previous recording as (n_ctas, 64) uint64."""
        marks = np.zeros((self.n_ctas, 64), dtype=np.uint64)
        _lib.check(_lib.lib().dmlp_net_trace(self._h, int(sample),
                                             marks.ctypes.data_as(ctypes.c_void_p)),
                   "dmlp_net_trace")
        return marks

    # -- training -----------------------------------------------------------------
    def train_step(self, x: np.ndarray, digit: int, eta: float) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32).ravel())
        if x.shape[0] != self.layer_sizes[0]:
            raise SizeMismatch(f"input length {x.shape[0]}, layer fan_in {self.layer_sizes[0]}")
        if eta < 0:
            raise ValueError("eta must be non-negative")
        y = np.empty(self.layer_sizes[-1], dtype=np.float32)
        _lib.check(_lib.lib().dmlp_train_step(self._h, x.ctypes.data_as(ctypes.c_void_p),
                                              int(digit), float(np.float32(eta)),
                                              y.ctypes.data_as(ctypes.c_void_p)),
                   "dmlp_train_step")
        return y

    def _check_cuda(self, name, t, dtype, dim=None):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name} must be a CUDA tensor on cuda:{self.device}")
        if t.dtype != dtype:
            raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
        if dim is not None and t.dim() != dim:
            raise SizeMismatch(f"{name} must have {dim} dimensions, got shape {tuple(t.shape)}")

    def train_epoch(self, x, labels, order, eta: float, wrong, y_last=None, stream=None,
                    pred=None, check_order: bool = True) -> None:
        """Asynchronous on `stream` (default: torch's current stream).

        x: (n, >=fan_in) f32 CUDA tensor, unit column stride; labels: (n,) u8;
        order: (m,) i32 with values in [0, n), or None; wrong: int64 CUDA
        scalar accumulating argmax errors; pred (optional): (m,) u8 receiving
        every sample's argmax in training order."""
        torch = _torch()
        if eta < 0:
            raise ValueError("eta must be non-negative")
        self._check_cuda("x", x, torch.float32, 2)
        self._check_cuda("labels", labels, torch.uint8, 1)
        self._check_cuda("wrong", wrong, torch.int64)
        if x.stride(1) != 1 or x.shape[1] < self.layer_sizes[0]:
            raise SizeMismatch(f"x must be (n, >= {self.layer_sizes[0]}) with unit column stride")
        if labels.numel() < x.shape[0] or not labels.is_contiguous():
            raise SizeMismatch(f"{labels.numel()} labels for {x.shape[0]} rows")
        if order is not None:
            self._check_cuda("order", order, torch.int32, 1)
            if not order.is_contiguous():
                raise ValueError("order must be contiguous")
            if check_order and order.numel() and (int(order.min()) < 0 or
                                                  int(order.max()) >= x.shape[0]):
                raise ValueError(f"order values must lie in [0, {x.shape[0]})")
        n = int(order.numel()) if order is not None else int(x.shape[0])
        if pred is not None:
            self._check_cuda("pred", pred, torch.uint8, 1)
            if pred.numel() < n or not pred.is_contiguous():
                raise SizeMismatch(f"pred holds {pred.numel()} entries for {n} samples")
        if y_last is not None:
            self._check_cuda("y_last", y_last, torch.float32)
        ldx = int(x.stride(0))
        st = stream if stream is not None else current_stream_handle(self.device)
        _lib.check(_lib.lib().dmlp_train_epoch(self._h, _ptr(x), ldx, _ptr(labels), _ptr(order),
                                               n, float(np.float32(eta)), _ptr(wrong),
                                               _ptr(y_last), _ptr(pred), st), "dmlp_train_epoch")

    # -- evaluation ---------------------------------------------------------------
    def forward_batch(self, x, out=None, stream=None):
        torch = _torch()
        n = int(x.shape[0])
        if x.dim() != 2 or x.shape[1] != self.layer_sizes[0] or not x.is_contiguous():
            raise SizeMismatch(f"batch shape {tuple(x.shape)}, want (n, {self.layer_sizes[0]})")
        if out is None:
            out = torch.empty((n, self.layer_sizes[-1]), dtype=torch.float32, device=x.device)
        st = stream if stream is not None else current_stream_handle(self.device)
        _lib.check(_lib.lib().dmlp_forward_batch(self._h, _ptr(x), n, _ptr(out), st),
                   "dmlp_forward_batch")
        return out

    def eval_counts(self, x, labels, counts=None, guess=None, stream=None):
        """counts (int64[102]) += {wrong, confusion[10][10], second_correct}."""
        torch = _torch()
        n = int(x.shape[0])
        if x.dim() != 2 or x.shape[1] != self.layer_sizes[0] or not x.is_contiguous():
            raise SizeMismatch(f"batch shape {tuple(x.shape)}, want (n, {self.layer_sizes[0]})")
        self._check_cuda("x", x, torch.float32, 2)
        self._check_cuda("labels", labels, torch.uint8, 1)
        if labels.numel() != n or not labels.is_contiguous():
            raise SizeMismatch(f"{labels.numel()} labels for {n} samples")
        if counts is None:
            counts = torch.zeros(102, dtype=torch.int64, device=x.device)
        self._check_cuda("counts", counts, torch.int64, 1)
        if counts.numel() != 102:
            raise SizeMismatch("counts must hold 102 int64")
        if guess is not None:
            self._check_cuda("guess", guess, torch.int32, 2)
            if tuple(guess.shape) != (n, 2) or not guess.is_contiguous():
                raise SizeMismatch(f"guess must be ({n}, 2) int32")
        st = stream if stream is not None else current_stream_handle(self.device)
        _lib.check(_lib.lib().dmlp_eval_counts(self._h, _ptr(x), _ptr(labels), n, _ptr(counts),
                                               _ptr(guess), st), "dmlp_eval_counts")
        return counts
