"""CPU oracle for the on-line BP / deformation / evaluation hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, and only as the checker or
the CPU baseline.  The product package (paper_1003_0358_b200) never imports
this module.

Arithmetic lives in dmlp_oracle.c (a C restatement of the reference's numba
kernels and numpy/scipy deformation, compiled by oracle/Makefile into
oracle/liboracle.so).  The pieces the reference computes with plain numpy
(output deltas with numpy's SIMD float32 tanh, kernels.py:229-236; the
batched OpenBLAS evaluation forward, network.py:118-130; ranking,
network.py:133-135) are restated here with the same numpy calls.

Pinned against the reference itself by tests/test_oracle_golden.py using
the fixtures that tests/golden/make_golden.py generated from
/root/reference (see that script).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

A = 1.7159  # network.py:13
B = 0.6666  # network.py:14
GRID = 29  # deform.py:21

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc)."""
    if force or not os.path.exists(LIB_PATH) or (
        os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "dmlp_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


class _DeformParamsC(ctypes.Structure):
    _fields_ = [
        ("sigma_lo", ctypes.c_double), ("sigma_hi", ctypes.c_double),
        ("alpha_lo", ctypes.c_double), ("alpha_hi", ctypes.c_double),
        ("beta_default", ctypes.c_double), ("beta_reduced", ctypes.c_double),
        ("gamma_lo", ctypes.c_double), ("gamma_hi", ctypes.c_double),
        ("kernel_size", ctypes.c_int),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64, f32 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
        L.or_splitmix64.restype = u64
        L.or_splitmix64.argtypes = [u64]
        L.or_stream_key.argtypes = [u64, P, i32, P]
        L.or_philox_words.argtypes = [P, i64, P]
        L.or_upscale_batch.argtypes = [P, i64, P]
        L.or_deform_batch.argtypes = [P, P, i64, i64, u64, u64, P, P, i32]
        L.or_deform_injected.argtypes = [P, P, P, ctypes.c_double, ctypes.c_double, i32,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         i32, P]
        L.or_fp_tiled.argtypes = [P, i32, i32, P, P, P]
        L.or_fp_naive.argtypes = [P, i32, i32, P, P, P]
        L.or_bp_tiled.argtypes = [P, i32, i32, P, P, P]
        L.or_bp_naive.argtypes = [P, i32, i32, P, P, P]
        L.or_update.argtypes = [P, i32, i32, P, P, f32]
        L.or_tanhf.restype = f32
        L.or_tanhf.argtypes = [f32]
        L.or_set_threads.restype = i32
        L.or_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> int:
    return lib().or_set_threads(int(n))


# --- RNG (rng.py) --------------------------------------------------------------

def stream_key(seed: int, *path: int) -> tuple[int, int]:
    """rng.py:27-32."""
    p = np.array([x & 0xFFFFFFFFFFFFFFFF for x in path], dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lib().or_stream_key(seed & 0xFFFFFFFFFFFFFFFF, _p(p), len(path), _p(out))
    return int(out[0]), int(out[1])


def philox_words(key: tuple[int, int], n: int) -> np.ndarray:
    """First n u64 outputs of numpy's Philox(key=key) (rng.py:35-38)."""
    k = np.array(key, dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    lib().or_philox_words(_p(k), n, _p(out))
    return out


def substream(seed: int, *path: int) -> np.random.Generator:
    """rng.py:35-38 (numpy Generator over Philox with the derived key)."""
    key = np.array(stream_key(seed, *path), dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


# --- deformation (deform.py) ---------------------------------------------------

@dataclass(frozen=True)
class DeformParams:
    """deform.py:40-68 defaults."""

    sigma_range: tuple = (5.0, 6.0)
    alpha_range: tuple = (36.0, 38.0)
    beta_default: float = 15.0
    beta_reduced: float = 7.5
    gamma_range: tuple = (15.0, 20.0)
    kernel_size: int = 21

    def c(self) -> _DeformParamsC:
        return _DeformParamsC(self.sigma_range[0], self.sigma_range[1], self.alpha_range[0],
                              self.alpha_range[1], self.beta_default, self.beta_reduced,
                              self.gamma_range[0], self.gamma_range[1], self.kernel_size)


def identity_params() -> DeformParams:
    return DeformParams(alpha_range=(0.0, 0.0), beta_default=0.0, beta_reduced=0.0,
                        gamma_range=(0.0, 0.0))


def upscale_dataset(images: np.ndarray) -> np.ndarray:
    """deform.py:250-257: (n,28,28) u8 -> (n,841) f32."""
    imgs = np.ascontiguousarray(images, dtype=np.uint8)
    out = np.empty((imgs.shape[0], GRID * GRID), dtype=np.float32)
    lib().or_upscale_batch(_p(imgs), imgs.shape[0], _p(out))
    return out


def deform_epoch(images, labels, params: DeformParams, seed: int, epoch: int,
                 first: int = 0, threads: int = 0) -> np.ndarray:
    """deform.py:217-247 over indices [first, first+n): (n,29,29) f32."""
    imgs = np.ascontiguousarray(images, dtype=np.uint8)
    labs = np.ascontiguousarray(labels, dtype=np.uint8)
    n = imgs.shape[0]
    out = np.empty((n, GRID, GRID), dtype=np.float32)
    pc = params.c()
    lib().or_deform_batch(_p(imgs), _p(labs), first, n, seed, epoch, ctypes.byref(pc),
                          _p(out), threads)
    return out


def deform_injected(image, noise_dx, noise_dy, sigma, alpha, mode, angle, sx, sy,
                    kernel_size: int = 21) -> np.ndarray:
    """deform.py:203-214 with the random draws supplied by the caller."""
    img = np.ascontiguousarray(image, dtype=np.uint8)
    ndx = np.ascontiguousarray(noise_dx, dtype=np.float64)
    ndy = np.ascontiguousarray(noise_dy, dtype=np.float64)
    out = np.empty((GRID, GRID), dtype=np.float32)
    lib().or_deform_injected(_p(img), _p(ndx), _p(ndy), sigma, alpha, int(mode), angle, sx,
                             sy, kernel_size, _p(out))
    return out


# --- training (kernels.py tiled variant) ---------------------------------------

def forward_tiled(w: np.ndarray, x: np.ndarray):
    """kernels.py:209-219."""
    fo, ld = w.shape
    a = np.empty(fo, dtype=np.float32)
    y = np.empty(fo, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    lib().or_fp_tiled(_p(w), fo, ld - 1, _p(x), _p(a), _p(y))
    return a, y


def forward_naive(w: np.ndarray, x: np.ndarray):
    """kernels.py:189-196."""
    fo, ld = w.shape
    a = np.empty(fo, dtype=np.float32)
    y = np.empty(fo, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    lib().or_fp_naive(_p(w), fo, ld - 1, _p(x), _p(a), _p(y))
    return a, y


def output_deltas(outputs: np.ndarray, pre: np.ndarray, digit: int) -> np.ndarray:
    """kernels.py:222-236 (numpy float32 arithmetic, numpy SIMD tanh)."""
    t = np.full(outputs.shape[0], -1.0, dtype=outputs.dtype)
    t[digit] = 1.0
    a = np.asarray(pre, dtype=outputs.dtype)
    th = np.tanh(outputs.dtype.type(B) * a)
    deriv = outputs.dtype.type(A) * outputs.dtype.type(B) * (1 - th * th)
    return (t - outputs) * deriv


def backprop_tiled(w: np.ndarray, delta_down: np.ndarray, a_up: np.ndarray) -> np.ndarray:
    """kernels.py:270-284."""
    fo, ld = w.shape
    du = np.empty(ld - 1, dtype=np.float32)
    dd = np.ascontiguousarray(delta_down, dtype=np.float32)
    au = np.ascontiguousarray(a_up, dtype=np.float32)
    lib().or_bp_tiled(_p(w), fo, ld - 1, _p(dd), _p(au), _p(du))
    return du


def backprop_naive(w: np.ndarray, delta_down: np.ndarray, a_up: np.ndarray) -> np.ndarray:
    """kernels.py:74-83 (the reference's naive variant)."""
    fo, ld = w.shape
    du = np.empty(ld - 1, dtype=np.float32)
    dd = np.ascontiguousarray(delta_down, dtype=np.float32)
    au = np.ascontiguousarray(a_up, dtype=np.float32)
    lib().or_bp_naive(_p(w), fo, ld - 1, _p(dd), _p(au), _p(du))
    return du


def update(w: np.ndarray, delta: np.ndarray, y_in: np.ndarray, eta: float) -> None:
    """kernels.py:299-310 (in place)."""
    fo, ld = w.shape
    d = np.ascontiguousarray(delta, dtype=np.float32)
    y = np.ascontiguousarray(y_in, dtype=np.float32)
    lib().or_update(_p(w), fo, ld - 1, _p(d), _p(y), float(np.float32(eta)))


def train_step(layers: list, x, digit: int, eta: float, variant: str = "tiled") -> np.ndarray:
    """kernels.py:329-361: FP all layers, output delta, BP, updates.  variant
    "tiled" (the one trainer.train uses) or "naive" (kernels.py:58-94; its
    arithmetic differs from "tiled" only in the summation orders).

    Mutates `layers` (list of C-contiguous float32 (fo, fi+1)) in place and
    returns the output activations."""
    fwd, bwd = (forward_tiled, backprop_tiled) if variant == "tiled" else (forward_naive,
                                                                          backprop_naive)
    x0 = np.ascontiguousarray(np.asarray(x, dtype=np.float32).ravel())
    pre, out = [], []
    h = x0
    for w in layers:
        a, y = fwd(w, h)
        pre.append(a)
        out.append(y)
        h = y
    deltas = [None] * len(layers)
    deltas[-1] = output_deltas(out[-1], pre[-1], digit)
    for li in range(len(layers) - 1, 0, -1):
        deltas[li - 1] = bwd(layers[li], deltas[li], pre[li - 1])
    for li, w in enumerate(layers):
        update(w, deltas[li], x0 if li == 0 else out[li - 1], eta)
    return out[-1]


def train_epoch(layers: list, images, labels, eta: float, order=None, preds=None,
                variant: str = "tiled") -> int:
    """trainer.py:104-123: returns the number of wrong argmax predictions;
    `preds` (optional list) receives every sample's argmax in training order."""
    n = len(labels)
    flat = np.asarray(images, dtype=np.float32).reshape(n, -1)
    order = np.arange(n) if order is None else order
    wrong = 0
    for i in order:
        y = train_step(layers, flat[i], int(labels[i]), eta, variant)
        p = int(np.argmax(y))
        if preds is not None:
            preds.append(p)
        if p != int(labels[i]):
            wrong += 1
    return wrong


# --- network / evaluation ------------------------------------------------------

def layer_shapes(sizes):
    """network.py:61-64."""
    return [(o, i + 1) for i, o in zip(sizes[:-1], sizes[1:])]


def count_weights(sizes) -> int:
    """network.py:70-73."""
    return sum((i + 1) * o for i, o in zip(sizes[:-1], sizes[1:]))


def init_layers(seed: int, sizes) -> list:
    """network.py:109-115 with substream(seed, STREAM_INIT=1) (trainer.py:144)."""
    rng = substream(seed, 1)
    return [rng.uniform(-0.05, 0.05, size=s).astype(np.float32) for s in layer_shapes(sizes)]


def forward_batch(layers: list, x: np.ndarray) -> np.ndarray:
    """network.py:118-130 (OpenBLAS sgemm + numpy tanh)."""
    x = np.asarray(x, dtype=np.float32)
    for w in layers:
        a = x @ w[:, :-1].T + w[:, -1]
        x = A * np.tanh(B * a)
    return x


def rank_outputs(outputs: np.ndarray) -> np.ndarray:
    """network.py:133-135."""
    return np.argsort(-outputs, axis=-1, kind="stable")


def eval_counts(outputs: np.ndarray, labels: np.ndarray):
    """eval_report.py:36-67 counting: (wrong, confusion (10,10), second_correct)."""
    ranked = rank_outputs(outputs)
    g1, g2 = ranked[:, 0], ranked[:, 1]
    truth = np.asarray(labels).astype(np.int64)
    conf = np.zeros((10, 10), dtype=np.int64)
    np.add.at(conf, (truth, g1), 1)
    wrong = np.nonzero(g1 != truth)[0]
    second = int(np.count_nonzero(g2[wrong] == truth[wrong]))
    return int(len(wrong)), conf, second, wrong
