"""ctypes binding of libdmlp.so (include/dmlp.h) and status-code mapping.

The product path has no CPU fallback: if libdmlp.so is missing or no
sm_100 device is present, every call raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import EvenSize, InvalidSigma, SizeMismatch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdmlp.so")

DMLP_OK, DMLP_ESIZE, DMLP_EINVAL, DMLP_ECUDA, DMLP_ENCCL = 0, 1, 2, 3, 4
RES_AUTO, RES_L2, RES_SMEM, RES_HYBRID = 0, 1, 2, 3
RESIDENCY = {"auto": RES_AUTO, "l2": RES_L2, "smem": RES_SMEM, "hybrid": RES_HYBRID}

# (function name, restype, argtypes) -- must match include/dmlp.h exactly.
P, i32, i64, u64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
I32P, I64P = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)


class DeformParamsC(ctypes.Structure):
    _fields_ = [
        ("sigma_lo", ctypes.c_double), ("sigma_hi", ctypes.c_double),
        ("alpha_lo", ctypes.c_double), ("alpha_hi", ctypes.c_double),
        ("beta_default", ctypes.c_double), ("beta_reduced", ctypes.c_double),
        ("gamma_lo", ctypes.c_double), ("gamma_hi", ctypes.c_double),
        ("kernel_size", ctypes.c_int32),
    ]


SIGNATURES = [
    ("dmlp_last_error", ctypes.c_char_p, []),
    ("dmlp_device_info", ctypes.c_int, [ctypes.c_int, I32P, I32P, I64P, I64P]),
    ("dmlp_net_create", ctypes.c_int, [ctypes.c_int, I32P, i32, i32, i32, ctypes.POINTER(P)]),
    ("dmlp_net_destroy", ctypes.c_int, [P]),
    ("dmlp_net_info", ctypes.c_int, [P, I32P, I32P, I32P, I32P]),
    ("dmlp_net_layer_residency", ctypes.c_int, [P, I32P]),
    ("dmlp_net_layer_regcols", ctypes.c_int, [P, I32P, I32P]),
    ("dmlp_net_layer_l1rows", ctypes.c_int, [P, I32P]),
    ("dmlp_net_profile", ctypes.c_int, [P, i32]),
    ("dmlp_net_read_profile", ctypes.c_int, [P, I64P]),
    ("dmlp_net_read_profile_all", ctypes.c_int, [P, I64P, i32]),
    ("dmlp_net_read_profile_cta", ctypes.c_int, [P, P]),
    ("dmlp_net_trace", ctypes.c_int, [P, i64, P]),
    ("dmlp_net_set_layer", ctypes.c_int, [P, i32, P, i64]),
    ("dmlp_net_get_layer", ctypes.c_int, [P, i32, P, i64]),
    ("dmlp_train_step", ctypes.c_int, [P, P, i32, f32, P]),
    ("dmlp_train_epoch", ctypes.c_int, [P, P, i64, P, P, i64, f32, P, P, P, P]),
    ("dmlp_forward_batch", ctypes.c_int, [P, P, i64, P, P]),
    ("dmlp_eval_counts", ctypes.c_int, [P, P, P, i64, P, P, P]),
    ("dmlp_deform", ctypes.c_int, [P, P, i64, i64, u64, u64, ctypes.POINTER(DeformParamsC), P, P]),
    ("dmlp_deform_injected", ctypes.c_int, [P, i64, P, P, P, i32, P, P]),
    ("dmlp_upscale", ctypes.c_int, [P, i64, P, P]),
    ("dmlp_bench", ctypes.c_int, [i32, i64, i32, i32, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]),
    ("dmlp_bench_prims", ctypes.c_int, [ctypes.POINTER(ctypes.c_double)]),
    ("dmlp_tanhf_check", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_uint32)]),
    ("dmlp_tanhf_eval", ctypes.c_int, [P, P, i64]),
    ("dmlp_tanhf_fast_check", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64)]),
    ("dmlp_tanhf_fast_eval", ctypes.c_int, [P, P, i64]),
    ("dmlp_gradient_check", ctypes.c_int, [I32P, i32, P, P, i32, ctypes.c_double, P, P,
                                           ctypes.POINTER(ctypes.c_double)]),
]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libdmlp.so (built in-tree by paper_1003_0358_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1003_0358_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().dmlp_last_error().decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    if rc == DMLP_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == DMLP_ESIZE:
        raise SizeMismatch(msg)
    if rc == DMLP_EINVAL:
        if "InvalidSigma" in msg:
            raise InvalidSigma(msg)
        if "EvenSize" in msg:
            raise EvenSize(msg)
        raise ValueError(msg)
    raise RuntimeError(msg)


def device_info(device: int = 0) -> dict:
    sms, smem = ctypes.c_int32(), ctypes.c_int32()
    l2, pl2 = ctypes.c_int64(), ctypes.c_int64()
    check(lib().dmlp_device_info(device, ctypes.byref(sms), ctypes.byref(smem), ctypes.byref(l2),
                                 ctypes.byref(pl2)), "dmlp_device_info")
    return {"sms": sms.value, "smem_per_block": smem.value, "l2_bytes": l2.value,
            "persisting_l2_max": pl2.value}
