"""K6 microbenchmarks: on-chip / L2 / HBM bandwidth and the exchange floor.

    python -m paper_1003_0358_b200.microbench
"""

from __future__ import annotations

import ctypes
import json

from . import _lib


def run(kind: int, nbytes: int = 0, iters: int = 1, n_ctas: int = 0) -> tuple[float, float]:
    s, c = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().dmlp_bench(kind, nbytes, iters, n_ctas, ctypes.byref(s),
                                     ctypes.byref(c)), "dmlp_bench")
    return s.value, c.value


def prims() -> dict:
    buf = (ctypes.c_double * 8)()
    _lib.check(_lib.lib().dmlp_bench_prims(buf), "dmlp_bench_prims")
    names = ["syncthreads", "scaled_tanh", "fdiv", "warp_reduce", "l2_load", "relaxed_load",
             "smem_load"]
    return {f"cyc_{k}": round(buf[i], 1) for i, k in enumerate(names)}


def exchange_only() -> dict:
    out = {}
    for R in (4, 16):
        for v in (4, 5):
            rounds = 3000
            s, cyc = run(5, v | (R << 8), rounds, 148)
            out[f"xchg_{'EF'[v - 4]}_R{R}_cycles"] = round(cyc / rounds, 1)
    return out


def measure() -> dict:
    info = _lib.device_info(0)
    out = {"sms": info["sms"], "l2_bytes": info["l2_bytes"], **prims()}
    for label, nbytes, iters in [("l2_48MB", 48 << 20, 20), ("l2_24MB", 24 << 20, 40),
                                 ("hbm_2GB", 2 << 30, 2)]:
        s, _ = run(0, nbytes, iters)
        out[f"read_{label}_GBs"] = round(nbytes * iters / s / 1e9, 1)
        s, _ = run(1, nbytes, iters)
        out[f"rw_{label}_GBs"] = round(2 * nbytes * iters / s / 1e9, 1)
    s, cyc = run(2, 0, 200)
    out["smem_rw_GBs"] = round(info["sms"] * 131072 * 2 * 200 / s / 1e9, 1)
    out["smem_rw_B_per_clk_per_sm"] = round(131072 * 2 * 200 / cyc, 1)
    names = ["relaxed", "cg", "backoff64ns", "line_per_producer", "replicas8", "replicas16",
             "mailbox"]
    for n in (148, 64, 16):
        for v, name in enumerate(names):
            if n != 148 and v not in (3, 6):
                continue
            rounds = 5000
            s, cyc = run(3, v, rounds, n)
            out[f"hop_cycles_{name}_{n}ctas"] = round(cyc / rounds, 1)
    for R in (4, 16):  # R <= 16: one value per warp of a 512-thread CTA
        for v, name in enumerate(["A_wordflags", "B_lineflags", "C_fence_flag", "D_release",
                                  "E_lines_allinflight", "F_warpwords_allinflight"]):
            rounds = 3000
            s, cyc = run(5, v | (R << 8), rounds, 148)
            out[f"xchg_{name}_R{R}_cycles"] = round(cyc / rounds, 1)
    return out


if __name__ == "__main__":
    print(json.dumps(measure()))
