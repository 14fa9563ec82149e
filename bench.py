"""Benchmark of the on-line BP hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A step = one persistent-kernel launch training `--samples` on-line samples
(batch size 1, sequential) of the C4 net 841-2500-2000-1500-1000-500-10
(12,115,010 weights) on deformed synthetic digits already resident in HBM.
`value` = samples/s over the K timed steps (CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks).  `e2e` = the
same metric through the public API (trainer.train_epoch) from pinned host
buffers: the H2D copy of the step's images/labels/order and the D2H read of
the error count are inside the timed region.  Extra keys report the
deformation and evaluation kernels (imgs/s) and the in-kernel profile.

Multi-GPU (torchrun, one rank per GPU): on-line training does not shard
(SPEC: sample s+1 needs the weights after sample s), so every rank trains an
independent replica (seed = rank); value = total samples/s of all replicas
("replicas only", scaling "weak").  Deformation and evaluation shard the
images; the eval counts are all-reduced with NCCL.

`--impl reference` times the reference algorithm on the host CPU through
the oracle port (oracle/, bit-exact with the reference package) on a
bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": (841, 1000, 500, 10),
    "C2": (841, 1500, 1000, 500, 10),
    "C3": (841, 2000, 1500, 1000, 500, 10),
    "C4": (841, 2500, 2000, 1500, 1000, 500, 10),
    "C5": (841,) + (1000,) * 9 + (10,),
}
METRIC = "on-line BP train samples/s (bs=1, 12.11M MLP)"
L2_BYTES = 126 * 1024 * 1024


def count_weights(sizes) -> int:
    return sum((i + 1) * o for i, o in zip(sizes[:-1], sizes[1:]))


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- data


def make_inputs(n_raw: int, seed: int, device: str):
    """Synthetic digits -> device, deformed once (epoch 0) by the CUDA kernel."""
    import numpy as np
    import torch

    from paper_1003_0358_b200.deform import DeformParams, deform_device
    from paper_1003_0358_b200.synthetic import make_digits

    images, labels = make_digits(n_raw, seed=12345 + seed)
    raw = torch.from_numpy(images).to(device)
    lab = torch.from_numpy(labels).to(device)
    x = deform_device(raw, lab, DeformParams(), seed, 0)
    torch.cuda.synchronize()
    return images, labels, raw, lab, x, np


# ----------------------------------------------------------------------------- CPU legs


def cpu_model() -> dict:
    """The host CPU the CPU legs ran on (model name from /proc/cpuinfo, nproc)."""
    name = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    name = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": name, "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


def cpu_train_rate(sizes, seconds: float = 12.0, threads: int | None = None,
                   variant: str = "tiled") -> dict:
    """The reference algorithm (oracle port of kernels.train_step, `variant`
    arithmetic) on the host cores: on-line samples/s over a bounded sample."""
    import numpy as np

    from oracle import oracle as O
    from paper_1003_0358_b200.synthetic import make_digits

    threads = threads or os.cpu_count() or 1
    O.set_threads(threads)
    imgs, labs = make_digits(64, seed=7)
    x = O.deform_epoch(imgs, labs, O.DeformParams(), seed=0, epoch=0).reshape(64, -1)
    layers = O.init_layers(0, sizes)
    for i in range(3):  # warm-up
        O.train_step(layers, x[i], int(labs[i]), 1e-3, variant)
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or n < 5:
        O.train_step(layers, x[n % 64], int(labs[n % 64]), 1e-3, variant)
        n += 1
    dt = time.perf_counter() - t0
    O.set_threads(os.cpu_count() or 1)
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} on-line train_step calls of {sizes} in {dt:.1f}s "
                      f"(oracle/dmlp_oracle.c, {variant} arithmetic, {threads} threads)"}


def cpu_deform_rate(seconds: float = 3.0, threads: int = 1) -> dict:
    """deform_epoch (deform.py:217-247) at lanes=`threads` on a bounded sample."""
    from oracle import oracle as O
    from paper_1003_0358_b200.synthetic import make_digits

    imgs, labs = make_digits(512, seed=3)
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or n == 0:
        O.deform_epoch(imgs, labs, O.DeformParams(), seed=0, epoch=n, threads=threads)
        n += len(imgs)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "imgs/s", "cores": threads, "kind": "port",
            "sample": f"{n} images deformed in {dt:.1f}s (oracle/dmlp_oracle.c, lanes={threads})"}


def cpu_forward_batch_rate(sizes, n_images: int = 10000) -> dict:
    """network.forward_batch (network.py:118-130: OpenBLAS sgemm + numpy tanh)
    on n_images un-deformed inputs, all host threads."""
    import numpy as np

    from oracle import oracle as O

    layers = O.init_layers(0, sizes)
    x = np.random.default_rng(5).uniform(-1, 1, size=(n_images, sizes[0])).astype(np.float32)
    O.forward_batch(layers, x[:256])  # warm-up (BLAS thread pool)
    t0 = time.perf_counter()
    O.forward_batch(layers, x)
    dt = time.perf_counter() - t0
    flops = 2 * sum(i * o for i, o in zip(sizes[:-1], sizes[1:])) * n_images
    return {"value": n_images / dt, "unit": "imgs/s", "cores": os.cpu_count(), "kind": "port",
            "TFLOPs": round(flops / dt / 1e12, 3),
            "sample": f"forward_batch of {n_images} images in {dt:.2f}s (numpy/OpenBLAS sgemm)"}


def cpu_baseline_block(sizes, seconds: float) -> dict:
    """cpu_baseline of the bench line: the headline leg (train_step tiled,
    every host thread) plus the context legs BASELINE.md §2 asks for."""
    cpu = cpu_train_rate(sizes, seconds=seconds)
    short = max(1.0, seconds / 4)
    cpu["cpu"] = cpu_model()
    cpu["legs"] = {
        "train_step_tiled_1thread": cpu_train_rate(sizes, seconds=short, threads=1),
        "train_step_naive_all_threads": cpu_train_rate(sizes, seconds=short, variant="naive"),
        "forward_batch_10k": cpu_forward_batch_rate(sizes),
        "deform_epoch_lanes1": cpu_deform_rate(seconds=short, threads=1),
    }
    for leg in cpu["legs"].values():
        leg["value"] = round(leg["value"], 2)
    cpu["value"] = round(cpu["value"], 2)
    return cpu


# ----------------------------------------------------------------------------- GPU arm


def run_gpu(args) -> dict | None:
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(device))

    from paper_1003_0358_b200 import trainer
    from paper_1003_0358_b200.deform import DeformParams, deform_device, upscale_device
    from paper_1003_0358_b200.device import DeviceNet
    from paper_1003_0358_b200.network import Architecture, init_mlp
    from paper_1003_0358_b200.rng import substream

    sizes = CONFIGS[args.config]
    W = count_weights(sizes)
    n = args.samples
    images, labels, raw, lab, x, _ = make_inputs(n, rank, device)
    order = torch.from_numpy(substream(rank, 3, 0).permutation(n).astype(np.int32)).to(device)

    mlp = init_mlp(substream(rank, 1), Architecture(sizes))
    dn = mlp.device_net(local, args.residency)
    wrong = torch.zeros((), dtype=torch.int64, device=device)
    stream = torch.cuda.current_stream(device)

    assert 0 <= int(order.min()) and int(order.max()) < n  # validated once, not per step

    def step():  # (no host-side range check of `order` inside the timed loop)
        dn.train_epoch(x, lab, order, 1e-3, wrong, check_order=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    for _ in range(args.warmup):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    per_launch_s = ms / 1e3 / args.steps
    sps_rank = n / per_launch_s
    value = world * n * args.steps / (ms_max / 1e3)

    # ---- in-kernel phase profile on one extra (untimed) launch
    dn.profile(True)
    step()
    torch.cuda.synchronize(device)
    prof = dn.read_profile()
    dn.profile(False)

    # ---- end to end through the public API, host (pinned) buffers
    x_host = torch.empty((n, 841), dtype=torch.float32).pin_memory()
    x_host.copy_(x.cpu())
    lab_host = torch.from_numpy(labels).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    trainer.train_epoch(mlp, x_host, lab_host, 1e-3, rng=substream(rank, 3, 99))  # warm-up
    barrier()
    t0 = time.perf_counter()
    for s in range(e2e_steps):
        trainer.train_epoch(mlp, x_host, lab_host, 1e-3, rng=substream(rank, 3, s))
    barrier()
    e2e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_dt], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e = {"value": world * n * e2e_steps / e2e_dt, "unit": "samples/s",
           "h2d_bytes_per_step": n * 841 * 4 + n + n * 4, "d2h_bytes_per_step": 8,
           "api": "paper_1003_0358_b200.trainer.train_epoch(mlp, pinned host images, "
                  "labels, eta, rng)"}

    # ---- deformation kernel: the whole epoch's images, sharded by rank
    nd = args.deform_images
    d_imgs = torch.from_numpy(np.resize(images, (nd, 28, 28))).to(device)
    d_lab = torch.from_numpy(np.resize(labels, nd)).to(device)
    lo, hi = rank * nd // world, (rank + 1) * nd // world
    d_out = torch.empty((hi - lo, 841), dtype=torch.float32, device=device)
    for _ in range(2):
        deform_device(d_imgs[lo:hi], d_lab[lo:hi], DeformParams(), 0, 1, first=lo, out=d_out)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for e in range(3):
        deform_device(d_imgs[lo:hi], d_lab[lo:hi], DeformParams(), 0, 2 + e, first=lo, out=d_out)
    b.record(stream)
    barrier()
    dms = a.elapsed_time(b) / 3
    if world > 1:
        t = torch.tensor([dms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dms = float(t.item())
    deform = {"imgs_per_s": nd / (dms / 1e3), "imgs_per_s_per_gpu": nd / (dms / 1e3) / world,
              "images": nd, "n_gpus": world, "sharding": "image index ranges, no collective",
              "ms_per_epoch": round(dms, 3),
              "bytes_per_img": 4149, "GBs": round(4149 * nd / (dms / 1e3) / 1e9, 1)}
    deform["roofline"] = deform_roofline(deform["imgs_per_s_per_gpu"])

    # ---- evaluation: validation pass over the un-deformed training images,
    # sharded by rank + one all-reduce of the counts (eval_counts_sharded)
    from paper_1003_0358_b200.distributed import broadcast_layers, eval_counts_sharded

    ev = DeviceNet(sizes, device=local)
    ev.set_layers(mlp.layers)
    broadcast_layers(ev, src=0)  # every rank evaluates rank 0's weights
    xv = upscale_device(d_imgs)
    eval_counts_sharded(ev, xv, d_lab)
    barrier()
    a.record(stream)
    counts = eval_counts_sharded(ev, xv, d_lab)
    b.record(stream)
    barrier()
    ems = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ems], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    flops = 2 * sum(i * o for i, o in zip(sizes[:-1], sizes[1:]))
    evaluation = {"imgs_per_s": nd / (ems / 1e3), "imgs_per_s_per_gpu": nd / (ems / 1e3) / world,
                  "images": nd, "n_gpus": world, "wrong": int(counts[0].item()),
                  "sharding": "samples by rank + one NCCL all_reduce of int64[102] (timed)",
                  "TFLOPs": round(flops * nd / (ems / 1e3) / 1e12, 2)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = 12.0 * W * sps_rank / 1e9
    l2 = l2_peak()
    smem_peak = smem_peak_gbs(clk.summary().get("sm_mhz"))
    levels = level_bytes(sizes, dn)
    # L1 shares the shared-memory datapath (128 B/clk/SM): same peak
    t_min = ((levels["smem"] + levels["l1"]) / (smem_peak * 1e9) + levels["l2"] / (l2 * 1e9)
             if l2 else None)
    traffic = profiled_traffic(args.config, n)
    roofline = {
        # the weights live in registers / shared memory / L2 (layer_residency),
        # never in HBM inside the loop: the bound is the L2 read+write peak
        # (BASELINE.md §3), measured live in this run (K6)
        "bound": "l2", "achieved": round(achieved, 1), "peak": l2, "unit": "GB/s",
        "frac": round(achieved / l2, 4) if l2 else None,
        "peak_source": "K6 L2-resident read+write copy (48 MB, one CTA per SM), measured in "
                       "this run (paper_1003_0358_b200/csrc/microbench.cu)",
        "traffic": traffic,
        "traffic_source": (f"DRAM bytes per sample from the committed ncu --set full capture "
                           f"profiles/ncu_train_{args.config.lower()}.json, scaled to {n} "
                           "samples (not measured in this run)") if traffic else None,
        "algorithmic_bytes_per_sample": 12 * W,
        "algorithmic_bytes_per_launch": 12 * W * n,
        "residency": dn.residency,
        # SURVEY.md §8(d) hybrid roofline: t_min = sum over levels of the 12 B
        # per weight each level serves / that level's peak (registers free)
        "hybrid": {
            "bytes_per_sample": levels,
            "smem_peak_GBs": round(smem_peak, 1), "l2_peak_GBs": l2,
            "t_min_us": round(t_min * 1e6, 3) if t_min else None,
            "t_measured_us": round(1e6 / sps_rank, 3),
            "frac_hybrid": round(t_min * sps_rank, 4) if t_min else None,
        },
        "hbm_peak_GBs": hbm_peak, "frac_of_hbm": round(achieved / hbm_peak, 4),
        "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
        "target_samples_per_s_at_0.70_of_l2": round(0.7 * l2 * 1e9 / (12 * W), 1) if l2 else None,
        "exchange_fraction": round(prof["exchange_fraction"], 3),
        "sync_bound": sync_bound(len(sizes) - 1, sps_rank),
    }
    cpu = cpu_baseline_block(sizes, args.cpu_seconds) if args.cpu_seconds > 0 else None
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, world),
        "e2e": {k: (round(v, 1) if isinstance(v, float) else v) for k, v in e2e.items()},
        "gpu_launches": args.steps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "deform": {k: (round(v, 1) if isinstance(v, float) else v) for k, v in deform.items()},
        "eval": {k: (round(v, 1) if isinstance(v, float) else v) for k, v in evaluation.items()},
        "profile_cycles_per_sample": {k: v // max(1, dn.n_ctas) // n for k, v in prof.items()
                                      if k not in ("exchange_fraction", "layers") and v},
        "profile_cycles_per_layer": [
            {k: v // max(1, dn.n_ctas) // n for k, v in lay.items()} for lay in prof["layers"]],
        "layer_residency": dn.layer_residency,
    }
    if world > 1:
        dist.destroy_process_group()
    return line


def bench_config(args, world: int) -> dict:
    """The workload description shared by both arms (same metric, same config)."""
    sizes = CONFIGS[args.config]
    n = args.samples
    return {"workload": f"{args.config} {'-'.join(map(str, sizes))} on-line BP (bs=1), "
                        f"{n} deformed synthetic digits per step",
            "weights": count_weights(sizes), "samples_per_step": n,
            "parallelism": "replicas only" if world > 1 else "single GPU",
            "input_bytes_per_step": n * 841 * 4,
            "l2": (f"inputs larger than L2 ({n * 841 * 4 / 1e6:.0f} MB per step > 126 MB), "
                   if n * 841 * 4 > L2_BYTES else
                   f"inputs SMALLER than L2 ({n * 841 * 4 / 1e6:.0f} MB per step), ")
                  + "each input row read once per step; weights are deliberately kept on chip "
                    "(smem / registers) or in L2"}


def smem_peak_gbs(sm_mhz) -> float:
    """Shared-memory bandwidth of the whole chip: 148 SMs x 128 B/clk at the
    SM clock sampled during the timed region (max clock if none)."""
    mhz = float(sm_mhz or measured_peaks().get("sm_max_mhz", 1965.0))
    return 148 * 128 * mhz * 1e6 / 1e9


def level_bytes(sizes, dn) -> dict:
    """Algorithmic bytes per sample (12 per weight) by the level that serves
    them in the training kernel: registers, shared memory, L1 (the streamed
    layer's rows the kernel keeps there), L2."""
    out = {"reg": 0, "smem": 0, "l1": 0, "l2": 0}
    for li, (fi, fo) in enumerate(zip(sizes[:-1], sizes[1:])):
        fi1 = fi + 1
        where = dn.layer_residency[li] if li < len(sizes) - 2 else "smem"  # output tile: smem
        if where == "reg":
            rc = dn.layer_reg_cols[li]
            out["reg"] += 12 * fo * rc
            out["smem"] += 12 * fo * (fi1 - rc)  # the plan's shared-memory tail
        elif where == "l2" and li < len(dn.layer_l1_rows) and dn.layer_l1_rows[li]:
            rows = -(-fo // dn.n_ctas)  # rows per CTA
            part = 12 * fo * fi1 * min(1.0, dn.layer_l1_rows[li] / rows)
            out["l1"] += int(part)
            out["l2"] += 12 * fo * fi1 - int(part)
        else:
            out[where] += 12 * fo * fi1
    return out


def relaunch_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` without torchrun: re-exec as N ranks (one
    process per GPU, 127.0.0.1 rendezvous), the same launch the driver uses."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def deform_roofline(imgs_per_s: float) -> dict | None:
    """K2 is issue-bound (profiles/ncu_deform.json): its bound is the SM issue
    rate (148 SMs x 4 warp instructions per cycle at the max SM clock) over
    the warp instructions one image takes in the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_deform.json")) as f:
            ipi = json.load(f)["warp_instructions_per_unit"]
    except Exception:
        return None
    mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
    bound = 148 * 4 * mhz * 1e6 / ipi
    return {"bound": "issue", "achieved_imgs_per_s": round(imgs_per_s, 1),
            "peak_imgs_per_s": round(bound, 1), "frac": round(imgs_per_s / bound, 4),
            "warp_instructions_per_img": ipi,
            "source": "profiles/ncu_deform.json (smsp__inst_executed / images)"}


def l2_peak() -> float | None:
    """K6: L2-resident read+write bandwidth (48 MB, one CTA per SM)."""
    try:
        from paper_1003_0358_b200 import microbench

        s, _ = microbench.run(1, 48 << 20, 10)
        return round(2 * (48 << 20) * 10 / s / 1e9, 1)
    except Exception:
        return None


def sync_bound(n_layers: int, sps: float) -> dict | None:
    """SURVEY.md §8(d) sync bound: the 2L-3 all-to-all exchanges a sample
    needs (forward y of hidden layers 0..H-2, output partials, backward
    partials of layers H-1..1), each at the measured floor of a bare
    148-CTA exchange (K6 protocol E, the kernel's poll discipline)."""
    try:
        from paper_1003_0358_b200 import microbench

        rounds = 3000
        s, cyc = microbench.run(5, 4 | (16 << 8), rounds, 148)
    except Exception:
        return None
    hops = max(2 * n_layers - 3, 0)
    hop_us = s / rounds * 1e6
    us = hops * hop_us
    return {"exchanges_per_sample": hops, "hop_us": round(hop_us, 3),
            "hop_cycles": round(cyc / rounds, 1), "us_per_sample": round(us, 2),
            "samples_per_s": round(1e6 / us, 1) if us > 0 else None,
            "share_of_measured_sample": round(us * sps / 1e6, 3)}


def profiled_traffic(cfg: str, samples: int):
    """DRAM bytes (read + write) per launch of `samples` samples, scaled from
    the committed `ncu --set full` capture of the same kernel and config."""
    p = os.path.join(ROOT, "profiles", f"ncu_train_{cfg.lower()}.json")
    try:
        with open(p) as f:
            return round(json.load(f)["dram_bytes_per_unit"] * samples)
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm


def run_reference(args) -> dict | None:
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    sizes = CONFIGS[args.config]
    W = count_weights(sizes)
    per = max(2.0, args.cpu_seconds)
    vals = []
    for _ in range(args.warmup):
        cpu_train_rate(sizes, seconds=per / 4)
    for _ in range(args.steps):
        vals.append(cpu_train_rate(sizes, seconds=per)["value"])
    v = statistics.median(vals)
    cpu = cpu_train_rate(sizes, seconds=1.0)
    cpu["value"] = v
    return {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * per, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": cpu,
        "e2e": {"value": round(v, 3), "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference algorithm = oracle/dmlp_oracle.c (bit-exact with the reference "
                "kernels.train_step tiled variant, pinned by tests/test_oracle_golden.py); the "
                "Python/numba reference itself cannot travel to the GPU host",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--samples", type=int, default=40000,
                    help="on-line samples per step (default: inputs > the 126 MB L2)")
    ap.add_argument("--deform-images", type=int, default=60000)
    ap.add_argument("--residency", default="auto")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    if args.gpus > 1 and dist_env()[1] != args.gpus:
        sys.exit(f"--gpus {args.gpus} but WORLD_SIZE={dist_env()[1]}")
    line = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
