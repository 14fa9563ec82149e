"""Multi-GPU plumbing for the sharded parts of the path.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  What
shards and how:
  * deformation -- rank r deforms images [r*n/G, (r+1)*n/G); every image
    re-derives its own substream (seed, 2, epoch, index) on the device, so
    the union is byte-identical to G = 1 and needs no collective;
    `gather_deformed` assembles the epoch on every rank when a trainer
    wants it (one all_gather);
  * evaluation -- rank r evaluates its shard, then ONE all_reduce(sum) of the
    int64[102] count vector {wrong, confusion[10][10], second_guess}
    (eval_report.py:36-67);
  * weights -- `broadcast_layers` sends the trainer rank's device weights to
    the evaluation ranks (dmlp_net_get_layer straight into device tensors).
On-line training itself does not shard (SPEC: sample s+1 needs the weights
after sample s); multi-GPU training runs independent replicas.
"""

from __future__ import annotations

import ctypes

import numpy as np

N_COUNTS = 102


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, disjoint, covering split of [0, n)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return n * rank // world, n * (rank + 1) // world


def _dist():
    import torch.distributed as dist

    return dist


def world_info(group=None) -> tuple[int, int]:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def allreduce_counts(counts, group=None):
    """Sum the count vector over ranks in place (NCCL on GPU, gloo on CPU)."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def deform_sharded(raw, labels, params, seed: int, epoch: int, group=None):
    """Deform this rank's shard of a split resident on the device.

    raw (n,28,28) u8 and labels (n,) u8 are the FULL split on every rank;
    returns (shard (hi-lo, 841) f32, lo, hi)."""
    from .deform import deform_device

    rank, world = world_info(group)
    lo, hi = shard_range(int(raw.shape[0]), rank, world)
    out = deform_device(raw[lo:hi], labels[lo:hi], params, seed, epoch, first=lo)
    return out, lo, hi


def gather_deformed(shard, n: int, group=None):
    """All-gather the deformed shards into the full (n, 841) epoch."""
    import torch

    rank, world = world_info(group)
    if world == 1:
        return shard
    sizes = [shard_range(n, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((width, shard.shape[1]), dtype=shard.dtype, device=shard.device)
    pad[: shard.shape[0]] = shard
    parts = [torch.empty_like(pad) for _ in range(world)]
    _dist().all_gather(parts, pad, group=group)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)])


def eval_counts_sharded(dev_net, x, labels, group=None):
    """Evaluate this rank's shard of (x, labels) (full split on every rank)
    and all-reduce the counts: returns the global int64[102] counts."""
    rank, world = world_info(group)
    lo, hi = shard_range(int(x.shape[0]), rank, world)
    counts = dev_net.eval_counts(x[lo:hi].contiguous(), labels[lo:hi].contiguous())
    return allreduce_counts(counts, group)


def _backend(group=None) -> str:
    return str(_dist().get_backend(group)).lower()


def _global(rank: int, group=None) -> int:
    """Group rank -> global rank (torch.distributed src/dst arguments)."""
    return rank if group is None else _dist().get_global_rank(group, rank)


def broadcast_layers(dev_net, src: int = 0, group=None) -> None:
    """Broadcast the device weights of `dev_net` on rank `src` to every rank's
    dev_net (layer by layer, device to device).

    dmlp_net_get_layer / dmlp_net_set_layer run on the net's own stream while
    torch allocates and broadcasts on its current stream, so the current
    stream is drained before the library writes a freshly allocated tensor
    and before it reads a received one."""
    import torch

    from . import _lib

    rank, world = world_info(group)
    if world == 1:
        return
    cur = torch.cuda.current_stream(dev_net.device)
    for li, (fo, fi1) in enumerate(dev_net.shapes):
        t = torch.empty((fo, fi1), dtype=torch.float32, device=f"cuda:{dev_net.device}")
        if rank == src:
            cur.synchronize()  # t's block may still be in use by queued torch work
            _lib.check(_lib.lib().dmlp_net_get_layer(dev_net._h, li, ctypes.c_void_p(t.data_ptr()),
                                                     t.numel()), "dmlp_net_get_layer")
        _dist().broadcast(t, src=_global(src, group), group=group)
        if rank != src:
            cur.synchronize()  # the broadcast landed before the library reads t
            _lib.check(_lib.lib().dmlp_net_set_layer(dev_net._h, li, ctypes.c_void_p(t.data_ptr()),
                                                     t.numel()), "dmlp_net_set_layer")


def peer_shard(n: int, rank: int, world: int, lead: int = 0) -> tuple[int, int]:
    """The images rank `rank` deforms when every rank except `lead` (the
    trainer) deforms: the non-lead ranks split [0, n) in rank order."""
    if world == 1:
        return 0, n
    if rank == lead:
        return 0, 0
    k = rank - (rank > lead)
    return shard_range(n, k, world - 1)


def deform_to_lead(raw, labels, params, seed: int, epoch: int, out, lead: int = 0, group=None):
    """Peer-GPU deformation of one epoch: every rank
    except `lead` deforms its peer_shard of the split (resident on every rank)
    and sends it to the lead, which receives into `out` (n, 841).

    Collective over `group`.  NCCL: point-to-point over NVLink; the lead's
    receives are queued behind its current stream (the training launch), so
    the peers deform while the lead trains and the transfer follows the
    training kernel.  gloo (tests): staged through host memory.  Returns the
    list of requests the lead must wait on (empty elsewhere)."""
    import torch

    from .deform import deform_device

    dist = _dist()
    rank, world = world_info(group)
    n = int(raw.shape[0])
    if world == 1:
        deform_device(raw, labels, params, seed, epoch, out=out)
        return []
    gloo = _backend(group) == "gloo"
    if rank != lead:
        lo, hi = peer_shard(n, rank, world, lead)
        if hi <= lo:
            return []
        shard = deform_device(raw[lo:hi], labels[lo:hi], params, seed, epoch, first=lo)
        if gloo:
            dist.send(shard.cpu(), dst=_global(lead, group), group=group)
            return []
        reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, shard, _global(lead, group),
                                                  group)])
        for r in reqs:
            r.wait()
        torch.cuda.current_stream(shard.device).synchronize()  # shard stays alive until sent
        return []
    ops, staged = [], []
    for r in range(world):
        lo, hi = peer_shard(n, r, world, lead)
        if r == lead or hi <= lo:
            continue
        if gloo:
            host = torch.empty((hi - lo, out.shape[1]), dtype=out.dtype)
            dist.recv(host, src=_global(r, group), group=group)
            staged.append((lo, hi, host))
        else:
            ops.append(dist.P2POp(dist.irecv, out[lo:hi], _global(r, group), group))
    for lo, hi, host in staged:
        out[lo:hi].copy_(host)
    return dist.batch_isend_irecv(ops) if ops else []


def counts_to_report(counts) -> dict:
    c = np.asarray(counts.cpu() if hasattr(counts, "cpu") else counts, dtype=np.int64)
    return {"wrong": int(c[0]), "confusion": c[1:101].reshape(10, 10),
            "second_guess_correct": int(c[101])}
