"""Instance sharding across GPUs (one process per GPU, torch.distributed plumbing).

The unit of parallelism is the disorder instance / independent chain: rank g
owns the contiguous block of GLOBAL instance ids [offset, offset + count).  Every RNG stream
is keyed by the global id, so a sharded run is bit-identical to a single-GPU
run of the same instances.  There is no data-path collective: replicas of one instance never
span GPUs.  The only collectives are the end-of-run observable reductions here (NCCL over
NVLink on the B200 box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard(total: int, world: int, rank: int):
    """(offset, count) of rank's contiguous block of global instance ids."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(int(total), int(world))
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def _dist():
    import torch.distributed as dist
    return dist


def reduce_sum(array, device=None, group=None):
    """Sum an integer/float numpy array (or torch tensor) over all ranks; returns numpy."""
    import torch
    dist = _dist()
    t = array if isinstance(array, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(array))
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def reduce_max(value: float, device=None, group=None) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_instances(local, total: int, device=None, group=None):
    """All-gather per-instance rows (first axis = local instances) into the global order."""
    import torch
    dist = _dist()
    local = np.ascontiguousarray(local)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    rows = [shard(total, world, r)[1] for r in range(world)]
    width = int(np.prod(local.shape[1:])) if local.ndim > 1 else 1
    buf = torch.zeros((max(rows), width), dtype=torch.float64, device=device)
    buf[: local.shape[0]] = torch.from_numpy(local.reshape(local.shape[0], width).astype(np.float64)).to(buf.device)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    full = np.concatenate([o.cpu().numpy()[:rows[r]] for r, o in enumerate(out)], axis=0)
    return full.reshape((total,) + local.shape[1:]).astype(local.dtype)


def reduce_observables(ens_obs, hist=None, device=None, group=None):
    """Per-slot observables summed over local instances then over ranks.
    ens_obs: [I][R][5] (count, sum E, sum E^2, sum |M|, sum M^2); hist: [R][nbins]."""
    per_slot = np.asarray(ens_obs, np.int64).sum(axis=0)
    out = {"obs": reduce_sum(per_slot, device, group)}
    if hist is not None:
        out["hist"] = reduce_sum(np.asarray(hist, np.int64), device, group)
    return out
