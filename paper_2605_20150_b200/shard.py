"""Block-id sharding of the table over the GPUs of one box.

Global block k is owned by rank ``k % G`` with local id ``k // G``; every rank
runs the whole working-set step on its shard with the replicated camera batch,
so no row data crosses ranks.  The only collectives are the per-batch
active-set exchange (C1: all-gather of each rank's ascending A = R n K global
ids, padded to the per-rank capacity) and the count reduction (C2: all-reduce
sum of an int64 count vector).  They run through ``torch.distributed`` (NCCL
over NVLink on the B200 box, gloo in the CPU tests): process groups are the
plumbing PyTorch supplies here.
"""
from __future__ import annotations

import numpy as np

PAD = -1


def owner(k: int, world_size: int) -> int:
    return int(k) % world_size


def local_id(k: int, world_size: int) -> int:
    return int(k) // world_size


def shard_blocks(K: int, world_size: int, rank: int) -> int:
    """Number of global blocks rank owns (K_loc)."""
    return (K - rank + world_size - 1) // world_size if K > rank else 0


def shard_capacity(C: int, world_size: int) -> int:
    """Per-rank resident capacity C_g = ceil(C / G)."""
    return -(-int(C) // world_size)


def exchange_active(active, cap: int, group=None, union=True):
    """C1: all-gather every rank's A list (global ids, ascending, <= cap
    entries).  `active` is a 1-D int32/int64 torch tensor (CUDA under NCCL, CPU
    under gloo).  Returns the [G, cap] gathered tensor (PAD-padded) and, if
    `union`, the sorted global active set as a 1-D tensor (that compaction
    needs its size on the host, i.e. a stream sync: the bench skips it so the
    host never waits for the device).  Nothing here synchronises otherwise."""
    import torch
    import torch.distributed as dist

    n = int(active.numel())
    if n > cap:
        raise ValueError(f"active list of {n} exceeds the per-rank capacity {cap}")
    G = dist.get_world_size(group)
    buf = torch.full((cap,), PAD, dtype=torch.int64, device=active.device)
    buf[:n] = active.to(torch.int64)
    out = torch.empty((G, cap), dtype=torch.int64, device=active.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:  # gloo (CPU tests, or a one-GPU functional run of the multi-rank bench)
        parts = [torch.empty_like(buf) for _ in range(G)]
        dist.all_gather(parts, buf, group=group)
        out = torch.stack(parts)
    if not union:
        return out, None
    flat = out.reshape(-1)
    return out, torch.sort(flat[flat != PAD]).values


def reduce_counts(counts, group=None):
    """C2: all-reduce (sum) of an int64 count vector, in place; returns it."""
    import torch.distributed as dist
    dist.all_reduce(counts, group=group)
    return counts


def global_from_local(local_ids: np.ndarray, world_size: int, rank: int) -> np.ndarray:
    return np.asarray(local_ids, np.int64) * world_size + rank
