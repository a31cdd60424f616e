"""Multi-GPU host plumbing (one process per GPU, torch.distributed for bootstrap only).

The data path's only exchange is inside the library: NCCL all-reduces of int64 histograms,
per-segment row counts and sampling statistics ("summed across all GPUs using
AllReduce").  This module holds the host logic around it: the row sharding and the
NCCL unique-id broadcast.  No arithmetic of the method lives here.
"""
from __future__ import annotations


def shard_rows(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous global rows [row0, row0 + n) owned by `rank`: the first
    n_global % world ranks get one extra row."""
    if world < 1 or not (0 <= rank < world) or n_global < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_global, world)
    n = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, n


def bootstrap_nccl_id(rank: int, make_id, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL id with `make_id()` (oocgb_nccl_unique_id) and every rank
    receives it through torch.distributed (any backend, e.g. gloo)."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    nid = obj[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("NCCL unique id must be 128 bytes")
    return bytes(nid)


def context_for_rank(make_context, rank: int, world: int, local_rank: int, stream: int = 0):
    """Create this rank's oocgb Context (world > 1: NCCL communicator from a broadcast id)."""
    import paper_2005_09148_b200 as ob
    nid = bootstrap_nccl_id(rank, ob.nccl_unique_id) if world > 1 else None
    return make_context(local_rank, rank, world, nid, stream)


def gloo_collective(group=None):
    """Host transport for Context(host_collective=...): op 0 sum, 1 max, 2 all-gather (the
    caller's buffer is zero outside its own block, so a sum gathers), through torch.distributed
    on CPU tensors (gloo).  Values are widened to int64 for the reduction (uint64 maxima here are
    bit patterns of non-negative doubles, < 2^63)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def fn(op, arr):
        t = torch.from_numpy(arr.astype(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM, group=group)
        arr[...] = t.numpy().astype(arr.dtype)

    return fn
