"""Multi-GPU plumbing: request sharding and end-of-run gathers.

Requests are independent units (engine.py:263-272: a request's output depends
only on its prompt, the model and (k, s)), so N GPUs serve N disjoint shards
with NO collective on the decode hot path.  torch.distributed
(NCCL on the B200 box, gloo in the CPU tests) is used only after the timed
region: token counts summed, device times max-reduced, optional per-request
outputs gathered to rank 0.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_total: int, rank: int, world: int) -> tuple:
    """Contiguous block of request ids for ``rank`` (sizes differ by at most 1)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_ids(n_total: int, rank: int, world: int) -> list:
    lo, hi = shard_bounds(n_total, rank, world)
    return list(range(lo, hi))


def gather_throughput(tokens: float, seconds: float, device=None) -> tuple:
    """(sum of tokens, max of seconds) over ranks; identity without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(tokens), float(seconds)
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    t = torch.tensor([tokens], dtype=torch.float64, device=dev)
    s = torch.tensor([seconds], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(s, op=dist.ReduceOp.MAX)
    return float(t.item()), float(s.item())


def gather_outputs(outputs: dict) -> dict | None:
    """Merge per-rank {request_id: tokens} dicts on rank 0 (None elsewhere)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(outputs)
    parts = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(outputs, parts, dst=0)
    if dist.get_rank() != 0:
        return None
    merged: dict = {}
    for p in parts:
        overlap = set(merged) & set(p)
        if overlap:
            raise RuntimeError(f"request ids served by two ranks: {sorted(overlap)[:5]}")
        merged.update(p)
    return merged
