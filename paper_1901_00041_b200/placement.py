"""Tenant-sharded placement across the GPUs of one box.

Tenants are independent (distinct weights, no shared state: PAPER.md:77,
SPEC.md:396-397), so a tenant is pinned to one GPU at registration and the
hot path needs no collective.  Placement is a deterministic
longest-processing-time bin packing by per-tenant FLOP demand, then weight
bytes, ties broken by tenant index; for a homogeneous tenant set it reduces
to ``tenant mod G``.  Latency samples are merged off the hot path with one
all-gather and the reference's nearest-rank percentile.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def place_tenants(demands: Sequence[Tuple[int, int]], n_gpus: int) -> List[int]:
    """demands[i] = (flops per pass, weight bytes) of tenant i -> GPU of tenant i."""
    if n_gpus < 1:
        raise ValueError("n_gpus must be >= 1")
    order = sorted(range(len(demands)), key=lambda i: (-demands[i][0], -demands[i][1], i))
    load = [(0, 0)] * n_gpus
    out = [0] * len(demands)
    for i in order:
        g = min(range(n_gpus), key=lambda j: (load[j], j))
        out[i] = g
        load[g] = (load[g][0] + demands[i][0], load[g][1] + demands[i][1])
    return out


def least_loaded(loads: Sequence[Tuple[int, int]], exclude: Sequence[int] = ()) -> int:
    """The GPU an evicted tenant is re-admitted on: least (FLOPs, weight
    bytes) load, ties to the lowest index, never one in ``exclude`` (the GPU
    it was evicted from)."""
    cand = [g for g in range(len(loads)) if g not in set(exclude)]
    if not cand:
        raise ValueError("no GPU to re-admit on")
    return min(cand, key=lambda g: (loads[g], g))


def tenants_of(rank: int, placement: Sequence[int]) -> List[int]:
    return [t for t, g in enumerate(placement) if g == rank]


def merged_percentile(local_samples: Sequence[float], pct: float, group=None) -> float:
    """Nearest-rank percentile over every rank's samples (one all_gather_object,
    off the hot path); single-process callers pass no group."""
    from .scheduler import percentile_nearest_rank
    samples = list(local_samples)
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            gathered: list = [None] * dist.get_world_size(group)
            dist.all_gather_object(gathered, samples, group=group)
            samples = [x for part in gathered for x in part]
    except ImportError:
        pass
    return percentile_nearest_rank(samples, pct)
