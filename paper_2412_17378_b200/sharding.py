"""Multi-GPU view sharding: camera views are independent units,
so N GPUs split a batch of views with no data-path collective.  The scene is
replicated (uploaded once per GPU); the only collectives are the timing
barrier and the max-over-ranks of the timed region.
"""
from __future__ import annotations

import math

import numpy as np

N_VIEWS = 64
PIVOT_Z = 5.5


def views_for_rank(rank: int, world: int, steps: int, n_views: int = N_VIEWS) -> list[int]:
    """View indices rank `rank` renders over `steps` steps (one view per step,
    round-robin over the orbit: step i renders view (rank + world*i) % n)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return [(rank + world * i) % n_views for i in range(steps)]


def contiguous_shard(n_views: int, rank: int, world: int) -> range:
    """Contiguous split of a view batch (64/N per GPU for N in 1,2,4,8)."""
    base, extra = divmod(n_views, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def batch_view_ids(rank: int, world: int, steps: int, batch: int = N_VIEWS) -> list[int]:
    """View ids rank `rank` renders over `steps` steps of the §8(e) batch
    schedule: every step is the same fixed batch of `batch` views
    (0..batch-1 of the orbit), split contiguously over the ranks
    (contiguous_shard) — the total work per step is fixed (strong scaling)."""
    mine = list(contiguous_shard(batch, rank, world))
    return mine * steps


def orbit_view(k: int, n_views: int = N_VIEWS, pivot_z: float = PIVOT_Z) -> np.ndarray:
    """World->camera 4x4 of view k: yaw -15..+15 deg about the y axis through
    (0, 0, pivot_z); the rotation block is orthonormal (src/scene.cpp:45-47)."""
    yaw = math.radians(-15.0 + 30.0 * k / max(1, n_views - 1))
    c, s = math.cos(yaw), math.sin(yaw)
    R = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
    piv = np.array([0.0, 0.0, pivot_z])
    V = np.eye(4)
    V[:3, :3] = R
    V[:3, 3] = piv - R @ piv
    return V.astype(np.float32)


def max_over_ranks(value_ms: float, dist=None, device=None) -> float:
    """Max of a per-rank timing over the process group (timing collective only)."""
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value_ms)
    import torch

    t = torch.tensor([float(value_ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
