"""Host-side data-parallel sharding of the rollout-to-loss path.

Trajectories/envs are independent units: rank p of P owns the contiguous env block
[p*E/P, (p+1)*E/P). All per-step and per-token work is rank-local; the only exchanges are
the tiny collectives inside the C ABI (C1 advantage-stat allreduce, C2 GRPO returns
allgather, C3 loss-stat allreduce). Nothing here touches GPU memory.
"""
from __future__ import annotations

import numpy as np


def env_range(n_env_global: int, nranks: int, rank: int) -> tuple[int, int]:
    if n_env_global % nranks:
        raise ValueError(f"{n_env_global} envs do not shard evenly over {nranks} ranks")
    e = n_env_global // nranks
    return rank * e, (rank + 1) * e


def owner_of(env_global: np.ndarray, n_env_global: int, nranks: int) -> np.ndarray:
    return np.asarray(env_global) // (n_env_global // nranks)


def route_records(env_global: np.ndarray, n_env_global: int, nranks: int, rank: int):
    """Indices (in arrival order) of the records rank `rank` owns and their local env ids.
    Out-of-range env ids stay with rank 0 so they are counted exactly once (as OOB)."""
    env_global = np.asarray(env_global)
    lo, hi = env_range(n_env_global, nranks, rank)
    inr = (env_global >= 0) & (env_global < n_env_global)
    mine = inr & (env_global >= lo) & (env_global < hi)
    if rank == 0:
        mine = mine | ~inr
    idx = np.nonzero(mine)[0]
    local = np.where(inr[idx], env_global[idx] - lo, env_global[idx])
    return idx, local.astype(np.int32)


def interleaved_groups(n_env_global: int, group_size: int) -> np.ndarray:
    """Group id g(e) = e mod (E/G): with P = G ranks every group has one member per rank
    (BASELINE.json config 5, 'GRPO groups spanning ranks')."""
    return (np.arange(n_env_global) % (n_env_global // group_size)).astype(np.int32)


def contiguous_groups(n_env_global: int, group_size: int) -> np.ndarray:
    return (np.arange(n_env_global) // group_size).astype(np.int32)
