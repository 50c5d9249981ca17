"""Realization sharding across GPUs (one process per GPU, torch.distributed).

Realizations are independent, so the batch is split into
contiguous global-index blocks, one per rank, with seeds derived from the
global index (lattice.py:273-276) -- results do not depend on the GPU count.
There is no collective on the data path; the only communication is the final
gather of the tiny per-realization reports, in index order (the fixed-order
reduction of homogenize.py:173-179).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple:
    """Contiguous block [lo, hi) of realization indices owned by ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


@dataclass(frozen=True)
class ShardRecord:
    index: int
    iterations: int
    final_residual: float
    status: int
    norm_u: float


def gather_records(local: list, world: int) -> list:
    """All-gather per-realization records (any backend: gloo on CPU, nccl on GPU)."""
    import torch.distributed as dist

    if world == 1:
        return sorted(local, key=lambda r: r.index)
    out = [None] * world
    dist.all_gather_object(out, local)
    merged = [rec for part in out for rec in part]
    merged.sort(key=lambda r: r.index)
    return merged


def solve_shard(config, total: int, master_seed: int, opts, rank: int, world: int,
                solve_fn=None) -> list:
    """Solve this rank's realizations; returns its ShardRecords.

    ``solve_fn(config, seeds, opts) -> (iterations, final_residual, status, norm_u)``
    defaults to the GPU batcher; tests inject a CPU stand-in to exercise the
    multi-process host logic without a device."""
    from .lattice import derive_seed

    lo, hi = shard_range(total, rank, world)
    seeds = [derive_seed(master_seed, m) for m in range(lo, hi)]
    if not seeds:
        return []
    if solve_fn is None:
        solve_fn = _gpu_solve
    its, fin, st, nu = solve_fn(config, seeds, opts)
    return [ShardRecord(lo + j, int(its[j]), float(fin[j]), int(st[j]), float(nu[j]))
            for j in range(len(seeds))]


def _gpu_solve(config, seeds, opts):
    import torch

    from .homogenize import corrector_rhs_batched
    from .lattice import sample_realization
    from .operators import StiffnessBatch
    from .solver import pcg_solve_batched

    beta = np.stack([sample_realization(config, s).beta_cells.ravel() for s in seeds])
    A = StiffnessBatch(config, beta)
    F = corrector_rhs_batched(A, 1)
    res = pcg_solve_batched(A, F, opts, record_history=False)
    nu = torch.linalg.norm(res.u, dim=1).cpu().numpy()
    return res.iterations, res.final_residual, res.status, nu
