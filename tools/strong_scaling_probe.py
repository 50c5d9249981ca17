"""Per-GPU throughput of config 3 at the per-GPU batch sizes of strong scaling
(256/N realizations for N = 1, 2, 4, 8): what each rank of `bench.py --gpus N`
solves.  Realization sharding has no collective, so N-GPU throughput =
N x the B = 256/N line (max-over-ranks time: the slowest shard decides).

    python tools/strong_scaling_probe.py [--steps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2007_06524_b200 as chk
from paper_2007_06524_b200.sharding import shard_range

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
cfg = chk.LatticeConfig(d=3, L=32, n0=4, alpha="1/2", lam=0.01)
opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
P = chk.make_preconditioner(3, cfg.n, opts)
nb = cfg.n ** 3
out = {}
for N in (1, 2, 4, 8):
    worst = 0.0
    dof_all = 0.0
    for rank in range(N):  # every shard of an N-GPU run, one after the other on this GPU
        lo, hi = shard_range(256, rank, N)
        seeds = [chk.derive_seed(0, m) for m in range(lo, hi)]
        A = chk.StiffnessBatch(cfg, chk.sample_cells_device(cfg, seeds))
        F = chk.corrector_rhs_batched(A, 1)
        U = torch.empty_like(F)
        ws = chk.solver.Workspace()
        chk.pcg_solve_batched(A, F, opts, P, out=U, record_history=False, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            res = chk.pcg_solve_batched(A, F, opts, P, out=U, record_history=False, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        worst = max(worst, ms)
        dof_all += float(np.sum(res.iterations)) * nb
        del A, F, U, ws
        torch.cuda.empty_cache()
    out[N] = {"per_gpu_batch": 256 // N, "max_shard_ms": round(worst, 2),
              "projected_value": dof_all / (worst / 1e3)}
    print(json.dumps({N: out[N]}), flush=True)
base = out[1]["projected_value"]
for N in (2, 4, 8):
    print(f"N={N}: projected strong-scaling efficiency {out[N]['projected_value'] / (N * base):.3f}")
