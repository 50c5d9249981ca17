"""Run batched solves of a BASELINE config (used under ncu / compute-sanitizer).

    python tools/run_solve.py --config 3 --batch 32 --solves 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2007_06524_b200 as chk

CFG = {1: (8, 4, 0.1, 1e-8), 2: (16, 4, 0.1, 1e-8), 3: (32, 4, 0.01, 1e-8), 4: (64, 4, 0.1, 1e-10),
       5: (32, 16, 0.1, 1e-8)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--kind", default="lkr")
a = ap.parse_args()
L, n0, lam, tol = CFG[a.config]
cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha="1/2", lam=lam)
beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(a.batch)])
A = chk.StiffnessBatch(cfg, beta)
F = chk.corrector_rhs_batched(A, 1)
opts = chk.SolveOptions(tol=tol, preconditioner=a.kind)
for _ in range(a.solves):
    res = chk.pcg_solve_batched(A, F, opts)
torch.cuda.synchronize()
print("iterations", res.iterations.tolist()[:8], "status", set(res.status.tolist()), "launches", res.launches)
