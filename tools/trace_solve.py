"""Per-launch timeline of one batched solve (library CUDA events per launch).

    CHK_PROF_TRACE=gpurun_out/trace.txt python tools/trace_solve.py --config 3 --batch 256

Prints the iteration histogram and the launch sequence grouped by kernel class
(1 fwd, 2 mid, 3 inv, 4 paired plane pass) -- where the time of a step goes
(steady-state iterations vs. initialisation and the convergence tail).
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2007_06524_b200 as chk
from paper_2007_06524_b200 import _lib

CFG = {1: (8, 4, 0.1, 1e-8), 2: (16, 4, 0.1, 1e-8), 3: (32, 4, 0.01, 1e-8), 4: (64, 4, 0.1, 1e-10),
       5: (32, 16, 0.1, 1e-8)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=256)
a = ap.parse_args()
L, n0, lam, tol = CFG[a.config]
cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha="1/2", lam=lam)
beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(a.batch)])
A = chk.StiffnessBatch(cfg, beta)
F = chk.corrector_rhs_batched(A, 1)
opts = chk.SolveOptions(tol=tol, preconditioner="lkr", eps_rank=1e-8)
P = chk.make_preconditioner(3, cfg.n, opts)
ws = chk.solver.Workspace()
res = chk.pcg_solve_batched(A, F, opts, P, workspace=ws)
lib = _lib.load()
trace = os.environ.get("CHK_PROF_TRACE")
assert trace, "set CHK_PROF_TRACE"
off = os.path.getsize(trace) if os.path.exists(trace) else 0
lib.chk_profile_enable(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = chk.pcg_solve_batched(A, F, opts, P, workspace=ws)
e1.record()
torch.cuda.synchronize()
lib.chk_profile_enable(0)
its = np.asarray(res.iterations)
print("solve ms %.2f  iterations min/mean/max %d %.2f %d" % (e0.elapsed_time(e1), its.min(), its.mean(), its.max()))
hist = np.bincount(its)
print("active realizations per iteration:", [int((its >= k).sum()) for k in range(1, its.max() + 1)])
with open(trace) as fh:
    fh.seek(off)
    rows = [l.split() for l in fh if l.strip()]
seq = [(int(k), float(t)) for k, t in rows]
tot = {}
for k, t in seq:
    tot[k] = tot.get(k, 0.0) + t
print("class totals ms:", {k: round(v, 2) for k, v in sorted(tot.items())}, "sum %.2f" % sum(tot.values()))
print("launch sequence (class:ms):")
print(" ".join("%d:%.2f" % (k, t) for k, t in seq))
