"""Time chk_stencil_apply (y = A x, + <x, y>) on a config-sized batch (microbenchmark)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2007_06524_b200 as chk

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=32)
ap.add_argument("--n0", type=int, default=4)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
cfg = chk.LatticeConfig(d=3, L=a.L, n0=a.n0, alpha="1/2", lam=0.01)
beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(a.batch)])
A = chk.StiffnessBatch(cfg, beta)
x = torch.randn(a.batch, cfg.n ** 3, dtype=torch.float64, device="cuda")
for _ in range(3):
    y, xy = A.matvec(x, with_dot=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    y, xy = A.matvec(x, with_dot=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nbytes = 16.0 * a.batch * cfg.n ** 3
print(f"stencil n={cfg.n} B={a.batch}: {ms:.3f} ms/apply, {nbytes / ms / 1e6:.0f} GB/s (read x + write y)")
