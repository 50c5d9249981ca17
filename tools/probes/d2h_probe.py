"""PCIe D2H bandwidth into pinned memory and its effect on a concurrent solve."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2007_06524_b200 as chk

N = 4 << 30
d = torch.empty(N // 8, dtype=torch.float64, device="cuda")
h = torch.empty(N // 8, dtype=torch.float64).pin_memory()
for chunk in (16 << 20, 256 << 20, 4 << 30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for o in range(0, N // 8, chunk // 8):
        h[o:o + chunk // 8].copy_(d[o:o + chunk // 8], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"D2H {chunk >> 20} MiB pieces: {N / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h.copy_(d, non_blocking=False) if False else None
d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"H2D: {N / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
# solve alone vs with a concurrent D2H stream
cfg = chk.LatticeConfig(d=3, L=32, n0=4, alpha="1/2", lam=0.01)
seeds = [chk.derive_seed(0, m) for m in range(256)]
A = chk.StiffnessBatch(cfg, chk.sample_cells_device(cfg, seeds))
F = chk.corrector_rhs_batched(A, 1)
opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
P = chk.make_preconditioner(3, cfg.n, opts)
U = torch.empty_like(F)
ws = chk.solver.Workspace()
for k in range(4):
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if k >= 2:
        with torch.cuda.stream(side):
            h.copy_(d, non_blocking=True)
    res = chk.pcg_solve_batched(A, F, opts, P, out=U, record_history=False, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"solve {'with 4 GiB D2H beside' if k >= 2 else 'alone'}: {e0.elapsed_time(e1):.1f} ms", flush=True)
