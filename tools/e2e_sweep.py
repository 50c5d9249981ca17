"""Seeds-to-host-solutions e2e of config 3 for several chunk sizes / lane counts
(CUDA events around pcg_solve_seeds, 3 timed runs after 2 warm-ups)."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch

    import paper_2007_06524_b200 as chk

    chunk = int(sys.argv[2])
    cfg = chk.LatticeConfig(d=3, L=32, n0=4, alpha="1/2", lam=0.01)
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    P = chk.make_preconditioner(3, cfg.n, opts)
    U = torch.empty((256, cfg.n ** 3), dtype=torch.float64).pin_memory()
    ws = chk.solver.Workspace()
    ms = []
    for k in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        seeds = [chk.derive_seed(0, m) for m in range(256)]
        res = chk.pcg_solve_seeds(cfg, seeds, opts, P, out=U, record_history=False, workspace=ws, chunk=chunk)
        e1.record()
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(e0.elapsed_time(e1))
    dof = float(np.sum(res.iterations)) * cfg.n ** 3
    print(f"lanes {os.environ.get('CHK_HOST_LANES', '3')} chunk {chunk}: {np.mean(ms):.1f} ms  {dof / np.mean(ms) * 1e3:.3e} DOF-it/s", flush=True)
else:
    for lanes in sys.argv[1].split(","):
        for chunk in sys.argv[2].split(","):
            subprocess.run([sys.executable, __file__, "child", chunk], env={**os.environ, "CHK_HOST_LANES": lanes})
