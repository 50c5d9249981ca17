"""Per-kernel timing of the standalone preconditioner apply (fwd APPLY, mid APPLY,
inv APPLY) on a batch: isolates the transform passes from the PCG state."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2007_06524_b200 as chk
from paper_2007_06524_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = a.n
t = chk.dc_correction(chk.canonical_reciprocal(chk.fourier_eigenvalues(n), 3, 1e-8))
x = torch.randn(a.batch, n ** 3, dtype=torch.float64, device="cuda")
lib = _lib.load()
for _ in range(2):
    chk.apply_lkr_preconditioner(t, x)
torch.cuda.synchronize()
lib.chk_profile_enable(1)
for _ in range(a.reps):
    chk.apply_lkr_preconditioner(t, x)
torch.cuda.synchronize()
ms = np.zeros(5)
cnt = np.zeros(5, dtype=np.int64)
lib.chk_profile_read(ms.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p))
lib.chk_profile_enable(0)
spec = 8.0 * (n // 2 + 1) / (n // 2)
dof = a.batch * n ** 3
for i, (name, bpd) in enumerate([("fwd_apply", 8 + spec), ("mid_apply", 2 * spec), ("inv_apply", spec + 8)]):
    avg = ms[i + 1] / max(1, cnt[i + 1])
    print(f"n={n} B={a.batch} {name}: {avg:.3f} ms  {bpd * dof / (avg * 1e-3) / 1e9:7.0f} GB/s  (flags={os.environ.get('CHK_DEBUG_FLAGS', '0')})")
