"""Corrector right-hand sides on the device (homogenize.py:75-89 of the reference).

f_i = h^(d-1) * 1/2 (c[x+e_i] - c[x-e_i]) with c the nodal 2^d-cell average of
the cell field (lattice.py:326-345); callers of the PCG scale by h^(2-d)
(homogenize.py:110), i.e. the PCG load is h * 1/2 (c[x+e_i] - c[x-e_i]).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .lattice import Realization


def corrector_rhs_batched(batch, i: int, pcg_scaled: bool = True):
    """Device corrector loads for a ``StiffnessBatch``: (B, n^3) float64."""
    torch = _lib.require_cuda()
    d = 3
    if not (1 <= i <= d):
        raise ValueError(f"direction must be in 1..{d}, got {i}")
    n = batch.n
    h = 1.0 / n
    scale = h ** (d - 1) * (h ** (2 - d) if pcg_scaled else 1.0)
    f = torch.empty((batch.B, n ** 3), dtype=torch.float64, device=batch.beta.device)
    _lib.check(_lib.load().chk_corrector_rhs(ctypes.byref(batch.grid), ctypes.c_void_p(batch.beta.data_ptr()),
                                             ctypes.c_void_p(f.data_ptr()), batch.B, i, float(scale),
                                             _lib.stream_handle()))
    return f


def corrector_rhs(r: Realization, i: int) -> np.ndarray:
    """Drop-in for homogenize.py:75-89 (numpy out, computed on the GPU)."""
    from .operators import StiffnessBatch

    batch = StiffnessBatch(r.config, r.beta_cells.reshape(1, -1))
    return corrector_rhs_batched(batch, i, pcg_scaled=False).reshape(-1).cpu().numpy()
