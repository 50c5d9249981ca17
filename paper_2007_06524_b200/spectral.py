"""Fourier setup (host) and the exact Fourier preconditioner apply (device).

Setup mirrors spectral.py:56-95 of the reference.  The apply runs the same
sm_100a FFT pipeline as the LKR preconditioner with the diagonal
1/(lam_i+lam_j+lam_k) (or +delta) evaluated on the fly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class EigenSpectrum:
    """spectral.py:17-22."""

    n: int
    values: np.ndarray


def fourier_eigenvalues(n: int) -> EigenSpectrum:
    """spectral.py:56-68: Re FFT of (2,-1,0,...,-1), negatives clipped."""
    if n < 3:
        raise ValueError(f"need n >= 3, got {n}")
    p = np.zeros(n)
    p[0] = 2.0
    p[1] = -1.0
    p[-1] = -1.0
    lam = np.fft.fft(p)
    assert np.max(np.abs(lam.imag)) <= 1e-12
    values = lam.real.copy()
    values[values < 0.0] = 0.0
    return EigenSpectrum(n=n, values=values)


def apply_fourier_preconditioner(n: int, x, delta: float = 0.0):
    """y = F* diag(g+) F x (spectral.py:98-112), g+ = pseudo-inverse of the
    eigensum (delta = 0) or 1/(g + delta) (regularized, spectral.py:90-95)."""
    from .lowrank import _device_apply, _plan_for

    kind = "regularized" if delta > 0.0 else "fourier"
    return _device_apply(_plan_for(3, n, kind, 0.0, float(delta)), x)
