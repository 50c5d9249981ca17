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


@dataclass(frozen=True)
class EigensumTensor:
    """spectral.py:26-44: eigenvalue sums lam_i + lam_j (+ lam_k), exact rank-d form."""

    d: int
    n: int
    spectrum: EigenSpectrum

    def value(self, idx) -> float:
        return float(sum(self.spectrum.values[i] for i in idx))

    def array(self) -> np.ndarray:
        lam = self.spectrum.values
        out = lam
        for _ in range(self.d - 1):
            out = out[..., None] + lam
        return out


@dataclass(frozen=True)
class PseudoInverseDiag:
    """spectral.py:47-53.  ``values`` (n,)*d is materialised lazily on the host
    only when read (the device apply evaluates 1/(g + delta) per spectral tile
    from the eigenvalues); ``delta`` = 0 is the pseudo-inverse."""

    d: int
    n: int
    values: np.ndarray = None
    delta: float = 0.0
    spectrum: EigenSpectrum = None

    def __post_init__(self):
        if self.values is None:
            g = EigensumTensor(self.d, self.n, self.spectrum or fourier_eigenvalues(self.n)).array()
            if self.delta > 0.0:
                out = 1.0 / (g + self.delta)
            else:
                out = np.zeros_like(g)
                mask = g > 0.0
                out[mask] = 1.0 / g[mask]
            object.__setattr__(self, "values", out)

    def value(self, idx) -> float:
        return float(self.values[tuple(idx)])


def eigensum_tensor(d: int, spectrum: EigenSpectrum) -> EigensumTensor:
    """spectral.py:71-74."""
    if d not in (2, 3):
        raise ValueError(f"dimension must be 2 or 3, got {d}")
    return EigensumTensor(d=d, n=spectrum.n, spectrum=spectrum)


def pseudoinverse_diag(g: EigensumTensor) -> PseudoInverseDiag:
    """spectral.py:77-87: reciprocal with the origin zeroed."""
    return PseudoInverseDiag(d=g.d, n=g.n, delta=0.0, spectrum=g.spectrum)


def regularized_inverse_diag(g: EigensumTensor, delta: float) -> PseudoInverseDiag:
    """spectral.py:90-95: 1/(g + delta); delta <= 0 falls back to the pseudo-inverse."""
    if delta <= 0.0:
        return pseudoinverse_diag(g)
    return PseudoInverseDiag(d=g.d, n=g.n, delta=float(delta), spectrum=g.spectrum)


def _diag_kind(g_plus) -> tuple:
    """(kind, delta) of a diagonal the device plans can evaluate on the fly.
    Diagonals built by pseudoinverse_diag / regularized_inverse_diag (this
    package's or the reference's) are recognised by value; anything else is
    not an eigensum reciprocal and is rejected (ValueError)."""
    if isinstance(g_plus, PseudoInverseDiag) and g_plus.spectrum is not None:
        sp = g_plus.spectrum.values
        if np.array_equal(sp, fourier_eigenvalues(g_plus.n).values):
            return ("regularized", g_plus.delta) if g_plus.delta > 0.0 else ("fourier", 0.0)
    vals = np.asarray(g_plus.values)
    n, d = int(g_plus.n), int(g_plus.d)
    if d != 3:
        raise ValueError("the GPU path implements d = 3 only")
    v0 = float(vals.flat[0])
    delta = 0.0 if v0 == 0.0 else 1.0 / v0
    ref = PseudoInverseDiag(d=d, n=n, delta=delta).values
    if vals.shape != ref.shape or not np.allclose(vals, ref, rtol=1e-13, atol=0.0):
        raise ValueError("only eigensum reciprocals (pseudoinverse_diag / regularized_inverse_diag) "
                         "have a device plan")
    return ("regularized", delta) if delta > 0.0 else ("fourier", 0.0)


def apply_fourier_preconditioner(g_plus, x, delta: float = 0.0):
    """y = F* diag(g+) F x (spectral.py:98-112) on the GPU.

    ``g_plus`` is a PseudoInverseDiag (reference signature); the legacy form
    ``apply_fourier_preconditioner(n, x, delta=...)`` is still accepted."""
    from .lowrank import _device_apply, _plan_for

    if isinstance(g_plus, (int, np.integer)):
        n = int(g_plus)
        kind = "regularized" if delta > 0.0 else "fourier"
    else:
        n = int(g_plus.n)
        kind, delta = _diag_kind(g_plus)
    size = n ** 3
    shape = tuple(getattr(x, "shape", np.shape(x)))
    if shape != (size,) and not (len(shape) == 2 and shape[1] == size):
        raise ValueError(f"expected vector of length {size}, got shape {shape}")
    return _device_apply(_plan_for(3, n, kind, 0.0, float(delta)), x)
