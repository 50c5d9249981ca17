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


# ----------------------------------------------------------------------------
# homogenized matrices and ensembles (homogenize.py:92-182), batched on the GPU
# ----------------------------------------------------------------------------
from dataclasses import dataclass  # noqa: E402


@dataclass(frozen=True)
class HomogenizedMatrix:
    """homogenize.py:38-52."""

    matrix: np.ndarray  # (d, d)
    seed: int
    L: int
    lam: float
    iterations: tuple   # PCG iterations per direction
    num_covered: int

    @property
    def d(self) -> int:
        return self.matrix.shape[0]


@dataclass(frozen=True)
class EnsembleStats:
    """homogenize.py:55-66."""

    d: int
    L: int
    M: int
    lam: float
    average: np.ndarray
    std: np.ndarray
    records: tuple
    failed_seeds: tuple = ()


def homogenized_matrix_batched(realizations, opts=None, precond=None, skip_failed=False):
    """The d = 3 corrector problems of every realization in ONE batched solve
    (B = 3 M systems sharing their cell arrays per realization) and the averaged
    matrices (homogenize.py:92-124):

        abar_ii = lambda + h^3 sum c - <f_i, u_i>,   abar_ij = -<f_j, u_i>.

    All loads, solves and inner products stay on the device.  Returns one
    HomogenizedMatrix per realization (None for a failed one when
    ``skip_failed``; otherwise SolverDidNotConverge is raised as in
    homogenize.py:111-117)."""
    torch = _lib.require_cuda()
    from .errors import SolverDidNotConverge
    from .operators import StiffnessBatch
    from .solver import SolveOptions, pcg_solve_batched

    opts = opts or SolveOptions()
    cfg = realizations[0].config
    d, n, M = 3, cfg.n, len(realizations)
    h = 1.0 / n
    beta = np.stack([r.beta_cells.ravel() for r in realizations])          # (M, L^3)
    A1 = StiffnessBatch(cfg, beta)
    loads = torch.stack([corrector_rhs_batched(A1, i, pcg_scaled=False) for i in (1, 2, 3)], dim=1)
    beta3 = np.repeat(beta, d, axis=0)                                     # realization-major
    A3 = StiffnessBatch(cfg, beta3)
    F = (h ** (2 - d)) * loads.reshape(M * d, n ** 3)                      # homogenize.py:110
    res = pcg_solve_batched(A3, F, opts, precond, record_history=True)
    U = res.u.reshape(M, d, n ** 3)
    # <f_j, u_i> for all (i, j): (M, d, d) on the device
    G = torch.einsum("mjx,mix->mij", loads, U)
    # integral of the nodal coefficient: h^d * sum(c) = h^d * sum of the cell field
    # (nodal averaging preserves the sum); k^3 h-cells per covered cell
    integral = (h ** d) * (float(cfg.k) ** 3) * torch.as_tensor(beta, device=U.device).sum(dim=1)
    mats = (-G).cpu().numpy()
    integral = integral.cpu().numpy()
    out = []
    for m, r in enumerate(realizations):
        st = res.status[m * d:(m + 1) * d]
        its = tuple(int(v) for v in res.iterations[m * d:(m + 1) * d])
        if np.any(st != 0):
            if not skip_failed:
                i = int(np.argmax(st != 0))
                raise SolverDidNotConverge(
                    f"corrector {i + 1} did not converge in {opts.max_iter} iterations",
                    report=res.report(m * d + i, "lkr" if precond is None else precond.name),
                    metadata={"seed": r.seed, "L": cfg.L, "lambda": cfg.lam, "direction": i + 1})
            out.append(None)
            continue
        mat = mats[m].copy()
        mat[np.diag_indices(d)] += cfg.lam + integral[m]
        out.append(HomogenizedMatrix(matrix=mat, seed=r.seed, L=cfg.L, lam=cfg.lam, iterations=its,
                                     num_covered=r.num_covered))
    return out


def homogenized_matrix(r: Realization, opts=None, precond=None) -> HomogenizedMatrix:
    """Drop-in for homogenize.py:92-124 (the three solves batched on the GPU)."""
    return homogenized_matrix_batched([r], opts, precond)[0]


def ensemble_run(config, M: int, master_seed: int, opts=None, skip_failed: bool = False,
                 chunk: int = 64) -> EnsembleStats:
    """Drop-in for homogenize.py:133-182: M realizations with sub-seeds from the
    master seed, solved in GPU batches of ``chunk`` realizations (3 chunk
    systems per launch) instead of a process pool; statistics in index order."""
    from .errors import SolverDidNotConverge
    from .lattice import derive_seed, sample_realization

    if M < 2:
        raise ValueError(f"need at least 2 realizations, got {M}")
    records: list = []
    failed = []
    for s in range(0, M, chunk):
        rs = [sample_realization(config, derive_seed(master_seed, m)) for m in range(s, min(M, s + chunk))]
        recs = homogenized_matrix_batched(rs, opts, skip_failed=skip_failed)
        for r, rec in zip(rs, recs):
            if rec is None:
                failed.append(r.seed)
            records.append(rec)
    kept = [rec for rec in records if rec is not None]
    if len(kept) < 2:
        raise SolverDidNotConverge(f"only {len(kept)} of {M} realizations usable", metadata={})
    stack = np.stack([rec.matrix for rec in kept])
    average = stack.mean(axis=0)
    std = np.sqrt(((stack - average) ** 2).sum(axis=0) / (len(kept) - 1))
    return EnsembleStats(d=3, L=config.L, M=len(kept), lam=config.lam, average=average, std=std,
                         records=tuple(kept), failed_seeds=tuple(failed))
