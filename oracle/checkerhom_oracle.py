"""CPU oracle for the PCG hot path of arXiv 2007.06524 (reference package ``checkerhom``).

TEST INFRASTRUCTURE ONLY.  This module is a plain-numpy restatement of the
reference algorithm, used as the checker by ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product
package ``paper_2007_06524_b200`` never imports it.

Parity status: PINNED.  Every function below is checked against golden vectors
produced by the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/checkerhom`` in the build container and commits the
outputs under ``tests/golden/``), see ``tests/test_oracle_golden.py``.

Each function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/checkerhom``; ``tests/oracles.py`` relative to
``/root/reference/pkg``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ----------------------------------------------------------------------------
# Lattice sampling (lattice.py)
# ----------------------------------------------------------------------------


def derive_seed(master_seed: int, index: int) -> int:
    """lattice.py:273-276 -- SeedSequence(entropy, spawn_key=(index,)) first u64."""
    ss = np.random.SeedSequence(entropy=int(master_seed), spawn_key=(int(index),))
    return int(ss.generate_state(1, np.uint64)[0])


def sample_beta_cells(L: int, lam: float, seed: int, d: int = 3, coverage_prob: float = 0.5,
                      contrast: str = "fixed", betas: tuple = ()) -> np.ndarray:
    """Per-cell beta array of shape (L,)*d, vectorised restatement of
    ``sample_realization`` (lattice.py:284-311) with the Philox stream of
    lattice.py:279-281.  Uncovered cells carry 0.

    Coverage consumes one uniform per cell in C order (lattice.py:293); the
    two_value choice consumes a second full block (lattice.py:294,304); the
    layered amplitude depends on the last cell coordinate (lattice.py:306-307).
    """
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(int(seed))))
    num = L ** d
    u_cover = rng.random(num)
    u_beta = rng.random(num) if contrast == "two_value" else None
    covered = u_cover < coverage_prob
    if contrast == "fixed":
        vals = np.full(num, 1.0 - lam)
    elif contrast == "two_value":
        vals = np.where(u_beta < 0.5, float(betas[0]), float(betas[1]))
    elif contrast == "layered":
        last = np.arange(num) % L
        vals = np.asarray(betas, dtype=float)[last % len(betas)]
    else:
        raise ValueError(f"unknown contrast kind {contrast!r}")
    return np.where(covered, vals, 0.0).reshape((L,) * d)


def subcell_geometry(n0: int, alpha_num: int, alpha_den: int, subcell_offset=None):
    """lattice.py:151-166: k = 2*alpha*n0, offset = (n0-k)//2 unless given."""
    k2 = 2 * alpha_num * n0
    assert k2 % alpha_den == 0
    k = k2 // alpha_den
    off = (n0 - k) // 2 if subcell_offset is None else int(subcell_offset)
    return k, off


def cell_field(beta_cells: np.ndarray, n0: int, k: int, offset: int) -> np.ndarray:
    """beta-weighted indicator over the n^d h-cells (lattice.py:314-317,326-332;
    tests/oracles.py:22-32).  h-cell j lies in cell j//n0 and inside the
    sub-cell iff offset <= j mod n0 < offset + k."""
    d = beta_cells.ndim
    L = beta_cells.shape[0]
    n = n0 * L
    j = np.arange(n)
    inside = ((j % n0) >= offset) & ((j % n0) < offset + k)
    cell = j // n0
    F = beta_cells
    for ax in range(d):
        F = np.take(F, cell, axis=ax)
    mask = inside
    for _ in range(d - 1):
        mask = mask[..., None] & inside
    # mask over axes in order (a0, a1, ..., ad-1)
    return np.where(mask.reshape((n,) * d), F, 0.0)


def coefficient_grid(F: np.ndarray) -> np.ndarray:
    """lattice.py:335-345: nodal average of the 2^d incident h-cells."""
    vals = F
    for axis in range(F.ndim):
        vals = 0.5 * (vals + np.roll(vals, 1, axis=axis))
    return vals


def corrector_rhs(F: np.ndarray, i: int) -> np.ndarray:
    """homogenize.py:75-89: h^(d-1) * 1/2 (c[x+e_i] - c[x-e_i]), axis = i-1."""
    d = F.ndim
    n = F.shape[0]
    c = coefficient_grid(F)
    axis = i - 1
    h = 1.0 / n
    diff = 0.5 * (np.roll(c, -1, axis=axis) - np.roll(c, 1, axis=axis))
    return (h ** (d - 1)) * diff.ravel()


def pcg_rhs_corrector(F: np.ndarray, i: int = 1) -> np.ndarray:
    """The PCG right-hand side used by the callers: h^(2-d) * corrector_rhs
    (homogenize.py:110, cli.py:340)."""
    d = F.ndim
    h = 1.0 / F.shape[0]
    return (h ** (2 - d)) * corrector_rhs(F, i)


def gaussian_rhs(n: int, seed: int, d: int = 3) -> np.ndarray:
    """Config-4 RHS: default_rng(seed).standard_normal(n^d), mean removed."""
    f = np.random.default_rng(int(seed)).standard_normal(n ** d)
    return f - f.mean()


# ----------------------------------------------------------------------------
# Stiffness (tests/oracles.py:35-82, operators.py:96-131)
# ----------------------------------------------------------------------------


def edge_weights(F: np.ndarray, lam: float) -> list:
    """g_a(x) for every axis a: conductivity of the edge x -> x+e_a, i.e.
    lam + mean of the 2^(d-1) h-cells adjacent to the edge
    (tests/oracles.py:60-70).  The h-cell along axis a is x_a itself and the
    transverse coordinates are x_b - delta_b, delta in {0,1}."""
    d = F.ndim
    gs = []
    for ax in range(d):
        acc = F
        for m in range(d):
            if m == ax:
                continue
            acc = acc + np.roll(acc, 1, axis=m)
        gs.append(lam + acc / 2 ** (d - 1))
    return gs


def stencil_apply(F: np.ndarray, lam: float, x: np.ndarray, gs=None) -> np.ndarray:
    """y = A x for the edge-weighted periodic graph Laplacian equal to the
    reference CSR stiffness (tests/oracles.py:72-75 entry pattern):
    y_x = sum_a g_a(x)(x_x - x_{x+e_a}) + g_a(x-e_a)(x_x - x_{x-e_a})."""
    d = F.ndim
    n = F.shape[0]
    if gs is None:
        gs = edge_weights(F, lam)
    X = np.asarray(x, dtype=float).reshape((n,) * d)
    Y = np.zeros_like(X)
    for ax in range(d):
        g = gs[ax]
        fwd = X - np.roll(X, -1, axis=ax)
        Y += g * fwd
        Y -= np.roll(g * fwd, 1, axis=ax)
    return Y.ravel()


class StencilMatrix:
    """Duck-typed stand-in for the reference CSR: ``matrix() @ x``
    (solver.py:150,162) evaluated matrix-free."""

    def __init__(self, F, lam):
        self.F = F
        self.lam = float(lam)
        self.gs = edge_weights(F, lam)
        self.d = F.ndim
        self.n = F.shape[0]

    def __matmul__(self, x):
        return stencil_apply(self.F, self.lam, x, self.gs)

    def matrix(self):
        return self

    def apply(self, x):
        return self @ x


# ----------------------------------------------------------------------------
# Spectral setup (spectral.py) and LKR factors (lowrank.py)
# ----------------------------------------------------------------------------


def fourier_eigenvalues(n: int) -> np.ndarray:
    """spectral.py:56-68: Re FFT of (2,-1,0,...,-1), negatives clipped."""
    if n < 3:
        raise ValueError(f"need n >= 3, got {n}")
    p = np.zeros(n)
    p[0] = 2.0
    p[1] = -1.0
    p[-1] = -1.0
    lam = np.fft.fft(p)
    values = lam.real.copy()
    values[values < 0.0] = 0.0
    return values


def _trapezoid_rule(rank: int, eps: float, rho: float):
    """lowrank.py:53-64."""
    s_min = math.log(eps / (8.0 * rho))
    s_max = math.log(math.log(8.0 / eps) + 4.0)
    s = np.linspace(s_min, s_max, rank)
    step = s[1] - s[0]
    nodes = np.exp(s)
    return nodes, step * nodes


def _sup_rel_error(nodes, weights, rho: float) -> float:
    """lowrank.py:67-71 (4096 geometric validation points)."""
    y = np.geomspace(1.0, rho, 4096)
    with np.errstate(under="ignore"):
        approx = np.exp(-np.outer(y, nodes)) @ weights
    return float(np.max(np.abs(approx * y - 1.0)))


def exp_sum_quadrature(a: float, b: float, eps: float, max_rank: int = 256):
    """lowrank.py:74-120: doubling + bisection on the rank; returns
    (nodes, weights) rescaled to [a, b]."""
    if not (0.0 < a < b):
        raise ValueError(f"need 0 < a < b, got a={a}, b={b}")
    if eps <= 0.0:
        raise ValueError(f"tolerance must be positive, got {eps}")
    rho = b / a

    def error_at(rank):
        nodes, weights = _trapezoid_rule(rank, eps, rho)
        return _sup_rel_error(nodes, weights, rho)

    rank, previous = 8, 2
    while rank <= max_rank:
        if error_at(rank) <= eps:
            break
        previous, rank = rank, rank * 2
    else:
        raise RuntimeError(f"no rank <= {max_rank} reaches eps={eps}")
    lo, hi = previous, rank
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if error_at(mid) <= eps:
            hi = mid
        else:
            lo = mid
    nodes, weights = _trapezoid_rule(hi, eps, rho)
    return nodes / a, weights / a


def lkr_factors(n: int, d: int = 3, eps: float = 1e-8) -> tuple:
    """canonical_reciprocal + dc_correction (lowrank.py:147-180): d arrays of
    shape (R+1, n).  Rows 0..R-1: w_k^(1/d) exp(-t_k lam_i); row R: the
    origin fix (-value(0,...,0) at [0] on mode 0, 1 at [0] elsewhere)."""
    lam = fourier_eigenvalues(n)
    positive = lam[lam > 0.0]
    a = float(positive.min())
    b = float(d * lam.max())
    nodes, weights = exp_sum_quadrature(a, b, eps)
    with np.errstate(under="ignore"):
        base = np.exp(-np.outer(nodes, lam))
    scale = weights ** (1.0 / d)
    factor = scale[:, None] * base
    # CanonicalTensor.value at the origin (lowrank.py:136-139)
    prod = factor[:, 0].copy()
    for _ in range(1, d):
        prod *= factor[:, 0]
    origin = float(prod.sum())
    out = []
    for axis in range(d):
        e0 = np.zeros((1, n))
        e0[0, 0] = -origin if axis == 0 else 1.0
        out.append(np.vstack([factor, e0]))
    return tuple(out)


def lkr_diagonal(factors) -> np.ndarray:
    """CanonicalTensor.diagonal (lowrank.py:141-144)."""
    if len(factors) == 3:
        return np.einsum("ka,kb,kc->abc", *factors, optimize=True)
    return np.einsum("ka,kb->ab", *factors, optimize=True)


def apply_lkr(factors, x: np.ndarray, diag=None) -> np.ndarray:
    """lowrank.py:183-192: Re ifftn(D * fftn(x))."""
    d = len(factors)
    n = factors[0].shape[1]
    x = np.asarray(x, dtype=float)
    if x.shape != (n ** d,):
        raise ValueError(f"expected vector of length {n ** d}, got shape {x.shape}")
    if diag is None:
        diag = lkr_diagonal(factors)
    spec = np.fft.fftn(x.reshape((n,) * d))
    spec *= diag
    return np.fft.ifftn(spec).real.ravel()


def pseudoinverse_diag(n: int, d: int = 3, delta: float = 0.0) -> np.ndarray:
    """spectral.py:77-95: 1/(lam_i+lam_j+lam_k) with the origin zeroed, or
    1/(g+delta) for the regularized kind."""
    lam = fourier_eigenvalues(n)
    g = lam
    for _ in range(d - 1):
        g = g[..., None] + lam
    if delta > 0.0:
        return 1.0 / (g + delta)
    out = np.zeros_like(g)
    mask = g > 0.0
    out[mask] = 1.0 / g[mask]
    return out


def apply_fourier(diag: np.ndarray, x: np.ndarray) -> np.ndarray:
    """spectral.py:98-112."""
    n = diag.shape[0]
    d = diag.ndim
    spec = np.fft.fftn(np.asarray(x, dtype=float).reshape((n,) * d))
    spec *= diag
    return np.fft.ifftn(spec).real.ravel()


# ----------------------------------------------------------------------------
# PCG (solver.py:103-194)
# ----------------------------------------------------------------------------


@dataclass
class OracleReport:
    iterations: int
    residuals: tuple
    converged: bool
    final_residual: float
    rhs_projected: bool = False
    breakdown: bool = False


def project_mean_zero(x):
    """solver.py:103-106."""
    x = np.asarray(x, dtype=float)
    return x - x.mean()


def pcg_solve(matvec, f, precond_apply, tol=1e-8, max_iter=500,
              precond_residual_stopping=False):
    """Restatement of solver.py:118-194 (warning -> flag, raise -> flag)."""
    f = np.asarray(f, dtype=float)
    norm_f = float(np.linalg.norm(f))
    if norm_f == 0.0:
        return np.zeros_like(f), OracleReport(0, (), True, 0.0)
    rhs_projected = False
    if abs(f.sum()) > 1e-10 * norm_f:
        f = project_mean_zero(f)
        norm_f = float(np.linalg.norm(f))
        rhs_projected = True
        if norm_f == 0.0:
            return np.zeros_like(f), OracleReport(0, (), True, 0.0, True)
    u = np.zeros_like(f)
    r = f.copy()
    z = project_mean_zero(precond_apply(r))
    p = z.copy()
    rz = float(r @ z)
    norm_pf = float(np.sqrt(abs(rz)))
    history = []
    converged = False
    iterations = 0
    for iterations in range(1, max_iter + 1):
        q = matvec(p)
        pq = float(p @ q)
        if not np.isfinite(pq) or pq <= 0.0:
            return u, OracleReport(iterations, tuple(history), False,
                                   history[-1] if history else float("nan"),
                                   rhs_projected, breakdown=True)
        step = rz / pq
        u += step * p
        r -= step * q
        u = project_mean_zero(u)
        rel = float(np.linalg.norm(r)) / norm_f
        if not np.isfinite(rel):
            return u, OracleReport(iterations, tuple(history), False, rel,
                                   rhs_projected, breakdown=True)
        history.append(rel)
        if not precond_residual_stopping and rel <= tol:
            converged = True
            break
        z = project_mean_zero(precond_apply(r))
        rz_next = float(r @ z)
        if precond_residual_stopping and np.sqrt(abs(rz_next)) / norm_pf <= tol:
            converged = True
            break
        p = z + (rz_next / rz) * p
        rz = rz_next
    return u, OracleReport(iterations, tuple(history), converged, history[-1],
                           rhs_projected)


# ----------------------------------------------------------------------------
# The BASELINE.json workloads
# ----------------------------------------------------------------------------

# name: (L, n0, lam, batch, tol, rhs)
CONFIGS = {
    1: dict(L=8, n0=4, lam=0.1, batch=1, tol=1e-8, rhs="corrector"),
    2: dict(L=16, n0=4, lam=0.1, batch=64, tol=1e-8, rhs="corrector"),
    3: dict(L=32, n0=4, lam=0.01, batch=256, tol=1e-8, rhs="corrector"),
    4: dict(L=64, n0=4, lam=0.1, batch=16, tol=1e-10, rhs="gaussian"),
    5: dict(L=32, n0=16, lam=0.1, batch=1, tol=1e-8, rhs="corrector"),
}


def config_problem(cfg: int, m: int, master_seed: int = 0):
    """(F, lam, f) for realization m of BASELINE config ``cfg`` with alpha=1/2."""
    c = CONFIGS[cfg]
    seed = derive_seed(master_seed, m)
    beta = sample_beta_cells(c["L"], c["lam"], seed)
    k, off = subcell_geometry(c["n0"], 1, 2)
    F = cell_field(beta, c["n0"], k, off)
    n = c["n0"] * c["L"]
    if c["rhs"] == "corrector":
        f = pcg_rhs_corrector(F, 1)
    else:
        f = gaussian_rhs(n, seed)
    return beta, F, f


def solve_config(cfg: int, m: int, factors=None, master_seed: int = 0):
    """Oracle PCG solve of realization m of a BASELINE config (lkr, eps 1e-8)."""
    c = CONFIGS[cfg]
    beta, F, f = config_problem(cfg, m, master_seed)
    n = F.shape[0]
    if factors is None:
        factors = lkr_factors(n)
    diag = lkr_diagonal(factors)
    A = StencilMatrix(F, c["lam"])
    return pcg_solve(A.__matmul__, f, lambda x: apply_lkr(factors, x, diag), tol=c["tol"])
