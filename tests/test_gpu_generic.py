"""Grid sizes without a fused fast path (n = n0 * L with any L; the reference's own
tests use n = 12 and 24): the generic CUDA kernels (chk_generic.cuh) through the
same C ABI and Python surface, against outputs of the reference itself
(tests/golden/generic.npz, written by make_golden.py generic).  Same bars as the
power-of-two sizes: iteration counts exact, histories 1e-8, solutions 1e-9."""

import numpy as np
import pytest

from conftest import golden_generic

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2007_06524_b200 as chk  # noqa: E402


def _ids(prefix):
    g = golden_generic()
    return sorted({k.split("_")[0] for k in g.files if k.startswith(prefix)})


def _cfg(g, case):
    d, L, n0, k, off, _ = (int(v) for v in g[case + "_meta"])
    return chk.LatticeConfig(d=3, L=L, n0=n0, alpha=f"{k}/{2 * n0}", lam=float(g[case + "_lam"]), subcell_offset=off)


@pytest.mark.parametrize("case", _ids("case"))
def test_stencil_and_rhs_generic(case):
    """chk_stencil_apply / chk_corrector_rhs at n = 12, 24, 20 vs the reference CSR
    product (operators.py:122-131) and corrector_rhs (homogenize.py:75-89)."""
    g = golden_generic()
    cfg = _cfg(g, case)
    n = cfg.n
    ci = int(case[4:])
    x = np.random.default_rng(3000 + ci).standard_normal(n ** 3)
    A = chk.StiffnessBatch(cfg, g[case + "_beta"].reshape(1, -1))
    y, xy = A.matvec(torch.as_tensor(x).reshape(1, -1), with_dot=True)
    ref = g[case + "_Ax"]
    assert np.linalg.norm(y.cpu().numpy().ravel() - ref) <= 1e-14 * np.linalg.norm(ref)
    assert abs(float(xy[0]) - x @ ref) <= 1e-12 * abs(x @ ref)
    for i in (1, 2, 3):
        f = chk.corrector_rhs_batched(A, i, pcg_scaled=False).cpu().numpy().ravel()
        assert np.allclose(f, g[case + f"_rhs{i}"], rtol=0, atol=1e-17)


@pytest.mark.parametrize("n", [12, 20])
def test_preconditioner_apply_generic(n):
    """chk_precond_apply (direct Fourier sums) vs the reference's pocketfft applies."""
    g = golden_generic()
    x = g[f"lkr_x_n{n}"]
    t = chk.dc_correction(chk.canonical_reciprocal(chk.fourier_eigenvalues(n), 3, 1e-8))
    assert np.array_equal(np.stack(t.factors), g[f"factors_n{n}"])
    y = chk.apply_lkr_preconditioner(t, x)
    ref = g[f"lkr_y_n{n}"]
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    yf = chk.apply_fourier_preconditioner(n, x)
    assert np.linalg.norm(yf - g[f"fourier_y_n{n}"]) <= 1e-13 * np.linalg.norm(yf)
    yr = chk.apply_fourier_preconditioner(n, x, delta=1e-3)
    assert np.linalg.norm(yr - g[f"reg_y_n{n}"]) <= 1e-13 * np.linalg.norm(yr)


@pytest.mark.parametrize("pid", _ids("pcg"))
def test_pcg_generic_golden(pid):
    """Reference pcg_solve runs at n = 12, 24, 20, 28 (lkr / fourier with a projected
    noisy load / regularized / precond-residual stopping / non-convergence)."""
    g = golden_generic()
    L, n0, k, off, its, conv, prs, max_iter, proj = (int(v) for v in g[pid + "_meta"])
    lam, tol = (float(v) for v in g[pid + "_lam_tol"])
    kind = str(g[pid + "_kind"])
    cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha=f"{k}/{2 * n0}", lam=lam, subcell_offset=off)
    A = chk.assemble_stiffness(chk.realization_from_beta(cfg, g[pid + "_beta"]))
    opts = chk.SolveOptions(tol=tol, preconditioner=kind, eps_rank=1e-8,
                            delta=1e-3 if kind == "regularized" else 0.0,
                            precond_residual_stopping=bool(prs), max_iter=max_iter)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        u, rep = chk.pcg_solve(A, g[pid + "_f"], opts)
    assert rep.iterations == its
    assert rep.converged == bool(conv)
    assert rep.rhs_projected == bool(proj)
    assert rep.preconditioner == str(g[pid + "_name"])
    assert np.allclose(rep.residuals, g[pid + "_res"], rtol=1e-8, atol=0)
    uref = g[pid + "_u"]
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    assert abs(u.mean()) <= 1e-12 * np.abs(u).max()


def test_generic_batch_matches_single_solves():
    """A ragged generic batch (n = 12: different realizations, a zero load among them)
    behaves like its own single solves, bit for bit, and through the seeds pipeline."""
    cfg = chk.LatticeConfig(d=3, L=3, n0=4, alpha="1/2", lam=0.05)
    rs = [chk.sample_realization(cfg, chk.derive_seed(9, m)) for m in range(5)]
    A = chk.StiffnessBatch(cfg, np.stack([r.beta_cells.ravel() for r in rs]))
    F = chk.corrector_rhs_batched(A, 2)
    F[3].zero_()
    opts = chk.SolveOptions(tol=1e-9, preconditioner="lkr")
    res = chk.pcg_solve_batched(A, F, opts)
    assert int(res.iterations[3]) == 0 and res.status[3] == 0
    assert float(res.u[3].abs().max()) == 0.0
    for m in (0, 2, 4):
        one = chk.pcg_solve_batched(chk.StiffnessBatch(cfg, rs[m].beta_cells.reshape(1, -1)), F[m:m + 1], opts)
        assert int(one.iterations[0]) == int(res.iterations[m])
        assert torch.equal(one.u[0], res.u[m])
    seeds = [chk.derive_seed(9, m) for m in range(5)]
    u_seeds = chk.pcg_solve_seeds(cfg, seeds, opts, rhs=2).u.reshape(5, -1)
    for m in (0, 1, 2, 4):
        assert torch.equal(u_seeds[m], res.u[m].cpu())


def test_homogenized_matrix_generic():
    """homogenize.py:92-124 at n = 12: the three corrector solves in one generic batch."""
    g = golden_generic()
    L, n0, k, off, seed = (int(v) for v in g["homog0_meta"])
    lam, tol = (float(v) for v in g["homog0_lam_tol"])
    cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha=f"{k}/{2 * n0}", lam=lam, subcell_offset=off)
    rec = chk.homogenized_matrix(chk.sample_realization(cfg, seed), chk.SolveOptions(tol=tol, preconditioner="lkr"))
    assert rec.iterations == tuple(int(v) for v in g["homog0_its"])
    ref = g["homog0_matrix"]
    assert np.max(np.abs(rec.matrix - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_unsupported_grids_raise_value_error():
    # d = 2 and n beyond the generic path's shared-memory bound stay ValueError
    with pytest.raises(ValueError):
        chk.make_preconditioner(3, 724, chk.SolveOptions(preconditioner="fourier")).apply(np.ones(724 ** 3))
    with pytest.raises(ValueError):
        chk.make_preconditioner(2, 12, chk.SolveOptions(preconditioner="fourier")).apply(np.ones(144))
