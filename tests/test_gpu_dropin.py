"""The drop-in surface on the GPU: the 3-D cases of the reference's own solver and
spectral test classes (pkg/tests/test_solver.py, test_spectral.py -- its 2-D cases
are outside the d = 3 GPU path), run against this package, plus the entry
points added for reference callers: ``apply_fourier_preconditioner(g_plus, x)``,
reference-named preconditioners, realization-carrying operators, ``residual``,
the device sampler and the seeds-to-solutions pipeline.

Dense references are built here from the pinned oracle stencil
(oracle/checkerhom_oracle.py, = tests/oracles.py:35-82) at n = 8 and 16.
"""

import numpy as np
import pytest

from oracle import checkerhom_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2007_06524_b200 as chk  # noqa: E402


def corrector_system(L=2, n0=4, lam=0.4, seed=1, alpha="1/4", direction=1, **kw):
    """The reference tests' helper (test_solver.py:21-27) at d = 3."""
    cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha=alpha, lam=lam, **kw)
    r = chk.sample_realization(cfg, seed)
    A = chk.assemble_stiffness(r)
    h = 1.0 / cfg.n
    f = (h ** (2 - 3)) * chk.corrector_rhs(r, direction)
    return A, f, r


def dense_matrix(r):
    cfg = r.config
    F = orc.cell_field(r.beta_cells, cfg.n0, cfg.k, cfg.offset)
    N = cfg.n ** 3
    S = orc.StencilMatrix(F, cfg.lam)
    return np.stack([S @ e for e in np.eye(N)], axis=1)


def dense_solve_mean_zero(Ad, f):
    w, V = np.linalg.eigh(Ad)
    inv = np.where(np.abs(w) > 1e-10, 1.0 / np.where(np.abs(w) > 1e-10, w, 1.0), 0.0)
    return (V * inv) @ V.T @ (f - f.mean())


# ---- test_solver.py TestPcg / TestResidual, d = 3 ---------------------------------


def test_exact_preconditioner_converges_immediately():
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, lam=1.0, coverage_prob=0.0)
    A = chk.assemble_stiffness(chk.sample_realization(cfg, 1))
    f = np.random.default_rng(2).standard_normal(cfg.n ** 3)
    f -= f.mean()
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-10))
    assert rep.converged and rep.iterations <= 2


def test_matches_dense_pseudo_inverse_solve():
    A, f, r = corrector_system(seed=3)
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-10))
    ref = dense_solve_mean_zero(dense_matrix(r), f)
    assert rep.converged
    assert np.linalg.norm(u - ref) <= 1e-6 * np.linalg.norm(ref)


def test_3d_iteration_bound_small():
    for seed in range(3):
        A, f, _ = corrector_system(L=4, lam=0.4, seed=seed)
        _, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-7))
        assert rep.converged and rep.iterations <= 20


def test_solution_mean_zero_and_residual_history():
    A, f, _ = corrector_system(seed=4)
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9))
    assert abs(u.mean()) <= 1e-12 * np.max(np.abs(u))
    assert rep.final_residual == rep.residuals[-1]
    assert chk.residual(A, u, f) <= 2.0 * rep.final_residual + 1e-15


def test_preconditioned_residual_stopping_and_regularized():
    A, f, _ = corrector_system(seed=9)
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9, precond_residual_stopping=True))
    assert rep.converged and chk.residual(A, u, f) <= 1e-6
    A, f, _ = corrector_system(seed=10)
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-8, preconditioner="regularized", delta=1e-3))
    assert rep.converged and "regularized" in rep.preconditioner


def test_residual_semantics():
    """solver.py:109-115 (test_solver.py TestResidual)."""
    A, f, r = corrector_system(seed=12)
    assert chk.residual(A, np.zeros_like(f), f) == pytest.approx(1.0)
    u = dense_solve_mean_zero(dense_matrix(r), f)
    assert chk.residual(A, u, f) <= 1e-12
    assert chk.residual(A, u, 2.0 * f) == pytest.approx(0.5, abs=1e-10)
    assert chk.residual(A, np.zeros_like(f), np.zeros_like(f)) == 0.0


def test_iterations_stable_across_lattice_sizes_3d():
    counts = []
    for L in (4, 8, 16):
        for seed in range(5):
            A, f, _ = corrector_system(L=L, lam=0.4, seed=seed)
            _, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-7))
            assert rep.converged
            counts.append(rep.iterations)
    assert max(counts) - min(counts) <= 5


def test_fourier_and_lkr_solutions_agree():
    for seed in range(3):
        A, f, _ = corrector_system(L=8, seed=seed)
        u_f, rep_f = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9))
        u_l, rep_l = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9, preconditioner="lkr", eps_rank=1e-8))
        assert np.linalg.norm(u_f - u_l) <= 1e-6 * np.linalg.norm(u_f)
        assert abs(rep_f.iterations - rep_l.iterations) <= 2


def test_factory_names():
    assert chk.make_preconditioner(3, 8, chk.SolveOptions()).name == "fourier"
    p = chk.make_preconditioner(3, 16, chk.SolveOptions(preconditioner="lkr"))
    assert p.name.startswith("lkr(eps=1e-08,rank=")
    assert chk.make_preconditioner(3, 8, chk.SolveOptions(preconditioner="regularized", delta=0.5)).name == \
        "regularized(delta=0.5)"


# ---- test_spectral.py TestApply, d = 3, reference signature ---------------------------


@pytest.mark.parametrize("n", [8, 16])
def test_fourier_apply_matches_dense_pseudo_inverse(n):
    gp = chk.pseudoinverse_diag(chk.eigensum_tensor(3, chk.fourier_eigenvalues(n)))
    cfg = chk.LatticeConfig(d=3, L=n // 4, n0=4, lam=1.0, coverage_prob=0.0)
    Ad = dense_matrix(chk.sample_realization(cfg, 0)) if n == 8 else None
    rng = np.random.default_rng(n)
    for _ in range(3):
        x = rng.standard_normal(n ** 3)
        y = chk.apply_fourier_preconditioner(gp, x)
        assert y.dtype == np.float64
        assert abs(y.sum()) <= 1e-11 * np.linalg.norm(y, 1)  # dc of the output vanishes
        if Ad is not None:
            w, V = np.linalg.eigh(Ad)
            inv = np.where(w > 1e-10, 1.0 / np.where(w > 1e-10, w, 1.0), 0.0)
            assert np.linalg.norm(y - (V * inv) @ V.T @ x) <= 1e-10 * np.linalg.norm(x)
            xm = x - x.mean()
            back = Ad @ chk.apply_fourier_preconditioner(gp, xm)
            assert np.linalg.norm(back - xm) <= 1e-10 * np.linalg.norm(xm)
    x, z = rng.standard_normal((2, n ** 3))
    px, pz = chk.apply_fourier_preconditioner(gp, x), chk.apply_fourier_preconditioner(gp, z)
    assert abs(px @ z - x @ pz) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(z)
    assert px @ x > 0.0
    assert np.max(np.abs(chk.apply_fourier_preconditioner(gp, np.full(n ** 3, 3.0)))) <= 1e-14
    with pytest.raises(ValueError):
        chk.apply_fourier_preconditioner(gp, np.ones(n ** 3 + 1))


def test_fourier_apply_golden_reference_signature():
    from conftest import golden_small

    g = golden_small()
    for n in (8, 16, 32):
        x = g[f"lkr_x_n{n}"]
        es = chk.eigensum_tensor(3, chk.fourier_eigenvalues(n))
        y = chk.apply_fourier_preconditioner(chk.pseudoinverse_diag(es), x)
        assert np.linalg.norm(y - g[f"fourier_y_n{n}"]) <= 1e-13 * np.linalg.norm(y)
        y = chk.apply_fourier_preconditioner(chk.regularized_inverse_diag(es, 1e-3), x)
        assert np.linalg.norm(y - g[f"reg_y_n{n}"]) <= 1e-13 * np.linalg.norm(y)


# ---- reference callers -------------------------------------------------------------


def test_reference_named_preconditioner_and_realization_operator():
    """A Preconditioner(name, apply) as the reference's make_preconditioner builds
    it (no device plan) is mapped to the device plan of the same name; an operator
    carrying its realization is accepted; anything else raises ValueError."""
    A, f, r = corrector_system(L=4, seed=2)
    u0, rep0 = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9, preconditioner="lkr"))
    ours = chk.make_preconditioner(3, A.n, chk.SolveOptions(preconditioner="lkr"))
    foreign = chk.Preconditioner(ours.name, lambda x: x)  # name + apply, no plan
    u1, rep1 = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-9, preconditioner="lkr"), precond=foreign)
    assert rep1.iterations == rep0.iterations and np.array_equal(u1, u0)

    class Carrier:  # any operator that carries its realization (d, n, realization)
        d, n, realization = 3, A.n, r

    u2, rep2 = chk.pcg_solve(Carrier(), f, chk.SolveOptions(tol=1e-9, preconditioner="lkr"))
    assert np.array_equal(u2, u0)
    with pytest.raises(ValueError):
        chk.pcg_solve(A, f, precond=chk.Preconditioner("my-own", lambda x: x))

    class Kron:  # the reference's StiffnessOperator shape: Kronecker terms only
        d, n = 3, A.n

        def matrix(self):
            return None

    with pytest.raises(ValueError):
        chk.pcg_solve(Kron(), f)


# ---- device sampler and the seeds-to-solutions pipeline ----------------------------


def test_device_sampler_bit_identical_config3():
    """chk_sample_cells vs sample_realization for all 256 config-3 seeds (and a
    two_value contrast with odd L, where the second uniform block is unaligned)."""
    cfg = chk.LatticeConfig(d=3, L=32, n0=4, alpha="1/2", lam=0.01)
    seeds = [chk.derive_seed(0, m) for m in range(256)]
    dev = chk.sample_cells_device(cfg, seeds).cpu().numpy()
    for m, s in enumerate(seeds):
        assert np.array_equal(dev[m], chk.sample_realization(cfg, s).beta_cells.ravel()), m
    cfg2 = chk.LatticeConfig(d=3, L=5, n0=4, alpha="1/4", lam=0.2, contrast=chk.ContrastModel.two_value(0.3, 0.7))
    seeds2 = [chk.derive_seed(9, m) for m in range(16)]
    dev2 = chk.sample_cells_device(cfg2, seeds2).cpu().numpy()
    for m, s in enumerate(seeds2):
        assert np.array_equal(dev2[m], chk.sample_realization(cfg2, s).beta_cells.ravel()), m
    with pytest.raises(ValueError):
        chk.sample_cells_device(chk.LatticeConfig(d=3, L=4, n0=4, contrast=chk.ContrastModel.layered([0.1, 0.2])),
                                seeds[:2])


@pytest.mark.parametrize("L,batch", [(16, 20), (32, 24)])
def test_seeds_pipeline_equals_device_batch(L, batch):
    """pcg_solve_seeds (keys -> device cells -> device corrector load -> solve ->
    host u) reproduces the device-resident batched solve bit for bit."""
    cfg = chk.LatticeConfig(d=3, L=L, n0=4, alpha="1/2", lam=0.1)
    seeds = [chk.derive_seed(0, m) for m in range(batch)]
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    A = chk.StiffnessBatch(cfg, np.stack([chk.sample_realization(cfg, s).beta_cells.ravel() for s in seeds]))
    res = chk.pcg_solve_batched(A, chk.corrector_rhs_batched(A, 1), opts)
    got = chk.pcg_solve_seeds(cfg, seeds, opts, chunk=max(1, batch // 3))
    assert np.array_equal(got.iterations, res.iterations)
    assert np.array_equal(got.status, res.status)
    assert np.array_equal(got.history, res.history)
    assert torch.equal(got.u, res.u.cpu())
    # host Gaussian loads through the same pipeline
    F = np.stack([orc.gaussian_rhs(cfg.n, s) for s in seeds[:4]])
    g1 = chk.pcg_solve_seeds(cfg, seeds[:4], opts, rhs=F)
    g2 = chk.pcg_solve_batched(chk.StiffnessBatch(cfg, A.beta[:4]), torch.as_tensor(F).cuda(), opts)
    assert np.array_equal(g1.iterations, g2.iterations)
    assert torch.equal(g1.u, g2.u.cpu())
