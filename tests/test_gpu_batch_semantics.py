"""Batched-solver semantics on the GPU against the CPU oracle: every
realization of a batch must behave exactly like its own reference pcg_solve
(solver.py:118-194), whatever its neighbours do.  Also the reference's 3-D
iteration-robustness acceptance criterion (SPEC criterion 4,
tests/test_acceptance.py:115-136)."""

import numpy as np
import pytest

from oracle import checkerhom_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2007_06524_b200 as chk  # noqa: E402


def _oracle_solve(cfg, beta, f, opts):
    F = orc.cell_field(beta, cfg.n0, cfg.k, cfg.offset)
    A = orc.StencilMatrix(F, cfg.lam)
    n = cfg.n
    if opts.preconditioner == "lkr":
        fac = orc.lkr_factors(n, eps=opts.eps_rank)
        dg = orc.lkr_diagonal(fac)
        P = lambda x: orc.apply_lkr(fac, x, dg)  # noqa: E731
    else:
        dg = orc.pseudoinverse_diag(n, delta=opts.delta if opts.preconditioner == "regularized" else 0.0)
        P = lambda x: orc.apply_fourier(dg, x)  # noqa: E731
    return orc.pcg_solve(A.__matmul__, f, P, tol=opts.tol, max_iter=opts.max_iter,
                         precond_residual_stopping=opts.precond_residual_stopping)


def _batch(cfg, betas, F, opts):
    A = chk.StiffnessBatch(cfg, np.stack([b.ravel() for b in betas]))
    return chk.pcg_solve_batched(A, torch.as_tensor(np.stack(F)).cuda(), opts)


def _check_against_oracle(cfg, betas, F, opts, res):
    for j, (beta, f) in enumerate(zip(betas, F)):
        u, rep = _oracle_solve(cfg, beta, f, opts)
        assert int(res.iterations[j]) == rep.iterations, j
        expect = 2 if rep.breakdown else (0 if rep.converged else 1)
        assert int(res.status[j]) == expect, j
        if rep.breakdown:
            continue
        assert bool(res.rhs_projected[j]) == rep.rhs_projected
        if rep.iterations:
            # relative residuals near 1e-10 carry ~1e-16 ||f|| of absolute roundoff
            assert np.allclose(res.history[j, :rep.iterations], rep.residuals, rtol=1e-7, atol=1e-14)
        ud = res.u[j].cpu().numpy()
        nu = np.linalg.norm(u)
        assert np.linalg.norm(ud - u) <= 1e-9 * max(nu, 1e-300) or nu == 0.0


@pytest.mark.parametrize("kind", ["lkr", "fourier", "regularized"])
def test_ragged_batch_mixed_outcomes(kind):
    """B = 7 (not a multiple of the middle-pass group): converged, zero RHS,
    RHS with a mean (projected), a two_value-contrast field -- in one launch."""
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/4", lam=0.3)
    rng = np.random.default_rng(7)
    betas, F = [], []
    for m in range(7):
        b = orc.sample_beta_cells(4, cfg.lam, 100 + m)
        if m == 5:
            b = orc.sample_beta_cells(4, cfg.lam, 5, contrast="two_value", betas=(0.2, 0.6))
        Fc = orc.cell_field(b, cfg.n0, cfg.k, cfg.offset)
        f = orc.pcg_rhs_corrector(Fc, 1 + m % 3)
        if m == 2:
            f = np.zeros_like(f)
        if m == 4:
            f = f + 0.25 * rng.standard_normal(f.size).mean() + 0.01
        betas.append(b)
        F.append(f)
    opts = chk.SolveOptions(tol=1e-9, preconditioner=kind, delta=1e-2 if kind == "regularized" else 0.0)
    res = _batch(cfg, betas, F, opts)
    _check_against_oracle(cfg, betas, F, opts, res)


def test_batch_with_nonconvergence_and_breakdown():
    """One realization hits max_iter, one breaks down (indefinite operator),
    the others converge -- statuses and iteration counts per realization."""
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.1)
    betas, F = [], []
    for m in range(4):
        b = orc.sample_beta_cells(4, cfg.lam, 200 + m)
        if m == 3:
            b = -40.0 * (b != 0)  # strongly indefinite operator: p'Ap < 0
        Fc = orc.cell_field(np.abs(b), cfg.n0, cfg.k, cfg.offset)
        betas.append(b)
        F.append(orc.pcg_rhs_corrector(Fc, 1))
    opts = chk.SolveOptions(tol=1e-10, preconditioner="lkr", max_iter=12)
    res = _batch(cfg, betas, F, opts)
    assert int(res.status[3]) == 2
    assert set(int(s) for s in res.status[:3]) <= {0, 1}
    _check_against_oracle(cfg, betas, F, opts, res)


def test_precond_residual_stopping_batched():
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.2)
    betas = [orc.sample_beta_cells(4, cfg.lam, 300 + m) for m in range(3)]
    F = [orc.pcg_rhs_corrector(orc.cell_field(b, cfg.n0, cfg.k, cfg.offset), 2) for b in betas]
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr", precond_residual_stopping=True)
    res = _batch(cfg, betas, F, opts)
    _check_against_oracle(cfg, betas, F, opts, res)


def test_layered_contrast_and_offset_window():
    cfg = chk.LatticeConfig(d=3, L=4, n0=8, alpha="1/4", lam=0.25,
                            contrast=chk.ContrastModel.layered([0.1, 0.7]), subcell_offset=1)
    rs = [chk.sample_realization(cfg, s) for s in (1, 2)]
    F = [orc.pcg_rhs_corrector(orc.cell_field(r.beta_cells, cfg.n0, cfg.k, cfg.offset), 3) for r in rs]
    opts = chk.SolveOptions(tol=1e-9, preconditioner="lkr")
    res = _batch(cfg, [r.beta_cells for r in rs], F, opts)
    _check_against_oracle(cfg, [r.beta_cells for r in rs], F, opts, res)


def test_bitwise_deterministic():
    """Fixed-order reductions: repeated solves give identical bits."""
    cfg = chk.LatticeConfig(d=3, L=16, n0=4, alpha="1/2", lam=0.1)
    beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(5)])
    A = chk.StiffnessBatch(cfg, beta)
    F = chk.corrector_rhs_batched(A, 1)
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    r1 = chk.pcg_solve_batched(A, F, opts)
    u1 = r1.u.clone()
    r2 = chk.pcg_solve_batched(A, F, opts)
    assert torch.equal(u1, r2.u)
    assert np.array_equal(r1.history, r2.history)


def test_acceptance_criterion_4_iteration_robustness():
    """tests/test_acceptance.py:115-136: lambda = 0.4, alpha = 1/4, tol 1e-7,
    L in {4, 8, 16}, 10 seeds x 3 directions: fourier <= 20, lkr <= 22."""
    worst = {"fourier": 0, "lkr": 0}
    for L in (4, 8, 16):
        cfg = chk.LatticeConfig(d=3, L=L, n0=4, alpha="1/4", lam=0.4)
        rs = [chk.sample_realization(cfg, seed) for seed in range(10)]
        A = chk.StiffnessBatch(cfg, np.stack([np.repeat(r.beta_cells.ravel()[None], 3, 0) for r in rs]).reshape(30, -1))
        A1 = chk.StiffnessBatch(cfg, np.stack([r.beta_cells.ravel() for r in rs]))
        F = torch.stack([chk.corrector_rhs_batched(A1, i) for i in (1, 2, 3)], dim=1).reshape(30, -1)
        for key, opts in (("fourier", chk.SolveOptions(tol=1e-7)),
                          ("lkr", chk.SolveOptions(tol=1e-7, preconditioner="lkr", eps_rank=1e-8))):
            res = chk.pcg_solve_batched(A, F, opts)
            assert np.all(res.status == 0)
            worst[key] = max(worst[key], int(res.iterations.max()))
    assert worst["fourier"] <= 20 and worst["lkr"] <= 22, worst


def test_host_buffer_pipeline_matches_device_batch():
    """chk_pcg_solve_host (chunked, copies overlapped) = chk_pcg_solve_batched, bit for bit:
    per-realization results do not depend on the batch composition."""
    cfg = chk.LatticeConfig(d=3, L=8, n0=4, alpha="1/2", lam=0.1)
    beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(7)])
    A = chk.StiffnessBatch(cfg, beta)
    F = chk.corrector_rhs_batched(A, 1)
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    ref = chk.pcg_solve_batched(A, F, opts)
    Fh = F.cpu().pin_memory()
    res = chk.pcg_solve_host(cfg, torch.from_numpy(beta).pin_memory(), Fh, opts, chunk=3)
    assert np.array_equal(res.iterations, ref.iterations)
    assert np.array_equal(res.status, ref.status)
    assert np.array_equal(res.history, ref.history)
    assert torch.equal(res.u, ref.u.cpu())


@pytest.mark.parametrize("kind", ["lkr", "fourier"])
def test_paired_schedule_matches_oracle(monkeypatch, kind):
    """CHK_PAIR=2 forces the paired schedule (two halves half an iteration apart,
    forward and inverse plane passes of different halves in one launch) on a small
    ragged batch with every outcome: converged at different iterations, zero RHS,
    projected mean, max_iter, breakdown."""
    monkeypatch.setenv("CHK_PAIR", "2")
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.1)
    betas, F = [], []
    for m in range(9):
        b = orc.sample_beta_cells(4, cfg.lam, 400 + m)
        if m == 7:
            b = -40.0 * (b != 0)
        Fc = orc.cell_field(np.abs(b), cfg.n0, cfg.k, cfg.offset)
        f = orc.pcg_rhs_corrector(Fc, 1 + m % 3)
        if m == 1:
            f = np.zeros_like(f)
        if m == 4:
            f = f + 0.03
        betas.append(b)
        F.append(f)
    for max_iter in (9, 500):
        opts = chk.SolveOptions(tol=1e-10, preconditioner=kind, max_iter=max_iter)
        res = _batch(cfg, betas, F, opts)
        assert int(res.status[7]) == 2
        _check_against_oracle(cfg, betas, F, opts, res)
        monkeypatch.setenv("CHK_PAIR", "0")
        ref = _batch(cfg, betas, F, opts)
        monkeypatch.setenv("CHK_PAIR", "2")
        assert np.array_equal(res.iterations, ref.iterations)
        assert torch.equal(res.u, ref.u)  # the schedule does not change any realization's bits


@pytest.mark.parametrize("n0,L,kind", [(4, 16, "lkr"), (4, 16, "fourier"), (4, 64, "lkr")])
def test_precomputed_diagonal_tiles_bitwise(monkeypatch, n0, L, kind):
    """Plans evaluate every middle-pass diagonal tile once (dtile_kernel) and the
    middle passes stream them; CHK_NO_DTILE=1 evaluates the same contraction per
    CTA.  Same formula, same order: identical bits (n = 64: register middle pass).
    n = 256 always uses the table (its register-phase middle pass reads it from
    L2), so there the two plans must simply agree."""
    from paper_2007_06524_b200.lowrank import _device_apply, _plan_for
    from paper_2007_06524_b200.solver import Preconditioner

    cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha="1/2", lam=0.1)
    B = 3 if L <= 16 else 1
    beta = np.stack([chk.sample_realization(cfg, chk.derive_seed(0, m)).beta_cells.ravel() for m in range(B)])
    A = chk.StiffnessBatch(cfg, beta)
    F = chk.corrector_rhs_batched(A, 1)
    opts = chk.SolveOptions(tol=1e-8, preconditioner=kind, eps_rank=1e-8)
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("CHK_NO_DTILE", flag)
        plan = _plan_for(3, cfg.n, kind, 1e-8 if kind == "lkr" else 0.0, 0.0)
        P = Preconditioner(kind, lambda x, p=plan: _device_apply(p, x), plan)
        r = chk.pcg_solve_batched(A, F, opts, P)
        assert np.all(r.status == 0)
        res[flag] = (r.iterations.copy(), r.u.clone(), P.apply(F))
    assert np.array_equal(res["0"][0], res["1"][0])
    assert torch.equal(res["0"][1], res["1"][1])
    assert torch.equal(res["0"][2], res["1"][2])
