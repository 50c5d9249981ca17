"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures in tests/golden/ come from tests/golden/make_golden.py, which
imports the reference ``checkerhom`` package; nothing here reads
/root/reference at run time.
"""

import json
import os

import numpy as np
import pytest

from oracle import checkerhom_oracle as orc

from conftest import GOLDEN_DIR, golden_small


def test_derive_seed_matches_reference():
    g = golden_small()
    for m in range(256):
        assert orc.derive_seed(0, m) == int(g["seeds_master0"][m])
    for m in range(16):
        assert orc.derive_seed(7, m) == int(g["seeds_master7"][m])


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512])
def test_lkr_factors_bit_identical(n):
    """canonical_reciprocal + dc_correction restatement vs reference (lowrank.py:147-180)."""
    g = golden_small()
    fac = orc.lkr_factors(n)
    assert np.array_equal(orc.fourier_eigenvalues(n), g[f"eig_n{n}"])
    if n <= 64:
        ref = g[f"factors_n{n}"]
        assert np.array_equal(np.stack(fac), ref)
    else:
        ref0 = g[f"factors_mode0_n{n}"]
        assert np.array_equal(fac[0], ref0)
        assert np.array_equal(fac[1][:-1], ref0[:-1])
        assert fac[1][-1, 0] == 1.0 and np.count_nonzero(fac[1][-1]) == 1


def test_lkr_rank_law():
    # R+1 = 66/69/72/75/78 for n = 32..512 at eps 1e-8
    for n, r1 in ((32, 66), (64, 69), (128, 72), (256, 75), (512, 78)):
        assert orc.lkr_factors(n)[0].shape[0] == r1


def test_quadrature_reference_interval():
    g = golden_small()
    nodes, weights = orc.exp_sum_quadrature(1.0, 12.0, 1e-8)
    assert np.array_equal(nodes, g["quad_1_12_nodes"])
    assert np.array_equal(weights, g["quad_1_12_weights"])


def _cases():
    g = golden_small()
    return sorted({k.split("_")[0] for k in g.files if k.startswith("case")})


@pytest.mark.parametrize("case", _cases())
def test_sampling_stencil_rhs(case):
    """Realization sampling, CSR stiffness (tests/oracles.py:35-82) and the
    corrector RHS (homogenize.py:75-89) against the reference."""
    g = golden_small()
    d, L, n0, k, off, _ = (int(v) for v in g[case + "_meta"])
    lam = float(g[case + "_lam"])
    beta = g[case + "_beta"]
    F = orc.cell_field(beta, n0, k, off)
    n = n0 * L
    ci = int(case[4:])
    x = np.random.default_rng(1000 + ci).standard_normal(n ** d)
    y = orc.stencil_apply(F, lam, x)
    ref = g[case + "_Ax"]
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
    assert np.allclose(orc.coefficient_grid(F), g[case + "_coef"], rtol=0, atol=1e-15)
    for i in (1, 2, 3):
        f = orc.corrector_rhs(F, i)
        assert np.allclose(f, g[case + f"_rhs{i}"], rtol=0, atol=1e-17)


def test_sampling_matches_reference_beta():
    g = golden_small()
    # case6 / case7 were drawn with the config-1 seeds (fixed contrast)
    for case, m, lam in (("case6", 0, 0.1), ("case7", 1, 0.01)):
        beta = orc.sample_beta_cells(8, lam, orc.derive_seed(0, m))
        assert np.array_equal(beta, g[case + "_beta"])
    # two_value (case4) and layered (case5)
    b4 = orc.sample_beta_cells(4, 0.2, 5, contrast="two_value", betas=(0.3, 0.7))
    assert np.array_equal(b4, g["case4_beta"])
    b5 = orc.sample_beta_cells(4, 0.2, 6, contrast="layered", betas=(0.1, 0.5, 0.8))
    assert np.array_equal(b5, g["case5_beta"])


@pytest.mark.parametrize("n", [8, 16, 32])
def test_preconditioner_applies(n):
    g = golden_small()
    x = g[f"lkr_x_n{n}"]
    y = orc.apply_lkr(orc.lkr_factors(n), x)
    ref = g[f"lkr_y_n{n}"]
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
    yf = orc.apply_fourier(orc.pseudoinverse_diag(n), x)
    assert np.linalg.norm(yf - g[f"fourier_y_n{n}"]) <= 1e-14 * np.linalg.norm(yf)
    yr = orc.apply_fourier(orc.pseudoinverse_diag(n, delta=1e-3), x)
    assert np.linalg.norm(yr - g[f"reg_y_n{n}"]) <= 1e-14 * np.linalg.norm(yr)


def _pcg_ids():
    g = golden_small()
    return sorted({k.split("_")[0] for k in g.files if k.startswith("pcg")})


@pytest.mark.parametrize("pid", _pcg_ids())
def test_oracle_pcg_small(pid):
    g = golden_small()
    L, n0, k, off, its, conv, prs, max_iter = (int(v) for v in g[pid + "_meta"])
    lam, tol = (float(v) for v in g[pid + "_lam_tol"])
    kind = str(g[pid + "_kind"])
    F = orc.cell_field(g[pid + "_beta"], n0, k, off)
    f = g[pid + "_f"]
    assert np.allclose(orc.pcg_rhs_corrector(F, 1), f, rtol=0, atol=1e-16)
    n = n0 * L
    if kind == "lkr":
        fac = orc.lkr_factors(n)
        dg = orc.lkr_diagonal(fac)
        P = lambda x: orc.apply_lkr(fac, x, dg)  # noqa: E731
    else:
        dg = orc.pseudoinverse_diag(n, delta=1e-3 if kind == "regularized" else 0.0)
        P = lambda x: orc.apply_fourier(dg, x)  # noqa: E731
    A = orc.StencilMatrix(F, lam)
    u, rep = orc.pcg_solve(A.__matmul__, f, P, tol=tol, max_iter=max_iter,
                           precond_residual_stopping=bool(prs))
    assert rep.iterations == its
    assert rep.converged == bool(conv)
    ref_res = g[pid + "_res"]
    assert np.allclose(rep.residuals, ref_res, rtol=1e-8, atol=0)
    uref = g[pid + "_u"]
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)


@pytest.mark.parametrize("m", [0, 1])
def test_oracle_config1(m):
    g = golden_small()
    u, rep = orc.solve_config(1, m)
    assert rep.iterations == int(g[f"cfg1_m{m}_its"])
    assert np.allclose(rep.residuals, g[f"cfg1_m{m}_res"], rtol=1e-8, atol=0)
    uref = g[f"cfg1_m{m}_u"]
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)


def test_oracle_config2_first_realization():
    path = os.path.join(GOLDEN_DIR, "config2_0_64.json")
    if not os.path.exists(path):
        pytest.skip("config-2 golden not generated")
    rec = json.load(open(path))["records"][0]
    u, rep = orc.solve_config(2, 0)
    assert rep.iterations == rec["iterations"]
    assert np.allclose(rep.residuals, rec["residuals"], rtol=1e-8, atol=0)
    assert abs(np.linalg.norm(u) - rec["norm_u"]) <= 1e-9 * rec["norm_u"]


# ---- grid sizes that are not powers of two (generic.npz: n = 12, 20, 24, 28) -------------
def _generic_ids(prefix):
    from conftest import golden_generic
    g = golden_generic()
    return sorted({k.split("_")[0] for k in g.files if k.startswith(prefix)})


@pytest.mark.parametrize("case", _generic_ids("case"))
def test_oracle_generic_stencil_rhs(case):
    from conftest import golden_generic
    g = golden_generic()
    d, L, n0, k, off, _ = (int(v) for v in g[case + "_meta"])
    F = orc.cell_field(g[case + "_beta"], n0, k, off)
    n = n0 * L
    x = np.random.default_rng(3000 + int(case[4:])).standard_normal(n ** 3)
    ref = g[case + "_Ax"]
    assert np.linalg.norm(orc.stencil_apply(F, float(g[case + "_lam"]), x) - ref) <= 1e-14 * np.linalg.norm(ref)
    for i in (1, 2, 3):
        assert np.allclose(orc.corrector_rhs(F, i), g[case + f"_rhs{i}"], rtol=0, atol=1e-17)


@pytest.mark.parametrize("n", [12, 20])
def test_oracle_generic_preconditioners(n):
    from conftest import golden_generic
    g = golden_generic()
    x = g[f"lkr_x_n{n}"]
    fac = orc.lkr_factors(n)
    assert np.array_equal(fac, g[f"factors_n{n}"])
    ref = g[f"lkr_y_n{n}"]
    assert np.linalg.norm(orc.apply_lkr(fac, x) - ref) <= 1e-14 * np.linalg.norm(ref)
    yf = orc.apply_fourier(orc.pseudoinverse_diag(n), x)
    assert np.linalg.norm(yf - g[f"fourier_y_n{n}"]) <= 1e-14 * np.linalg.norm(yf)
    yr = orc.apply_fourier(orc.pseudoinverse_diag(n, delta=1e-3), x)
    assert np.linalg.norm(yr - g[f"reg_y_n{n}"]) <= 1e-14 * np.linalg.norm(yr)


@pytest.mark.parametrize("pid", _generic_ids("pcg"))
def test_oracle_generic_pcg(pid):
    from conftest import golden_generic
    g = golden_generic()
    L, n0, k, off, its, conv, prs, max_iter, proj = (int(v) for v in g[pid + "_meta"])
    lam, tol = (float(v) for v in g[pid + "_lam_tol"])
    kind = str(g[pid + "_kind"])
    F = orc.cell_field(g[pid + "_beta"], n0, k, off)
    n = n0 * L
    if kind == "lkr":
        fac = orc.lkr_factors(n)
        dg = orc.lkr_diagonal(fac)
        P = lambda x: orc.apply_lkr(fac, x, dg)  # noqa: E731
    else:
        dg = orc.pseudoinverse_diag(n, delta=1e-3 if kind == "regularized" else 0.0)
        P = lambda x: orc.apply_fourier(dg, x)  # noqa: E731
    A = orc.StencilMatrix(F, lam)
    u, rep = orc.pcg_solve(A.__matmul__, g[pid + "_f"], P, tol=tol, max_iter=max_iter,
                           precond_residual_stopping=bool(prs))
    assert rep.iterations == its and rep.converged == bool(conv)
    assert np.allclose(rep.residuals, g[pid + "_res"], rtol=1e-8, atol=0)
    uref = g[pid + "_u"]
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
