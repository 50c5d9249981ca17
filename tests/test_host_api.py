"""Host-side logic and the C ABI surface (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, golden_small

import paper_2007_06524_b200 as chk
from paper_2007_06524_b200 import _lib


def _header_symbols():
    text = open(os.path.join(REPO, "include", "chk_pcg.h")).read()
    return sorted(set(re.findall(r"\b(chk_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    declared = _header_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes binding out of sync with chk_pcg.h"
    assert lib.chk_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_abi_rejects_bad_arguments_without_gpu():
    lib = _lib.load()
    h = ctypes.c_void_p()
    # n = 12 runs the generic kernels; 724 (> 720, not a power of two) and 10 (not n0 * L) do not exist
    assert lib.chk_precond_plan_create(1, 724, 5, None, None, 0.0, ctypes.byref(h)) == _lib.CHK_EUNSUPPORTED
    assert lib.chk_precond_plan_create(1, 10, 5, None, None, 0.0, ctypes.byref(h)) == _lib.CHK_EUNSUPPORTED
    assert lib.chk_precond_plan_create(1, 12, 5, None, None, 0.0, ctypes.byref(h)) == _lib.CHK_EINVAL  # no factors
    assert lib.chk_precond_plan_create(7, 16, 5, None, None, 0.0, ctypes.byref(h)) == _lib.CHK_EINVAL
    g = _lib.ChkGrid(2, 16, 4, 4, 2, 1, 0.4)
    assert lib.chk_stencil_apply(ctypes.byref(g), None, None, None, None, 1, None) == _lib.CHK_EUNSUPPORTED
    # n0 must be a power of two >= 4 (lattice.py:122-123); checked before any device work
    g2 = _lib.ChkGrid(3, 16, 8, 2, 2, 0, 0.4)
    assert lib.chk_stencil_apply(ctypes.byref(g2), None, None, None, None, 1, None) == _lib.CHK_EINVAL
    assert b">= 4" in lib.chk_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.CHK_EINVAL)
    assert lib.chk_pcg_workspace_bytes(ctypes.byref(g), None, 1, 10) == 0


def test_sampling_bit_identical_to_reference():
    g = golden_small()
    for m in range(256):
        assert chk.derive_seed(0, m) == int(g["seeds_master0"][m])
    cfg = chk.LatticeConfig(d=3, L=8, n0=4, alpha="1/2", lam=0.1)
    r = chk.sample_realization(cfg, chk.derive_seed(0, 0))
    assert np.array_equal(r.beta_cells, g["case6_beta"])
    cfg2 = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.2,
                             contrast=chk.ContrastModel.two_value(0.3, 0.7))
    assert np.array_equal(chk.sample_realization(cfg2, 5).beta_cells, g["case4_beta"])
    cfg3 = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/4", lam=0.2,
                             contrast=chk.ContrastModel.layered([0.1, 0.5, 0.8]), subcell_offset=0)
    assert np.array_equal(chk.sample_realization(cfg3, 6).beta_cells, g["case5_beta"])


def test_coefficient_grid_matches_reference():
    g = golden_small()
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/4", lam=0.4)
    r = chk.sample_realization(cfg, 2)
    grid = chk.coefficient_grid(r)
    assert isinstance(grid, chk.CoefficientGrid) and grid.n == cfg.n and grid.d == 3
    assert np.allclose(grid.values, g["case1_coef"], rtol=0, atol=1e-15)


def test_realization_reference_constructor():
    """Realization(config, covered, cell_beta, seed) as in lattice.py:208-227, and
    the lazily derived views agree with the dense sampler's."""
    cfg = chk.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.2,
                            contrast=chk.ContrastModel.two_value(0.3, 0.7))
    r = chk.sample_realization(cfg, 5)
    r2 = chk.Realization(cfg, r.covered, r.cell_beta, r.seed)
    assert r2 == r and r2.num_covered == r.num_covered
    assert np.array_equal(r2.beta_cells, r.beta_cells)
    assert np.array_equal(r2.covered_mask, r.covered_mask)
    assert r2.to_json() == r.to_json()
    assert chk.Realization.coerce(r2) is r2
    with pytest.raises(AttributeError):
        r2.seed = 1
    with pytest.raises(chk.ConfigurationError):
        chk.Realization(cfg, {(0, 0, 0)}, {}, 1)
    # duck-typed foreign realization (same fields as the reference's)
    class Foreign:
        config = cfg
        covered = r.covered
        cell_beta = r.cell_beta
        seed = r.seed
    assert chk.Realization.coerce(Foreign()) == r
    assert np.array_equal(chk.coefficient_grid(Foreign()).values, chk.coefficient_grid(r).values)


def test_spectral_api_matches_oracle():
    """eigensum_tensor / pseudoinverse_diag / regularized_inverse_diag
    (spectral.py:26-95) against the pinned oracle's diagonals."""
    from oracle import checkerhom_oracle as orc
    from paper_2007_06524_b200.spectral import _diag_kind

    for n in (8, 16):
        g = chk.eigensum_tensor(3, chk.fourier_eigenvalues(n))
        assert g.value((1, 2, 3)) == pytest.approx(g.array()[1, 2, 3])
        pinv = chk.pseudoinverse_diag(g)
        assert np.array_equal(pinv.values, orc.pseudoinverse_diag(n))
        reg = chk.regularized_inverse_diag(g, 1e-3)
        assert np.allclose(reg.values, orc.pseudoinverse_diag(n, delta=1e-3), rtol=1e-15, atol=0)
        assert chk.regularized_inverse_diag(g, 0.0).values is not None
        assert _diag_kind(pinv) == ("fourier", 0.0)
        assert _diag_kind(reg) == ("regularized", 1e-3)
        # a foreign object carrying only (d, n, values), e.g. the reference's dataclass
        Bare = type("Bare", (), {"d": 3, "n": n, "values": reg.values})
        kind, delta = _diag_kind(Bare())
        assert kind == "regularized" and delta == pytest.approx(1e-3, rel=1e-15)
        Other = type("Other", (), {"d": 3, "n": n, "values": np.ones((n, n, n))})
        with pytest.raises(ValueError):
            _diag_kind(Other())
    with pytest.raises(ValueError):
        chk.eigensum_tensor(4, chk.fourier_eigenvalues(8))


def test_philox_keys_are_the_reference_stream_keys():
    """The keys the device sampler consumes are those of
    Philox(SeedSequence(seed)) (lattice.py:279-281)."""
    seeds = [chk.derive_seed(0, m) for m in range(4)]
    keys = chk.philox_keys(seeds)
    for s, k in zip(seeds, keys):
        st = np.random.Philox(np.random.SeedSequence(s)).state
        assert np.array_equal(st["state"]["key"], k)
        assert not st["state"]["counter"].any() and st["buffer_pos"] == 4


def test_philox4x64_restatement_matches_numpy():
    """Pure-Python Philox4x64-10 with the counter / word mapping the CUDA sampler
    uses (chk_sample.cuh) reproduces Generator(Philox).random()."""
    M = (1 << 64) - 1

    def block(ctr, key):
        c = [ctr, 0, 0, 0]
        k = list(key)
        for r in range(10):
            if r:
                k = [(k[0] + 0x9E3779B97F4A7C15) & M, (k[1] + 0xBB67AE8584CAA73B) & M]
            p0, p1 = 0xD2E7470EE14C6C93 * c[0], 0xCA5A826395121157 * c[2]
            c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & M, (p0 >> 64) ^ c[3] ^ k[1], p0 & M]
        return c

    seed = chk.derive_seed(0, 7)
    key = [int(v) for v in chk.philox_keys([seed])[0]]
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed))).random(37)
    mine = [(block(i // 4 + 1, key)[i % 4] >> 11) * (1.0 / 9007199254740992.0) for i in range(37)]
    assert np.array_equal(ref, np.asarray(mine))


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512])
def test_device_plan_factors_bit_identical(n):
    """The factors the GPU plan consumes equal the reference setup's."""
    g = golden_small()
    t = chk.dc_correction(chk.canonical_reciprocal(chk.fourier_eigenvalues(n), 3, 1e-8))
    fac = np.stack(t.factors)
    if n <= 64:
        assert np.array_equal(fac, g[f"factors_n{n}"])
    else:
        assert np.array_equal(fac[0], g[f"factors_mode0_n{n}"])
        assert np.array_equal(fac[2, :-1], g[f"factors_mode0_n{n}"][:-1])


def test_solve_options_validation():
    with pytest.raises(chk.ConfigurationError):
        chk.SolveOptions(tol=0.0)
    with pytest.raises(chk.ConfigurationError):
        chk.SolveOptions(max_iter=0)
    with pytest.raises(chk.ConfigurationError):
        chk.SolveOptions(preconditioner="amg")
    with pytest.raises(chk.ConfigurationError):
        chk.SolveOptions(delta=-1.0)
    assert issubclass(chk.ConfigurationError, ValueError)


def test_lattice_validation():
    with pytest.raises(chk.ConfigurationError):
        chk.LatticeConfig(d=3, L=4, n0=6)
    with pytest.raises(chk.ConfigurationError):
        chk.LatticeConfig(d=3, L=4, n0=4, alpha="3/4")
    with pytest.raises(chk.ConfigurationError):
        chk.LatticeConfig(d=3, L=4, n0=4, lam=0.0)


def test_no_oracle_import_in_product():
    pkg = os.path.join(REPO, "paper_2007_06524_b200")
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith(".py"):
                text = open(os.path.join(root, fn)).read()
                assert "oracle" not in re.sub(r"#.*", "", text).split("\"\"\"")[-1] or "import oracle" not in text
                assert "from oracle" not in text and "import oracle" not in text


def test_vectorised_seed_hashing_is_numpy_seedsequence():
    """derive_seeds / philox_keys (the host work of the seeds pipeline, hashed for the whole
    batch at once) against numpy's SeedSequence and the reference's golden seeds."""
    from conftest import golden_small

    g = golden_small()
    assert np.array_equal(chk.derive_seeds(0, range(256)), g["seeds_master0"])
    assert np.array_equal(chk.derive_seeds(7, range(16)), g["seeds_master7"])
    for master in (0, 3, 2 ** 40 + 3, 12345678901234567890123):
        idx = list(range(40)) + [65536, 2 ** 31, 2 ** 32 - 1]
        ref = [chk.derive_seed(master, m) for m in idx]
        assert [int(v) for v in chk.derive_seeds(master, idx)] == ref
    assert int(chk.derive_seeds(5, [2 ** 32 + 1])[0]) == chk.derive_seed(5, 2 ** 32 + 1)  # numpy fallback
    rng = np.random.default_rng(3)
    seeds = [int(v) for v in rng.integers(0, 2 ** 63, size=200, dtype=np.uint64)] + [0, 1, 2 ** 32 - 1, 2 ** 32, 2 ** 64 - 1]
    ref = np.stack([np.random.SeedSequence(s).generate_state(2, np.uint64) for s in seeds])
    from paper_2007_06524_b200.lattice import philox_keys
    assert np.array_equal(philox_keys(seeds), ref)
