"""Generate golden fixtures from the REFERENCE package (build container only).

Imports the read-only reference ``checkerhom`` from /root/reference/pkg/src and
records its outputs for the hot path.  The fixtures pin both the CPU oracle
(oracle/checkerhom_oracle.py) and the CUDA path.  Run:

    python tests/golden/make_golden.py small            # -> tests/golden/small.npz
    python tests/golden/make_golden.py config 3 0 16    # -> tests/golden/config3_0_16.json
    python tests/golden/make_golden.py formats          # -> tests/golden/formats.json
    python tests/golden/make_golden.py pool 3 0 256 8   # -> tests/golden/config3_full.json
    python tests/golden/make_golden.py generic          # -> tests/golden/generic.npz (n = 12, 20, 24)

Large arrays are never committed: for configs 2-5 we keep iteration counts,
the full residual history, ||u||, <u, f>, <u, w> for a seeded Gaussian w and
u at 4096 seeded positions (see ``u_probe``).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import checkerhom as ch  # noqa: E402  (reference, read-only)
from checkerhom.solver import make_preconditioner  # noqa: E402
from checkerhom.spectral import regularized_inverse_diag  # noqa: E402

from oracle import checkerhom_oracle as orc  # noqa: E402

PROBE_SEED = 12345
PROJ_SEED = 777
N_PROBE = 4096


N_PROJ = 16          # independent Gaussian projections per record (pool mode)
N_PROBE_POOL = 512


def proj_vector(N: int, k: int) -> np.ndarray:
    """k-th projection vector w_k ~ N(0, I_N); E[(e.w_k)^2] = ||e||^2, so
    mean_k (u.w_k - u_ref.w_k)^2 estimates ||u - u_ref||^2 (16 draws: ~+-18 %
    on ||u - u_ref||)."""
    return np.random.default_rng([PROJ_SEED, k]).standard_normal(N)


def u_projections(u: np.ndarray) -> list:
    return [float(u @ proj_vector(u.size, k)) for k in range(N_PROJ)]


def u_probe(u: np.ndarray, f: np.ndarray) -> dict:
    N = u.size
    idx = np.random.default_rng(PROBE_SEED).integers(0, N, size=N_PROBE)
    w = np.random.default_rng(PROJ_SEED).standard_normal(N)
    return {
        "norm_u": float(np.linalg.norm(u)),
        "u_dot_f": float(u @ f),
        "u_dot_w": float(u @ w),
        "probe_idx_seed": PROBE_SEED,
        "proj_seed": PROJ_SEED,
        "u_probe": [float(v) for v in u[idx]],
        "sum_u": float(u.sum()),
    }


def ref_factors(n, d=3, eps=1e-8):
    t = ch.dc_correction(ch.canonical_reciprocal(ch.fourier_eigenvalues(n), d, eps))
    return np.stack(t.factors)


def small():
    out = {}
    out["seeds_master0"] = np.array([ch.derive_seed(0, m) for m in range(256)], dtype=np.uint64)
    out["seeds_master7"] = np.array([ch.derive_seed(7, m) for m in range(16)], dtype=np.uint64)
    # LKR factors as produced by the reference setup (consumed as-is by the GPU path)
    for n in (8, 16, 32, 64, 128, 256, 512):
        fac = ref_factors(n)
        if n <= 64:
            out[f"factors_n{n}"] = fac
        else:
            # rows 0..R-1 are identical across the three modes; the last row is
            # the dc fix (-origin at [0] on mode 0, 1 at [0] on modes 1, 2)
            assert np.array_equal(fac[0, :-1], fac[1, :-1]) and np.array_equal(fac[0, :-1], fac[2, :-1])
            assert np.count_nonzero(fac[1, -1]) == 1 and fac[1, -1, 0] == 1.0
            out[f"factors_mode0_n{n}"] = fac[0]
        out[f"eig_n{n}"] = ch.fourier_eigenvalues(n).values
    out["factors2d_n8"] = np.stack(ch.dc_correction(
        ch.canonical_reciprocal(ch.fourier_eigenvalues(8), 2, 1e-8)).factors)
    q = ch.exp_sum_quadrature(1.0, 12.0, 1e-8)
    out["quad_1_12_nodes"], out["quad_1_12_weights"] = q.nodes, q.weights

    # realizations -> beta cell arrays
    cases = []
    cfgs = [
        dict(d=3, L=2, n0=4, alpha="1/4", lam=0.4, seed=1),
        dict(d=3, L=4, n0=4, alpha="1/4", lam=0.4, seed=2),
        dict(d=3, L=4, n0=4, alpha="1/2", lam=0.1, seed=3),
        dict(d=3, L=2, n0=8, alpha="1/4", lam=0.3, seed=4),
        dict(d=3, L=4, n0=4, alpha="1/2", lam=0.2, seed=5,
             contrast=ch.ContrastModel.two_value(0.3, 0.7)),
        dict(d=3, L=4, n0=4, alpha="1/4", lam=0.2, seed=6,
             contrast=ch.ContrastModel.layered([0.1, 0.5, 0.8]), subcell_offset=0),
        dict(d=3, L=8, n0=4, alpha="1/2", lam=0.1, seed=int(out["seeds_master0"][0])),
        dict(d=3, L=8, n0=4, alpha="1/2", lam=0.01, seed=int(out["seeds_master0"][1])),
    ]
    rng = np.random.default_rng(2024)
    for ci, kw in enumerate(cfgs):
        kw = dict(kw)
        seed = kw.pop("seed")
        cfg = ch.LatticeConfig(**kw)
        r = ch.sample_realization(cfg, seed)
        L, d = cfg.L, cfg.d
        beta = np.zeros((L,) * d)
        for c, b in r.cell_beta.items():
            beta[c] = b
        A = ch.assemble_stiffness(r)
        n = cfg.n
        x = np.random.default_rng(1000 + ci).standard_normal(n ** d)
        y = A.matrix() @ x
        pre = f"case{ci}_"
        out[pre + "meta"] = np.array([d, L, cfg.n0, cfg.k, cfg.offset, seed % (2**62)], dtype=np.int64)
        out[pre + "lam"] = np.array(cfg.lam)
        out[pre + "beta"] = beta
        out[pre + "Ax"] = y
        for i in (1, 2, 3):
            out[pre + f"rhs{i}"] = ch.corrector_rhs(r, i)
        out[pre + "coef"] = ch.coefficient_grid(r).values
        print("case", ci, cfg.n, r.num_covered, flush=True)

    # preconditioner applies
    for n in (8, 16, 32):
        t = ch.dc_correction(ch.canonical_reciprocal(ch.fourier_eigenvalues(n), 3, 1e-8))
        x = rng.standard_normal(n ** 3)
        out[f"lkr_x_n{n}"] = x
        out[f"lkr_y_n{n}"] = ch.apply_lkr_preconditioner(t, x)
        gp = ch.pseudoinverse_diag(ch.eigensum_tensor(3, ch.fourier_eigenvalues(n)))
        out[f"fourier_y_n{n}"] = ch.apply_fourier_preconditioner(gp, x)
        rd = regularized_inverse_diag(ch.eigensum_tensor(3, ch.fourier_eigenvalues(n)), 1e-3)
        out[f"reg_y_n{n}"] = ch.apply_fourier_preconditioner(rd, x)

    # small PCG solves through the reference public API
    pcg_cases = [
        dict(L=2, n0=4, alpha="1/4", lam=0.4, seed=0, tol=1e-7, pre="lkr"),
        dict(L=4, n0=4, alpha="1/4", lam=0.4, seed=1, tol=1e-7, pre="lkr"),
        dict(L=4, n0=4, alpha="1/4", lam=0.4, seed=2, tol=1e-10, pre="fourier"),
        dict(L=4, n0=4, alpha="1/2", lam=0.1, seed=3, tol=1e-9, pre="regularized"),
        dict(L=4, n0=4, alpha="1/2", lam=0.1, seed=4, tol=1e-9, pre="lkr", prs=True),
        dict(L=4, n0=4, alpha="1/4", lam=0.4, seed=5, tol=1e-30, pre="lkr", max_iter=3),
    ]
    for pi, kw in enumerate(pcg_cases):
        cfg = ch.LatticeConfig(d=3, L=kw["L"], n0=kw["n0"], alpha=kw["alpha"], lam=kw["lam"])
        r = ch.sample_realization(cfg, kw["seed"])
        A = ch.assemble_stiffness(r)
        h = 1.0 / cfg.n
        f = (h ** (2 - 3)) * ch.corrector_rhs(r, 1)
        opts = ch.SolveOptions(tol=kw["tol"], preconditioner=kw["pre"], eps_rank=1e-8,
                               delta=1e-3 if kw["pre"] == "regularized" else 0.0,
                               precond_residual_stopping=kw.get("prs", False),
                               max_iter=kw.get("max_iter", 500))
        u, rep = ch.pcg_solve(A, f, opts)
        beta = np.zeros((cfg.L,) * 3)
        for c, b in r.cell_beta.items():
            beta[c] = b
        pre = f"pcg{pi}_"
        out[pre + "meta"] = np.array([cfg.L, cfg.n0, cfg.k, cfg.offset, rep.iterations,
                                      int(rep.converged), int(kw.get("prs", False)),
                                      kw.get("max_iter", 500)], dtype=np.int64)
        out[pre + "lam_tol"] = np.array([cfg.lam, kw["tol"]])
        out[pre + "kind"] = np.array(kw["pre"])
        out[pre + "beta"] = beta
        out[pre + "f"] = f
        out[pre + "u"] = u
        out[pre + "res"] = np.array(rep.residuals)
        out[pre + "name"] = np.array(rep.preconditioner)
        print("pcg", pi, rep.iterations, rep.converged, rep.preconditioner, flush=True)

    # homogenized matrices (homogenize.py:92-124), d = 3
    homog = [
        dict(L=2, n0=4, alpha="1/4", lam=0.4, seed=11, tol=1e-8),
        dict(L=4, n0=4, alpha="1/2", lam=0.1, seed=12, tol=1e-8),
        dict(L=4, n0=4, alpha="1/4", lam=0.2, seed=13, tol=1e-9),
    ]
    for hi, kw in enumerate(homog):
        cfg = ch.LatticeConfig(d=3, L=kw["L"], n0=kw["n0"], alpha=kw["alpha"], lam=kw["lam"])
        r = ch.sample_realization(cfg, kw["seed"])
        rec = ch.homogenized_matrix(r, ch.SolveOptions(tol=kw["tol"], preconditioner="lkr"))
        pre = f"homog{hi}_"
        out[pre + "meta"] = np.array([cfg.L, cfg.n0, cfg.k, cfg.offset, kw["seed"]], dtype=np.int64)
        out[pre + "lam_tol"] = np.array([cfg.lam, kw["tol"]])
        out[pre + "matrix"] = rec.matrix
        out[pre + "its"] = np.array(rec.iterations)
        print("homog", hi, rec.iterations, flush=True)

    # config 1 (n=32): full u for m = 0, 1
    for m in (0, 1):
        rec, u, f = config_run(1, m)
        out[f"cfg1_m{m}_u"] = u
        out[f"cfg1_m{m}_res"] = np.array(rec["residuals"])
        out[f"cfg1_m{m}_its"] = np.array(rec["iterations"])
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("wrote small.npz", os.path.getsize(os.path.join(HERE, "small.npz")))


def config_run(cfg_id: int, m: int, compact: bool = False):
    c = orc.CONFIGS[cfg_id]
    seed = ch.derive_seed(0, m)
    cfg = ch.LatticeConfig(d=3, L=c["L"], n0=c["n0"], alpha="1/2", lam=c["lam"])
    r = ch.sample_realization(cfg, seed)
    n = cfg.n
    h = 1.0 / n
    t0 = time.perf_counter()
    if cfg_id == 5:
        beta = np.zeros((cfg.L,) * 3)
        for cc, b in r.cell_beta.items():
            beta[cc] = b
        k, off = cfg.k, cfg.offset
        F = orc.cell_field(beta, cfg.n0, k, off)

        class MF:
            d = 3

        A = MF()
        A.n = n
        sm = orc.StencilMatrix(F, cfg.lam)
        A.matrix = lambda: sm
        del F
    else:
        A = ch.assemble_stiffness(r)
        A.matrix()
    t_asm = time.perf_counter() - t0
    if c["rhs"] == "corrector":
        f = (h ** (2 - 3)) * ch.corrector_rhs(r, 1)
    else:
        f = np.random.default_rng(seed).standard_normal(n ** 3)
        f -= f.mean()
    opts = ch.SolveOptions(tol=c["tol"], preconditioner="lkr", eps_rank=1e-8)
    P = make_preconditioner(3, n, opts)
    t0 = time.perf_counter()
    u, rep = ch.pcg_solve(A, f, opts, precond=P)
    t_solve = time.perf_counter() - t0
    rec = {"config": cfg_id, "m": m, "seed": str(seed), "n": n,
           "iterations": rep.iterations, "converged": rep.converged,
           "residuals": list(rep.residuals), "final_residual": rep.final_residual,
           "preconditioner": rep.preconditioner, "rhs_projected": rep.rhs_projected,
           "norm_f": float(np.linalg.norm(f)), "num_covered": r.num_covered,
           "t_assembly_s": t_asm, "t_solve_s": t_solve}
    rec.update(u_probe(u, f))
    if compact:
        rec["u_probe"] = rec["u_probe"][:N_PROBE_POOL]
        rec["u_proj"] = u_projections(u)
        rec["n_proj"] = N_PROJ
        return rec, None, None
    return rec, u, f


def configs(cfg_id: int, start: int, count: int):
    recs = []
    path = os.path.join(HERE, f"config{cfg_id}_{start}_{count}.json")
    for m in range(start, start + count):
        rec, _, _ = config_run(cfg_id, m)
        recs.append(rec)
        print(cfg_id, m, rec["iterations"], rec["t_solve_s"], flush=True)
        with open(path, "w") as fh:
            json.dump({"generator": "tests/golden/make_golden.py (reference checkerhom)",
                       "numpy": np.__version__, "records": recs}, fh, indent=1)


def _pool_one(args):
    cfg_id, m = args
    rec, _, _ = config_run(cfg_id, m, compact=True)
    return rec


def pool(cfg_id: int, start: int, count: int, workers: int):
    """Every realization of a BASELINE config through the reference, one per
    worker process (the pattern of homogenize.py:149-161), compact records
    with N_PROJ projections each -> config{cfg}_full.json."""
    from concurrent.futures import ProcessPoolExecutor
    path = os.path.join(HERE, f"config{cfg_id}_full.json")
    recs = {}
    if os.path.exists(path):
        recs = {r["m"]: r for r in json.load(open(path))["records"]}
    todo = [m for m in range(start, start + count) if m not in recs]
    with ProcessPoolExecutor(max_workers=workers) as ex:
        for rec in ex.map(_pool_one, [(cfg_id, m) for m in todo]):
            recs[rec["m"]] = rec
            print(cfg_id, rec["m"], rec["iterations"], round(rec["t_solve_s"], 1), flush=True)
            with open(path + ".tmp", "w") as fh:
                json.dump({"generator": "tests/golden/make_golden.py pool (reference checkerhom)",
                           "numpy": np.__version__, "n_proj": N_PROJ, "proj_seed": PROJ_SEED,
                           "records": [recs[k] for k in sorted(recs)]}, fh)
            os.replace(path + ".tmp", path)


def generic():
    """Grid sizes that are not powers of two (n = n0 * L, any L; lattice.py:117-123):
    the reference's own tests use n = 12 and 24.  Stiffness products, corrector
    loads, the three preconditioner applies and pcg_solve runs -> generic.npz."""
    out = {}
    cfgs = [
        dict(d=3, L=3, n0=4, alpha="1/4", lam=0.4, seed=21),                       # n = 12
        dict(d=3, L=3, n0=8, alpha="1/4", lam=0.4, seed=22, subcell_offset=1),     # n = 24
        dict(d=3, L=5, n0=4, alpha="1/2", lam=0.1, seed=23,
             contrast=ch.ContrastModel.layered([0.1, 0.5, 0.8])),                    # n = 20
    ]
    for ci, kw in enumerate(cfgs):
        kw = dict(kw)
        seed = kw.pop("seed")
        cfg = ch.LatticeConfig(**kw)
        r = ch.sample_realization(cfg, seed)
        beta = np.zeros((cfg.L,) * 3)
        for c, b in r.cell_beta.items():
            beta[c] = b
        A = ch.assemble_stiffness(r)
        x = np.random.default_rng(3000 + ci).standard_normal(cfg.n ** 3)
        pre = f"case{ci}_"
        out[pre + "meta"] = np.array([3, cfg.L, cfg.n0, cfg.k, cfg.offset, seed], dtype=np.int64)
        out[pre + "lam"] = np.array(cfg.lam)
        out[pre + "beta"] = beta
        out[pre + "Ax"] = A.matrix() @ x
        for i in (1, 2, 3):
            out[pre + f"rhs{i}"] = ch.corrector_rhs(r, i)
        print("generic case", ci, cfg.n, r.num_covered, flush=True)
    rng = np.random.default_rng(2025)
    for n in (12, 20):
        t = ch.dc_correction(ch.canonical_reciprocal(ch.fourier_eigenvalues(n), 3, 1e-8))
        x = rng.standard_normal(n ** 3)
        out[f"lkr_x_n{n}"] = x
        out[f"lkr_y_n{n}"] = ch.apply_lkr_preconditioner(t, x)
        gp = ch.pseudoinverse_diag(ch.eigensum_tensor(3, ch.fourier_eigenvalues(n)))
        out[f"fourier_y_n{n}"] = ch.apply_fourier_preconditioner(gp, x)
        rd = regularized_inverse_diag(ch.eigensum_tensor(3, ch.fourier_eigenvalues(n)), 1e-3)
        out[f"reg_y_n{n}"] = ch.apply_fourier_preconditioner(rd, x)
        out[f"factors_n{n}"] = np.stack(t.factors)
    pcg_cases = [
        dict(L=3, n0=4, alpha="1/2", lam=0.1, seed=31, tol=1e-8, pre="lkr"),                     # n = 12
        dict(L=3, n0=8, alpha="1/4", lam=0.4, seed=32, tol=1e-8, pre="lkr", off=1),              # n = 24
        dict(L=5, n0=4, alpha="1/2", lam=0.05, seed=33, tol=1e-10, pre="fourier", rhs="noise"),  # n = 20
        dict(L=6, n0=4, alpha="1/2", lam=0.01, seed=34, tol=1e-9, pre="regularized"),            # n = 24
        dict(L=3, n0=4, alpha="1/4", lam=0.4, seed=35, tol=1e-9, pre="lkr", prs=True),           # n = 12
        dict(L=7, n0=4, alpha="1/2", lam=0.1, seed=36, tol=1e-30, pre="lkr", max_iter=4),        # n = 28
    ]
    for pi, kw in enumerate(pcg_cases):
        cfg = ch.LatticeConfig(d=3, L=kw["L"], n0=kw["n0"], alpha=kw["alpha"], lam=kw["lam"],
                               subcell_offset=kw.get("off"))
        r = ch.sample_realization(cfg, kw["seed"])
        A = ch.assemble_stiffness(r)
        h = 1.0 / cfg.n
        if kw.get("rhs") == "noise":
            # a load with a non-zero mean: pcg_solve projects it (solver.py:139-143)
            f = np.random.default_rng(kw["seed"]).standard_normal(cfg.n ** 3) + 0.25
        else:
            f = (h ** (2 - 3)) * ch.corrector_rhs(r, 1)
        opts = ch.SolveOptions(tol=kw["tol"], preconditioner=kw["pre"], eps_rank=1e-8,
                               delta=1e-3 if kw["pre"] == "regularized" else 0.0,
                               precond_residual_stopping=kw.get("prs", False),
                               max_iter=kw.get("max_iter", 500))
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            u, rep = ch.pcg_solve(A, f, opts)
        beta = np.zeros((cfg.L,) * 3)
        for c, b in r.cell_beta.items():
            beta[c] = b
        pre = f"pcg{pi}_"
        out[pre + "meta"] = np.array([cfg.L, cfg.n0, cfg.k, cfg.offset, rep.iterations, int(rep.converged),
                                      int(kw.get("prs", False)), kw.get("max_iter", 500),
                                      int(rep.rhs_projected)], dtype=np.int64)
        out[pre + "lam_tol"] = np.array([cfg.lam, kw["tol"]])
        out[pre + "kind"] = np.array(kw["pre"])
        out[pre + "beta"] = beta
        out[pre + "f"] = f
        out[pre + "u"] = u
        out[pre + "res"] = np.array(rep.residuals)
        out[pre + "name"] = np.array(rep.preconditioner)
        print("generic pcg", pi, cfg.n, rep.iterations, rep.converged, rep.preconditioner, rep.rhs_projected, flush=True)
    # homogenized matrix at n = 12 (homogenize.py:92-124)
    cfg = ch.LatticeConfig(d=3, L=3, n0=4, alpha="1/2", lam=0.1)
    r = ch.sample_realization(cfg, 41)
    rec = ch.homogenized_matrix(r, ch.SolveOptions(tol=1e-8, preconditioner="lkr"))
    out["homog0_meta"] = np.array([cfg.L, cfg.n0, cfg.k, cfg.offset, 41], dtype=np.int64)
    out["homog0_lam_tol"] = np.array([cfg.lam, 1e-8])
    out["homog0_matrix"] = rec.matrix
    out["homog0_its"] = np.array(rec.iterations)
    print("generic homog", rec.iterations, flush=True)
    np.savez_compressed(os.path.join(HERE, "generic.npz"), **out)
    print("wrote generic.npz", os.path.getsize(os.path.join(HERE, "generic.npz")))


def formats():
    """Wire formats around the path: realization JSON
    (lattice.py:229-250) for every contrast kind / offset, and the CSV cell
    formatting of cli.py:264-267,281-287 applied to a pcg_solve trace."""
    cases = [
        dict(d=3, L=4, n0=4, alpha="1/2", lam=0.1),
        dict(d=3, L=3, n0=8, alpha="1/4", lam=0.4, subcell_offset=1),
        dict(d=3, L=4, n0=4, alpha="1/2", lam=0.2, contrast=ch.ContrastModel.two_value(0.3, 0.7)),
        dict(d=3, L=5, n0=4, alpha="1/4", lam=0.4, contrast=ch.ContrastModel.layered([0.1, 0.5, 0.2])),
        dict(d=2, L=6, n0=4, alpha="1/2", lam=0.5, coverage_prob=0.3),
    ]
    recs = []
    for i, kw in enumerate(cases):
        cfg = ch.LatticeConfig(**kw)
        r = ch.sample_realization(cfg, ch.derive_seed(3, i))
        recs.append({"config_dict": cfg.to_dict(), "seed": int(r.seed), "json": r.to_json()})
    cfg = ch.LatticeConfig(d=3, L=4, n0=4, alpha="1/2", lam=0.1)
    r = ch.sample_realization(cfg, ch.derive_seed(0, 0))
    A = ch.assemble_stiffness(r)
    f = (1.0 / cfg.n) ** (2 - 3) * ch.corrector_rhs(r, 1)
    u, rep = ch.pcg_solve(A, f, ch.SolveOptions(tol=1e-8, preconditioner="lkr"))
    from checkerhom.cli import _fmt
    rows = [",".join(_fmt(v) for v in row) for row in enumerate(rep.residuals, start=1)]
    doc = {"generator": "tests/golden/make_golden.py formats (reference checkerhom)",
           "realizations": recs,
           "trace": {"config": cfg.to_dict(), "seed": int(r.seed), "iterations": rep.iterations,
                     "residuals": [float(x) for x in rep.residuals], "csv_rows": rows,
                     "preconditioner": rep.preconditioner}}
    with open(os.path.join(HERE, "formats.json"), "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "small":
        small()
    elif sys.argv[1] == "formats":
        formats()
    elif sys.argv[1] == "generic":
        generic()
    elif sys.argv[1] == "pool":
        pool(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
    else:
        configs(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
