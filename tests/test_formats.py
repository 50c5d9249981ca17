"""Wire formats around the solve against fixtures written by the reference
(tests/golden/make_golden.py formats): realization JSON (lattice.py:229-250)
byte for byte, and the trace.csv rows of the reference CLI (cli.py:264-287)."""

import json
import os

import numpy as np
import pytest

import paper_2007_06524_b200 as chk
from paper_2007_06524_b200 import formats
from paper_2007_06524_b200.solver import PcgReport

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "formats.json")))


@pytest.mark.parametrize("i", range(len(GOLD["realizations"])))
def test_realization_json_matches_reference(i):
    rec = GOLD["realizations"][i]
    cfg = chk.LatticeConfig.from_dict(rec["config_dict"])
    assert cfg.to_dict() == rec["config_dict"]
    r = chk.sample_realization(cfg, rec["seed"])
    assert r.to_json() == rec["json"]                      # identical bytes
    back = chk.Realization.from_json(rec["json"])
    assert back.to_json() == rec["json"]                   # round trip
    assert back.config == cfg and back.seed == rec["seed"]
    assert np.array_equal(back.beta_cells, r.beta_cells)
    assert back.covered == r.covered and back.num_covered == r.num_covered


def test_realization_json_keeps_zero_beta_covered_cells():
    cfg = chk.LatticeConfig(d=3, L=3, n0=4, alpha="1/2", lam=0.5,
                            contrast=chk.ContrastModel.two_value(0.0, 0.5))
    r = chk.sample_realization(cfg, 11)
    back = chk.Realization.from_json(r.to_json())
    assert back.covered == r.covered
    assert back.num_covered > np.count_nonzero(back.beta_cells)


def test_trace_csv_rows_match_reference_cli():
    t = GOLD["trace"]
    rep = PcgReport(iterations=t["iterations"], residuals=tuple(t["residuals"]), converged=True,
                    final_residual=t["residuals"][-1], preconditioner=t["preconditioner"])
    lines = formats.trace_csv_lines(rep)
    assert lines[0] == "iteration,rel_residual"
    assert lines[1:] == t["csv_rows"]


def test_write_trace_csv(tmp_path):
    rep = PcgReport(iterations=2, residuals=(0.5, 1e-9), converged=True, final_residual=1e-9,
                    preconditioner="fourier")
    formats.write_trace_csv(tmp_path / "trace.csv", rep, header_lines=["# command = solve"])
    assert (tmp_path / "trace.csv").read_text() == "# command = solve\niteration,rel_residual\n1,0.5\n2,1e-09\n"


@pytest.mark.gpu
def test_gpu_solve_trace_csv_matches_reference_trace():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    t = GOLD["trace"]
    cfg = chk.LatticeConfig.from_dict(t["config"])
    r = chk.sample_realization(cfg, t["seed"])
    A = chk.assemble_stiffness(r)
    f = (1.0 / cfg.n) ** (2 - 3) * chk.corrector_rhs(r, 1)
    u, rep = chk.pcg_solve(A, f, chk.SolveOptions(tol=1e-8, preconditioner="lkr"))
    assert rep.iterations == t["iterations"] and rep.preconditioner == t["preconditioner"]
    np.testing.assert_allclose(rep.residuals, t["residuals"], rtol=1e-7, atol=0)
    lines = formats.trace_csv_lines(rep)
    assert [l.split(",")[0] for l in lines[1:]] == [row.split(",")[0] for row in t["csv_rows"]]
