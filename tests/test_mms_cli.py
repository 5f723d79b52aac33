"""Manufactured-solution layer and experiment CLI (SURVEY §8 f rows 2-3),
against fixtures recorded from the unmodified reference
(tests/golden/reference_mms.npz, oracle/make_golden.py mms)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, rel


@pytest.fixture(scope="module")
def mg():
    return np.load(GOLDEN / "reference_mms.npz")


# ------------------------------------------------------------ CPU (no GPU)


def test_cli_parser_matches_reference_interface():
    from paper_2403_08084_b200 import cli

    ap = cli.build_parser()
    a = ap.parse_args(["converge"])
    assert (a.mode, a.cfl, a.tfinal, a.nx, a.n_list, a.dt_list, a.problem) == (
        "spatial", 4.0, 1.0, 32, [8, 16, 32, 64], [0.2, 0.1, 0.05, 0.025], "dahlquist")
    assert (a.tableau, a.stage_type, a.splitting, a.pc, a.rtol, a.out) == (
        "radau-iia:2", "deriv", "ai", "rana-ld", 1e-8, "out.csv")
    b = ap.parse_args(["precond-bench"])
    assert (b.splitting, b.nx, b.dt, b.steps) == ("ia", 64, None, 16)
    c = ap.parse_args(["bc-compare"])
    assert (c.tableau, c.nx, c.dt, c.tfinal, c.out) == ("lobatto-iiic:3", 10, 0.05, 0.5,
                                                         "bc-compare")


def test_cli_tableau_and_config_errors(capsys):
    from paper_2403_08084_b200 import cli

    assert cli.main(["tableau", "--tableau", "radau-iia:3"]) == 0
    out = capsys.readouterr().out
    assert "stiffly accurate : True" in out and "B(5) residual" in out
    assert cli.main(["tableau", "--tableau", "nosuch:3"]) == 2
    assert cli.main(["precond-bench", "--pc", "none"]) == 2


# ------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(1, 10), (2, 8)])
def test_load_vector_matches_reference(cuda, mg, dim, n):
    from paper_2403_08084_b200 import problems as pb

    grid = pb.StructuredGrid(dim, n)
    mms = pb.heat_mms_2d() if dim == 2 else pb.heat_mms_1d()
    # host-evaluated forcing: same f values as the reference, same
    # accumulation order on the device -> bitwise equal
    f_host = lambda t, *x: mms.f(t, *x)  # noqa: E731
    ref = mg[f"load{dim}d"]
    assert np.array_equal(pb.assemble_load(grid, f_host, 0.3), ref)
    # built-in forcing evaluated on the device (device sin/cos)
    assert rel(pb.assemble_load(grid, mms.f, 0.3), ref) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(1, 10), (2, 8)])
def test_error_norms_match_reference(cuda, mg, dim, n):
    from paper_2403_08084_b200 import problems as pb

    grid = pb.StructuredGrid(dim, n)
    mms = pb.heat_mms_2d() if dim == 2 else pb.heat_mms_1d()
    uh = mg[f"uh{dim}d"]
    assert abs(pb.l2_error(grid, uh, mms.u, 0.3) / mg[f"l2_{dim}d"] - 1) < 1e-12
    assert abs(pb.h1_error(grid, uh, mms.u, mms.grad, 0.3) / mg[f"h1_{dim}d"] - 1) < 1e-12
    assert abs(pb.fe_l2_norm(grid, uh) / mg[f"norm_{dim}d"] - 1) < 1e-12


@pytest.mark.gpu
def test_mms_trajectory_matches_reference(cuda, mg):
    import paper_2403_08084_b200 as irk

    grid = irk.StructuredGrid(2, 8)
    prob = irk.mms_heat_problem(grid)
    st = irk.TimeStepper(prob, irk.radau_iia(2), 0.1, krylov=irk.KrylovSettings(rtol=1e-12),
                         pc_kind=irk.PreconditionerKind.RANA_LD)
    u, reps = irk.advance(st, prob, 0.5)
    assert len(reps) == 5
    assert rel(u, mg["mms_u"]) < 1e-9
    mms = irk.heat_mms_2d()
    assert abs(irk.l2_error(grid, u, mms.u, 0.5) / mg["mms_l2"] - 1) < 1e-8
    assert abs(irk.h1_error(grid, u, mms.u, mms.grad, 0.5) / mg["mms_h1"] - 1) < 1e-8


@pytest.mark.gpu
def test_cli_sweeps_match_reference(cuda, mg, tmp_path):
    from paper_2403_08084_b200 import cli

    conv = tmp_path / "conv.csv"
    assert cli.main(["converge", "--mode", "spatial", "--n-list", "4", "8", "--tfinal", "0.2",
                     "--rtol", "1e-12", "--out", str(conv)]) == 0
    assert conv.read_text().splitlines()[0] == "N,L2err,H1err"
    got = np.loadtxt(conv, delimiter=",", skiprows=1)
    assert np.array_equal(got[:, 0], mg["cli_converge"][:, 0])
    assert rel(got[:, 1:], mg["cli_converge"][:, 1:]) < 1e-8

    temp = tmp_path / "temp.csv"
    assert cli.main(["converge", "--mode", "temporal", "--problem", "dahlquist", "--dt-list",
                     "0.2", "0.1", "--tfinal", "1.0", "--out", str(temp)]) == 0
    got = np.genfromtxt(temp, delimiter=",", skip_header=1)
    ref = mg["cli_temporal"]
    assert rel(got[:, :2], ref[:, :2]) < 1e-9
    assert np.isnan(got[0, 2]) and abs(got[1, 2] - ref[1, 2]) < 1e-3

    bc = tmp_path / "bc"
    assert cli.main(["bc-compare", "--nx", "6", "--dt", "0.1", "--tfinal", "0.3", "--rtol",
                     "1e-12", "--out", str(bc)]) == 0
    for name, key in (("daenorm.csv", "cli_dae"), ("odenorm.csv", "cli_ode")):
        got = np.loadtxt(bc / name, delimiter=",", skiprows=1)
        assert rel(got, mg[key]) < 1e-9


@pytest.mark.gpu
def test_cli_precond_bench_runs(cuda, tmp_path):
    from paper_2403_08084_b200 import cli

    out = tmp_path / "pb.csv"
    assert cli.main(["precond-bench", "--nx", "16", "--steps", "2", "--out", str(out)]) == 0
    rows = np.loadtxt(out, delimiter=",", skiprows=1)
    assert out.read_text().splitlines()[0] == "ns,time,Its"
    assert rows.shape == (4, 3) and np.all(rows[:, 2] >= 1)
    dout = tmp_path / "dirk.csv"
    assert cli.main(["precond-bench", "--stage-type", "dirk", "--nx", "16", "--steps", "2",
                     "--out", str(dout)]) == 0
    assert np.loadtxt(dout, delimiter=",", skiprows=1).shape == (3, 3)


@pytest.mark.gpu
def test_cli_solver_failure_exit_3(cuda, tmp_path, monkeypatch):
    """NonConvergenceError -> exit code 3 (cli.py:358-360): FGMRES capped at
    2 iterations cannot reach rtol 1e-12 on bc-compare's 40-cell problem."""
    from paper_2403_08084_b200 import cli
    from paper_2403_08084_b200.sparsela import KrylovSettings

    monkeypatch.setattr(cli, "KrylovSettings",
                        lambda **kw: KrylovSettings(**{**kw, "maxit": 2}))
    assert cli.main(["bc-compare", "--rtol", "1e-12", "--nx", "40",
                     "--out", str(tmp_path / "x")]) == 3


@pytest.mark.gpu
def test_cli_dirk_rows_count_one_iteration_per_stage(cuda, tmp_path):
    """precond-bench --stage-type dirk reports one FGMRES-equivalent
    iteration per stage, as the reference's exact-factor FGMRES does
    (pkg/tests/test_cli.py:140-149)."""
    from paper_2403_08084_b200 import cli

    out = tmp_path / "dirk.csv"
    assert cli.main(["precond-bench", "--stage-type", "dirk", "--nx", "16", "--steps", "3",
                     "--out", str(out)]) == 0
    rows = np.loadtxt(out, delimiter=",", skiprows=1)
    assert np.all(rows[:, 2] == 1.0)
