"""Time stepping on the GPU vs the reference (goldens), dense oracles and the
reference test-suite's analytic known answers (gpu)."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def irk(cuda):
    import paper_2403_08084_b200 as irk

    return irk


AI = "STAGE_DERIVATIVE_AI"


def build(irk, oracle, k, n, inner_rtol=1e-6):
    """The CUDA twin of oracle.config(k, n): same grid, seeds, tableau, BCs."""
    cfg = oracle.config(k, n)
    p = cfg["problem"]
    grid = irk.structured_grid(cfg["dim"], cfg["n"])
    if k == 5:
        prob = irk.allen_cahn_problem(grid, 0.02, p.u0)
    else:
        g = None
        if k == 3:
            g = lambda t, x, y, z: np.exp(-t) * np.sin(np.pi * x)  # noqa: E731
        prob = irk.heat_problem(grid, p.u0, g=g)
        np.testing.assert_array_equal(prob.u0, p.u0)
    tab = {1: irk.radau_iia(2), 2: irk.radau_iia(3), 3: irk.gauss_legendre(4),
           4: irk.alexander_dirk(), 5: irk.radau_iia(3)}[k]
    st = cfg["settings"]
    form = {"ai": irk.StageFormulation.STAGE_DERIVATIVE_AI, "value": irk.StageFormulation.STAGE_VALUE,
            "dirk": irk.StageFormulation.DIRK}[st["form"]]
    pc = {"jacobi": irk.PreconditionerKind.BLOCK_DIAGONAL, "gs-lower": irk.PreconditionerKind.BLOCK_LOWER,
          "schur": irk.PreconditionerKind.SCHUR, None: None}[st["pc"]]
    kw = dict(formulation=form, krylov=irk.KrylovSettings(rtol=st["rtol"]), pc_kind=pc,
              block_solver=irk.BlockSolveSettings(rtol=inner_rtol))
    if k == 5:
        kw["newton"] = irk.NewtonSettings(rtol=1e-10, atol=1e-10)
    return prob, irk.TimeStepper(prob, tab, cfg["dt"], **kw), cfg


@pytest.mark.parametrize("k,n", [(1, None), (2, 32), (3, 6), (4, 32), (5, 32)])
def test_config_trajectory_vs_reference(irk, oracle, golden, k, n):
    prob, st, cfg = build(irk, oracle, k, n)
    key = f"traj{k}_n{cfg['n']}"
    U = golden[key + "_u"]
    X = golden[key + "_x"] if key + "_x" in golden.files else None
    worst_u = worst_x = 0.0
    for i in range(cfg["steps"]):
        u, rep = st.step(prob)
        worst_u = max(worst_u, rel(u, U[i]))
        if X is not None:
            worst_x = max(worst_x, rel(st.stage_vectors, X[i]))
    assert worst_u < 1e-9, worst_u
    assert worst_x < 1e-9, worst_x
    assert X is not None, "every config golden records the reference's stage vectors"
    assert worst_x > 0.0


# ------------------------------------------- reference-suite known answers


def scalar(irk, kval, u0=1.0):
    return irk.SemidiscreteProblem(m=1, mass=irk.SparseMatrix.from_dense([[1.0]]),
                                   stiffness=irk.SparseMatrix.from_dense([[kval]]),
                                   load=lambda t: np.zeros(1), u0=np.array([u0]))


TIGHT = dict(rtol=1e-13, atol=1e-14, maxit=400)


def test_backward_euler_halves(irk):
    st = irk.TimeStepper(scalar(irk, 1.0), irk.radau_iia(1), 1.0, krylov=irk.KrylovSettings(**TIGHT))
    assert st.step()[0][0] == pytest.approx(0.5, abs=1e-13)


def test_radau2_stability_function(irk):
    st = irk.TimeStepper(scalar(irk, 1.0), irk.radau_iia(2), 1.0, krylov=irk.KrylovSettings(**TIGHT))
    assert st.step()[0][0] == pytest.approx(4.0 / 11.0, abs=1e-12)


@pytest.mark.parametrize("form", ["STAGE_DERIVATIVE_AI", "STAGE_DERIVATIVE_IA", "STAGE_VALUE"])
def test_zero_dynamics_identity(irk, form):
    st = irk.TimeStepper(scalar(irk, 0.0, 1.7), irk.radau_iia(2), 0.5,
                         formulation=getattr(irk.StageFormulation, form),
                         krylov=irk.KrylovSettings(**TIGHT))
    u, rep = st.step()
    assert u[0] == pytest.approx(1.7, abs=1e-11)


def test_midpoint_value_recombination(irk):
    mid = irk.gauss_legendre(1)
    for form in (irk.StageFormulation.STAGE_VALUE, irk.StageFormulation.STAGE_DERIVATIVE_AI):
        st = irk.TimeStepper(scalar(irk, 1.0), mid, 1.0, formulation=form,
                             krylov=irk.KrylovSettings(**TIGHT))
        assert st.step()[0][0] == pytest.approx(1 / 3, abs=1e-12)


def test_radau2_heat_vs_dense(irk):
    grid = irk.StructuredGrid(1, 4)
    M, K, _ = irk.assemble_heat(grid)
    u0 = np.sin(np.pi * grid.coords()[:, 0])
    p = irk.SemidiscreteProblem(m=grid.npoints, mass=M, stiffness=K, load=lambda t: np.zeros(5), u0=u0)
    tab, dt = irk.radau_iia(2), 0.1
    u1, _ = irk.TimeStepper(p, tab, dt, krylov=irk.KrylovSettings(**TIGHT)).step()
    S = np.kron(np.eye(2), M.to_dense()) + dt * np.kron(tab.A, K.to_dense())
    k = np.linalg.solve(S, np.concatenate([-K.to_dense() @ u0] * 2)).reshape(2, 5)
    np.testing.assert_allclose(u1, u0 + dt * (tab.b @ k), atol=1e-11)


def incompatible_heat(irk, n):
    grid = irk.StructuredGrid(1, n)
    M, K, bd = irk.assemble_heat(grid)
    bc = irk.DirichletBC(dofs=bd, g=lambda t: np.ones(2), g_dot=lambda t: np.zeros(2))
    return irk.SemidiscreteProblem(m=grid.npoints, mass=M, stiffness=K,
                                   load=lambda t: np.zeros(grid.npoints), dirichlet=bc,
                                   u0=np.zeros(grid.npoints))


def test_formulation_equivalence(irk):
    p = incompatible_heat(irk, 16)
    res = {}
    for f in ("STAGE_DERIVATIVE_AI", "STAGE_DERIVATIVE_IA", "STAGE_VALUE"):
        st = irk.TimeStepper(p, irk.radau_iia(3), 0.1, formulation=getattr(irk.StageFormulation, f),
                             krylov=irk.KrylovSettings(rtol=1e-10),
                             pc_kind=irk.PreconditionerKind.RANA_LD)
        res[f], _ = irk.advance(st, p, 0.5)
    nrm = np.linalg.norm(res["STAGE_DERIVATIVE_AI"])
    for a in res.values():
        for b in res.values():
            assert np.linalg.norm(a - b) <= 10 * 1e-10 * nrm
    np.testing.assert_allclose(res["STAGE_VALUE"][[0, -1]], 1.0, atol=1e-10)


def test_stiffly_accurate_value_update_bit_exact(irk):
    from paper_2403_08084_b200 import stepper as stp

    p = incompatible_heat(irk, 8)
    tab = irk.radau_iia(2)
    st = irk.TimeStepper(p, tab, 0.1, formulation=irk.StageFormulation.STAGE_VALUE,
                         krylov=irk.KrylovSettings(rtol=1e-10), pc_kind=irk.PreconditionerKind.RANA_LD)
    op, rhs = stp._stage_value_system(p, tab, st.t, st.dt, st.u)
    x, _ = stp._solve_constrained(st, p, op, rhs, irk.StageUnknown.VALUE, st.t)
    u1, _ = st.step(p)
    assert np.array_equal(u1, x.reshape(tab.s, p.m)[-1])


def test_dirk_matches_coupled(irk):
    p = incompatible_heat(irk, 8)
    t = irk.KrylovSettings(rtol=1e-12)
    s1 = irk.TimeStepper(p, irk.alexander_dirk(), 0.1, formulation=irk.StageFormulation.DIRK, krylov=t)
    s2 = irk.TimeStepper(p, irk.alexander_dirk(), 0.1, krylov=t, pc_kind=irk.PreconditionerKind.BLOCK_LOWER)
    for _ in range(3):
        u1, _ = s1.step(p)
        u2, _ = s2.step(p)
    assert np.linalg.norm(u1 - u2) <= 1e-10 * max(1.0, np.linalg.norm(u1))


def test_warm_start_and_reproducibility(irk):
    p = incompatible_heat(irk, 16)
    kw = dict(krylov=irk.KrylovSettings(rtol=1e-10), pc_kind=irk.PreconditionerKind.RANA_LD)
    cold1, _ = irk.advance(irk.TimeStepper(p, irk.radau_iia(2), 0.05, **kw), p, 0.3)
    cold2, _ = irk.advance(irk.TimeStepper(p, irk.radau_iia(2), 0.05, **kw), p, 0.3)
    assert np.array_equal(cold1, cold2)  # deterministic reductions: bit-for-bit
    warm, _ = irk.advance(irk.TimeStepper(p, irk.radau_iia(2), 0.05, warm_start=True, **kw), p, 0.3)
    assert np.linalg.norm(warm - cold1) < 1e-8


def test_riccati_newton(irk):
    case = irk.riccati()
    tab, dt = irk.radau_iia(2), 0.1
    st = irk.TimeStepper(case.problem, tab, dt, krylov=irk.KrylovSettings(**TIGHT),
                         newton=irk.NewtonSettings(rtol=1e-13, atol=1e-14))
    u1, rep = st.step(case.problem)
    k = np.zeros(2)
    for _ in range(60):
        ui = 1.0 + dt * (tab.A @ k)
        R = k - ui**2
        if np.linalg.norm(R) < 1e-14:
            break
        k = k - np.linalg.solve(np.eye(2) - dt * np.diag(2 * ui) @ tab.A, R)
    assert u1[0] == pytest.approx(1.0 + dt * (tab.b @ k), abs=1e-10)


@pytest.mark.parametrize("form", ["STAGE_DERIVATIVE_AI", "STAGE_DERIVATIVE_IA", "STAGE_VALUE"])
def test_riccati_formulations(irk, form):
    case = irk.riccati()
    st = irk.TimeStepper(case.problem, irk.radau_iia(3), 0.05,
                         formulation=getattr(irk.StageFormulation, form),
                         krylov=irk.KrylovSettings(**TIGHT), newton=irk.NewtonSettings(rtol=1e-13, atol=1e-14))
    u, _ = irk.advance(st, case.problem, 0.5)
    assert u[0] == pytest.approx(case.exact(0.5), abs=2e-8)


def test_nonlinear_dirk(irk):
    case = irk.riccati()
    st = irk.TimeStepper(case.problem, irk.alexander_dirk(), 0.02, formulation=irk.StageFormulation.DIRK,
                         krylov=irk.KrylovSettings(**TIGHT))
    u, _ = irk.advance(st, case.problem, 0.2)
    assert u[0] == pytest.approx(case.exact(0.2), abs=5e-6)


def test_cubic_reaction_semilinear_vs_dense_newton(irk):
    """Device semilinear Newton vs a dense stacked Newton (recipe of
    tests/test_stepper.py:282-334: M u' + K u + M u^3 = load)."""
    grid = irk.StructuredGrid(1, 12)
    M, K, _ = irk.assemble_heat(grid)
    m = grid.npoints
    x = grid.coords()[:, 0]
    load = np.sin(np.pi * x)
    prob = irk.SemidiscreteProblem(m=m, mass=M, stiffness=K, load=lambda t: load,
                                   u0=0.5 * np.sin(np.pi * x),
                                   semilinear=irk.SemilinearForm(1.0, (0.0, 0.0, 0.0, 1.0)))
    tab, dt = irk.radau_iia(2), 0.05
    for kind in (irk.PreconditionerKind.BLOCK_DIAGONAL, irk.PreconditionerKind.RANA_LD):
        st = irk.TimeStepper(prob, tab, dt, krylov=irk.KrylovSettings(**TIGHT),
                             newton=irk.NewtonSettings(rtol=1e-13, atol=1e-14), pc_kind=kind,
                             block_solver=irk.BlockSolveSettings(rtol=1e-10))
        u1, rep = st.step(prob)
        assert 2 <= rep.newton_iters <= 8
        Md, Kd = M.to_dense(), K.to_dense()
        k = np.zeros((2, m))
        for _ in range(60):
            U = prob.u0[None, :] + dt * (tab.A @ k)
            R = np.stack([Md @ k[i] + Kd @ U[i] + Md @ U[i] ** 3 - load for i in range(2)])
            if np.linalg.norm(R) < 1e-13:
                break
            J = np.zeros((2 * m, 2 * m))
            for i in range(2):
                Ki = Kd + Md @ np.diag(3 * U[i] ** 2)
                for j in range(2):
                    J[i * m:(i + 1) * m, j * m:(j + 1) * m] = dt * tab.A[i, j] * Ki + (Md if i == j else 0)
            k = k - np.linalg.solve(J, R.ravel()).reshape(2, m)
        np.testing.assert_allclose(u1, prob.u0 + dt * (tab.b @ k), atol=1e-10)


def test_newton_divergence_and_step_failure(irk):
    case = irk.riccati()
    st = irk.TimeStepper(case.problem, irk.radau_iia(1), 0.3, krylov=irk.KrylovSettings(**TIGHT),
                         newton=irk.NewtonSettings(maxit=20))
    with np.errstate(over="ignore", invalid="ignore"):
        with pytest.raises(irk.NonlinearDivergenceError) as err:
            st.step(case.problem)
    assert len(err.value.residuals) > 5
    st = irk.TimeStepper(case.problem, irk.radau_iia(1), 0.2, krylov=irk.KrylovSettings(**TIGHT),
                         newton=irk.NewtonSettings(maxit=10))
    with np.errstate(over="ignore", invalid="ignore"):
        with pytest.raises(irk.StepFailure) as err:
            irk.advance(st, case.problem, 1.0)
    assert 1 <= err.value.completed_steps < 5


def test_advance_and_clock(irk):
    case = irk.dahlquist(-1.0)
    st = irk.TimeStepper(case.problem, irk.radau_iia(2), 0.3, krylov=irk.KrylovSettings(**TIGHT))
    u, reps = irk.advance(st, case.problem, 1.0)
    assert len(reps) == 4 and st.t == pytest.approx(1.0, abs=1e-12) and st.dt == 0.3
    assert abs(u[0] - np.exp(-1.0)) < 5e-4
    st = irk.TimeStepper(case.problem, irk.radau_iia(3), 0.1, krylov=irk.KrylovSettings(**TIGHT))
    u, _ = irk.advance(st, case.problem, 1.0)
    assert abs(u[0] - np.exp(-1.0)) < 1e-9
    with pytest.raises(ValueError):
        irk.advance(irk.TimeStepper(case.problem, irk.radau_iia(1), 0.1, t0=1.0), case.problem, 0.5)


def test_wsodirk433_dirk_path_vs_dense_stages(irk):
    """WSODIRK433 (tableaux.py:257-277) through the device DIRK path on a
    Dirichlet 1D heat problem: every stage derivative and the state against
    a dense stage-by-stage solve (the reference's DIRK recurrence,
    stepper.py:391-421), 3 steps."""
    grid = irk.StructuredGrid(1, 12)
    M, K, bd = irk.assemble_heat(grid)
    x = grid.coords()[:, 0]
    u0 = np.sin(np.pi * x) + 0.3 * x * (1 - x)
    u0[bd] = 0.0
    p = irk.SemidiscreteProblem(m=grid.npoints, mass=M, stiffness=K,
                                load=lambda t: np.zeros(grid.npoints),
                                dirichlet=irk.DirichletBC(dofs=bd, g=lambda t: np.zeros(2)), u0=u0)
    tab, dt = irk.wsodirk433(), 0.05
    st = irk.TimeStepper(p, tab, dt, formulation=irk.StageFormulation.DIRK,
                         krylov=irk.KrylovSettings(rtol=1e-13, atol=1e-15))
    Md, Kd = M.to_dense(), K.to_dense()
    u = u0.copy()
    interior = np.setdiff1d(np.arange(grid.npoints), bd)
    for _ in range(3):
        ks = np.zeros((tab.s, grid.npoints))
        for i in range(tab.s):
            acc = u + dt * (tab.A[i, :i] @ ks[:i])
            S = Md + dt * tab.A[i, i] * Kd
            rhs = -Kd @ acc
            ks[i, interior] = np.linalg.solve(S[np.ix_(interior, interior)], rhs[interior])
        u = u + dt * (tab.b @ ks)
        un, rep = st.step(p)
        assert rel(un, u) < 1e-11
        assert rel(st.stage_vectors, ks.ravel()) < 1e-11
        assert rep.krylov_iters == tab.s and len(rep.inner_iters) == tab.s


def test_matrix_market_round_trip(irk, tmp_path):
    """mm_write / mm_read (sparsela.py:410-416): coordinate real general
    banner, pattern bit-exact (explicit zeros of the P1 stiffness kept),
    values exact; a symmetric-format file written by scipy reads back whole."""
    import scipy.io

    M, K, _ = irk.assemble_p1(irk.StructuredGrid(2, 6))
    path = tmp_path / "k.mtx"
    irk.mm_write(path, K)
    assert path.read_text().splitlines()[0].startswith("%%MatrixMarket matrix coordinate real general")
    back = irk.mm_read(path)
    np.testing.assert_array_equal(back.row_offsets, K.row_offsets)
    np.testing.assert_array_equal(back.col_indices, K.col_indices)
    np.testing.assert_array_equal(back.values, K.values)
    sym = tmp_path / "m_sym.mtx"
    scipy.io.mmwrite(str(sym), M.to_scipy(), symmetry="symmetric")
    np.testing.assert_array_equal(irk.mm_read(sym).to_dense(), M.to_dense())
