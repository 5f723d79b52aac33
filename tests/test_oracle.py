"""Pin the CPU oracle against the reference's own outputs (golden fixtures
made by oracle/make_golden.py from the unmodified implicitrk) and against the
known answers of the pieces the reference lacks (CPU only)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import rel


def test_tableaux(golden, oracle):
    for s in range(1, 6):
        t = oracle.radau(s)
        np.testing.assert_array_equal(t.A, golden[f"tab_radau{s}_A"])
        np.testing.assert_array_equal(t.b, golden[f"tab_radau{s}_b"])
    a = oracle.alexander()
    np.testing.assert_array_equal(a.A, golden["tab_alexander_A"])


@pytest.mark.parametrize("dim,n", [(2, 4), (2, 7)])
def test_q1_assembly_bit_exact(golden, oracle, dim, n):
    M, K = oracle.q1_matrices(n)
    for name, A in (("M", M), ("K", K)):
        key = f"asm{dim}d{n}_{name}"
        np.testing.assert_array_equal(A.indptr, golden[key + "_rowptr"])
        np.testing.assert_array_equal(A.indices, golden[key + "_col"])
        np.testing.assert_array_equal(A.data, golden[key + "_val"])
    np.testing.assert_array_equal(oracle.grid_boundary(dim, n), golden[f"asm{dim}d{n}_bd"])


@pytest.mark.parametrize("n", [5, 9])
def test_p1_1d_assembly_bit_exact(golden, oracle, n):
    M, K = oracle.p1_matrices(1, n)
    for name, A in (("M", M), ("K", K)):
        key = f"asm1d{n}_{name}"
        np.testing.assert_array_equal(A.indptr, golden[key + "_rowptr"])
        np.testing.assert_array_equal(A.indices, golden[key + "_col"])
        np.testing.assert_array_equal(A.data, golden[key + "_val"])


@pytest.mark.parametrize("dim,n,nnz", [(2, 4, 137), (2, 32, 7361), (3, 2, 223), (3, 4, 1333)])
def test_p1_known_answers(oracle, dim, n, nnz):
    M, K = oracle.p1_matrices(dim, n)
    m = (n + 1) ** dim
    assert M.nnz == K.nnz == nnz
    np.testing.assert_array_equal(M.indptr, K.indptr)
    np.testing.assert_array_equal(M.indices, K.indices)
    assert M.sum() == pytest.approx(1.0, abs=1e-14)          # total mass = |domain|
    assert np.abs(K @ np.ones(m)).max() < 1e-14               # constants in ker K
    assert abs(M - M.T).max() == 0 and abs(K - K.T).max() == 0
    h = 1.0 / n
    c = (n + 1) ** dim // 2  # an interior vertex
    row = K[c].toarray().ravel()
    if dim == 2:
        assert sorted(np.round(row[row != 0] , 12)) == [-1, -1, -1, -1, 4]
        assert M[c, c] == pytest.approx(h * h / 2)
    else:
        assert row[c] == pytest.approx(6 * h) and np.sum(np.isclose(row, -h)) == 6
        assert K[c].nnz == 15


def test_kron_apply(golden, oracle):
    for s, m in ((1, 5), (2, 8), (3, 6), (4, 5)):
        key = f"kron_s{s}m{m}"
        M = sp.csr_matrix(golden[key + "_M"])
        K = sp.csr_matrix(golden[key + "_K"])
        C1, C2, v = golden[key + "_C1"], golden[key + "_C2"], golden[key + "_v"]
        y = oracle.kron_apply(C1, C2, M, [K], 0.37, v)
        np.testing.assert_allclose(y, golden[key + "_y"], rtol=1e-13, atol=1e-12)
        Kl = [sp.csr_matrix(k) for k in golden[key + "_Kl"]]
        np.testing.assert_allclose(oracle.kron_apply(C1, C2, M, Kl, 0.37, v), golden[key + "_yl"],
                                   rtol=1e-13, atol=1e-12)
        idx = oracle.stage_index(s, m, [0, m - 1])
        op = lambda w: oracle.kron_apply(C1, C2, M, [K], 0.37, w)  # noqa: E731
        np.testing.assert_allclose(oracle.constrained(op, idx)(v), golden[key + "_yc"],
                                   rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("n", [6, 12, 30])
def test_fgmres(golden, oracle, n):
    A, b = golden[f"fgmres{n}_A"], golden[f"fgmres{n}_b"]
    x, its, hist = oracle.fgmres(lambda v: A @ v, b, rtol=1e-12, restart=5, maxit=200)
    assert its == int(golden[f"fgmres{n}_its"])
    np.testing.assert_allclose(x, golden[f"fgmres{n}_x"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(hist, golden[f"fgmres{n}_res"], rtol=1e-9)


@pytest.mark.parametrize("tname", ["radau3", "lobatto3"])
@pytest.mark.parametrize("kind", ["jacobi", "gs-lower", "gs-upper", "rana-ld", "rana-du"])
@pytest.mark.parametrize("form", ["ai", "ia"])
def test_preconditioners_exact_blocks(golden, oracle, tname, kind, form):
    key = f"pc_{tname}_{kind}_{form}"
    if key not in golden.files:
        pytest.skip("reference rejects this kind/form/tableau")
    n = 10
    M, K = oracle.p1_matrices(1, n)
    tab = oracle.radau(3) if tname == "radau3" else oracle.Tab(
        np.array([[1 / 6, -1 / 3, 1 / 6], [1 / 6, 5 / 12, -1 / 12], [1 / 6, 2 / 3, 1 / 6]]),
        np.array([1 / 6, 2 / 3, 1 / 6]), np.array([0.0, 0.5, 1.0]), "lobatto-iiic:3")
    pc = oracle.StagePC(kind, tab, M, [K], 0.05, form, oracle.grid_boundary(1, n), "lu")
    np.testing.assert_allclose(pc.apply(golden[f"pc_{tname}_v"]), golden[key], rtol=1e-10,
                               atol=1e-11)
    pcg = oracle.StagePC(kind, tab, M, [K], 0.05, form, oracle.grid_boundary(1, n), "pcg", 1e-13)
    assert rel(pcg.apply(golden[f"pc_{tname}_v"]), golden[key]) < 1e-10


def test_bc_stage_values(golden, oracle):
    tab = oracle.radau(3)
    u_b = np.array([0.3, -0.2])
    G = np.stack([np.array([np.sin(0.2 + c * 0.1), 1.0 + 0.2 + c * 0.1]) for c in tab.c])
    for unk in ("value", "w", "derivative"):
        np.testing.assert_allclose(oracle.stage_values(tab, u_b, G, 0.1, unk), golden[f"bc_{unk}"],
                                   rtol=1e-13)


@pytest.mark.parametrize("k,n", [(1, None), (2, 32), (3, 6), (4, 32), (5, 32)])
@pytest.mark.parametrize("block", ["lu", "pcg"])
def test_config_trajectories(golden, oracle, k, n, block):
    cfg = oracle.config(k, n, block)
    st = oracle.run_config(k, n, block=block)
    key = f"traj{k}_n{cfg['n']}"
    U = golden[key + "_u"]
    tol = 1e-12 if block == "lu" and k != 3 else 1e-9
    np.testing.assert_array_equal(cfg["problem"].u0, golden[key + "_u0"])
    assert rel(st.u, U[-1]) < tol
    if key + "_x" in golden.files:
        X = golden[key + "_x"]
        assert max(rel(a, b) for a, b in zip(st.stages, X)) < 1e-9


def test_schur_preconditioner_exactness(oracle):
    """With exact blocks and the FULL T the Schur preconditioner is exact
    (1 FGMRES iteration); block-diagonal T gives the survey's 2 iterations."""
    n = 4
    M, K = oracle.p1_matrices(3, n)
    tab = oracle.gauss(4)
    dofs = oracle.grid_boundary(3, n)
    s, m = tab.s, M.shape[0]
    rng = np.random.default_rng(0)
    b = rng.standard_normal(s * m)
    idx = oracle.stage_index(s, m, dofs)
    op = oracle.constrained(lambda v: oracle.kron_apply(np.eye(s), tab.A, M, [K], 5e-3, v), idx)
    pc = oracle.StagePC("schur", tab, M, [K], 5e-3, "ai", dofs, "lu")
    x, its, _ = oracle.fgmres(op, b, pc.apply, rtol=1e-12)
    assert its <= 3
    assert rel(op(x), b) < 1e-11


def test_sketch_detects_differences(oracle):
    rng = np.random.default_rng(1)
    v = rng.standard_normal(50000)
    P = oracle.sketch_rows(len(v))
    a, b = oracle.sketch(v, P), oracle.sketch(v * (1 + 1e-9), P)
    proj, samp = oracle.sketch_rel_err(b, a)
    assert 0.5e-9 < proj < 2e-9 and 0.5e-9 < samp < 2e-9
