"""CUDA path vs the oracle / reference goldens: assembly, stage operator,
Krylov building blocks, inner block solvers and preconditioners (gpu)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def irk(cuda):
    import paper_2403_08084_b200 as irk

    return irk


# ------------------------------------------------------------------ assembly


@pytest.mark.parametrize("dim,n", [(1, 5), (1, 9), (2, 4), (2, 7)])
def test_reference_assembly_bit_exact(irk, golden, dim, n):
    """assemble_heat (1D P1 / 2D Q1) reproduces the reference bit for bit."""
    M, K, bd = irk.assemble_heat(irk.structured_grid(dim, n))
    for name, A in (("M", M), ("K", K)):
        key = f"asm{dim}d{n}_{name}"
        np.testing.assert_array_equal(A.row_offsets, golden[key + "_rowptr"])
        np.testing.assert_array_equal(A.col_indices, golden[key + "_col"])
        np.testing.assert_array_equal(A.values, golden[key + "_val"])
    np.testing.assert_array_equal(bd, golden[f"asm{dim}d{n}_bd"])


@pytest.mark.parametrize("dim,n", [(1, 7), (2, 4), (2, 32), (2, 129), (3, 2), (3, 5), (3, 12),
                                   (2, 1024), (3, 96), (2, 2048)])
def test_p1_assembly_vs_oracle(irk, oracle, dim, n):
    """Indices bit-exact (as int64), values to 1 ulp-scale -- also at the
    BASELINE config grids (1024^2: configs 2/5, 96^3: config 3, 2048^2:
    config 4), as north_star asks for the workloads themselves."""
    M, K, bd = irk.assemble_p1(irk.structured_grid(dim, n))
    Mo, Ko = oracle.p1_matrices(dim, n)
    for A, B in ((M, Mo), (K, Ko)):
        np.testing.assert_array_equal(A.row_offsets, B.indptr.astype(np.int64))
        np.testing.assert_array_equal(A.col_indices, B.indices.astype(np.int64))
        np.testing.assert_allclose(A.values, B.data, rtol=4e-16, atol=4e-16 * np.abs(B.data).max())
    np.testing.assert_array_equal(bd, oracle.grid_boundary(dim, n))


def test_p1_config_sizes(irk):
    """nnz = m + 2 #edges at the config grids."""
    for dim, n, m, nnz in ((2, 1024, 1050625, 7346177), (3, 96, 912673, 13465441),
                           (2, 2048, 4198401, 29372417)):
        M, K, bd = irk.assemble_p1(irk.structured_grid(dim, n))
        assert M.nrows == m and M.nnz == nnz and K.nnz == nnz
        assert M.device().same_pattern(K.device())


def test_sparse_matrix_roundtrip_and_validation(irk):
    A = sp.random(30, 30, density=0.2, random_state=1, format="csr") + sp.eye(30)
    S = irk.SparseMatrix.from_scipy(A)
    x = np.random.default_rng(0).standard_normal(30)
    np.testing.assert_allclose(irk.spmv(S, x), A @ x, rtol=1e-14, atol=1e-14)
    with pytest.raises(ValueError):
        irk.spmv(S, np.ones(29))
    with pytest.raises(ValueError):
        irk.SparseMatrix(2, 2, [0, 2, 2], [1, 0], [1.0, 2.0])  # decreasing columns


def test_dirichlet_constrain(irk):
    A = np.array([[4.0, -1, 0], [-1, 4, -1], [0, -1, 4]])
    C = irk.dirichlet_constrain(irk.SparseMatrix.from_dense(A), [0])
    expect = A.copy()
    expect[0, :] = expect[:, 0] = 0
    expect[0, 0] = 1
    np.testing.assert_array_equal(C.to_dense(), expect)
    with pytest.raises(ValueError):
        irk.dirichlet_constrain(irk.SparseMatrix.identity(3), [7])


# ------------------------------------------------------------- stage apply


@pytest.mark.parametrize("s,m", [(1, 5), (2, 8), (3, 6), (4, 5)])
def test_kronecker_apply_vs_reference(irk, golden, s, m):
    key = f"kron_s{s}m{m}"
    M = irk.SparseMatrix.from_dense(golden[key + "_M"])
    K = irk.SparseMatrix.from_dense(golden[key + "_K"])
    C1, C2, v = golden[key + "_C1"], golden[key + "_C2"], golden[key + "_v"]
    op = irk.KroneckerStageOperator(C1, C2, M, [K], 0.37)
    y = op.apply(v)
    np.testing.assert_allclose(y, golden[key + "_y"], rtol=0, atol=1e-12 * max(1, np.abs(y).max()))
    Kl = [irk.SparseMatrix.from_dense(k) for k in golden[key + "_Kl"]]
    yl = irk.KroneckerStageOperator(C1, C2, M, Kl, 0.37).apply(v)
    np.testing.assert_allclose(yl, golden[key + "_yl"], rtol=0, atol=1e-12 * max(1, np.abs(yl).max()))
    yc = irk.ConstrainedStageOperator(op, [0, m - 1]).apply(v)
    np.testing.assert_allclose(yc, golden[key + "_yc"], rtol=0, atol=1e-12 * max(1, np.abs(yc).max()))
    np.testing.assert_allclose(op.to_dense() @ v, golden[key + "_y"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5])
def test_stage_apply_p1_vs_oracle(irk, oracle, s):
    n = 40
    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    Mo, Ko = oracle.p1_matrices(2, n)
    tab = irk.radau_iia(s)
    rng = np.random.default_rng(s)
    v = rng.standard_normal(s * M.nrows)
    for C1, C2 in ((np.eye(s), tab.A), (np.linalg.inv(tab.A), np.eye(s))):
        op = irk.KroneckerStageOperator(C1, C2, M, [K], 1e-3)
        ref = oracle.kron_apply(C1, C2, Mo, [Ko], 1e-3, v)
        assert rel(op.apply(v), ref) < 1e-14
        idx = oracle.stage_index(s, M.nrows, bd)
        refc = oracle.constrained(lambda w: oracle.kron_apply(C1, C2, Mo, [Ko], 1e-3, w), idx)(v)
        assert rel(irk.ConstrainedStageOperator(op, bd).apply(v), refc) < 1e-14


def test_semilinear_jacobian_apply(irk, oracle):
    """Fused Jacobian stage apply == KroneckerStageOperator with explicit
    per-stage Jacobians kscale K + M diag(D_i) (stepper.py:550-551)."""
    import torch

    from paper_2403_08084_b200 import stepper as stp
    from paper_2403_08084_b200 import sparsela as la

    n, s, dt, ks = 24, 3, 1e-3, 0.02 ** 2
    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    m = M.nrows
    tab = irk.radau_iia(s)
    rng = np.random.default_rng(3)
    D = rng.uniform(-1, 2, size=(s, m))
    Ks = [irk.SparseMatrix.from_scipy(ks * K.to_scipy() + M.to_scipy() @ sp.diags(D[i])) for i in range(s)]
    v = rng.standard_normal(s * m)
    ref = irk.KroneckerStageOperator(np.eye(s), tab.A, M, Ks, dt).apply(v)
    Md, Kd = la.shared_pattern([M.device(), K.device()])
    Dil = la.to_dev(D.T.copy().ravel())
    op = stp._SemilinearJacobianOp(np.eye(s), tab.A, dt, Md, Kd, ks, Dil, None, m, s)
    x = la.to_dev(v.reshape(s, m).T.copy().ravel())
    out = la.dev_empty(m * s)
    op.dev_apply(x, out)
    got = out.cpu().numpy().reshape(m, s).T.ravel()
    assert rel(got, ref) < 1e-13
    # masked variant against the constrained reference form
    mask = la.dof_mask(m, bd)
    opm = stp._SemilinearJacobianOp(np.eye(s), tab.A, dt, Md, Kd, ks, Dil, mask, m, s)
    opm.dev_apply(x, out)
    refc = irk.ConstrainedStageOperator(irk.KroneckerStageOperator(np.eye(s), tab.A, M, Ks, dt), bd).apply(v)
    assert rel(out.cpu().numpy().reshape(m, s).T.ravel(), refc) < 1e-13
    assert torch.isfinite(out).all()


# ------------------------------------------------------------------ FGMRES


@pytest.mark.parametrize("n", [6, 12, 30])
def test_fgmres_vs_reference(irk, golden, n):
    A, b = golden[f"fgmres{n}_A"], golden[f"fgmres{n}_b"]
    res = irk.fgmres(A, b, settings=irk.KrylovSettings(rtol=1e-12, restart=5, maxit=200))
    np.testing.assert_allclose(res.x, golden[f"fgmres{n}_x"], rtol=1e-10, atol=1e-11)
    assert abs(res.iterations - int(golden[f"fgmres{n}_its"])) <= 1
    assert res.residuals[-1] <= 1e-12 * np.linalg.norm(b)


def test_fgmres_behaviours(irk):
    # identity -> 1 iteration; zero rhs -> 0; x0 exact -> 0; non-finite rejected
    b = np.arange(1.0, 6.0)
    r = irk.fgmres(np.eye(5), b)
    assert r.iterations == 1
    np.testing.assert_allclose(r.x, b, atol=1e-12)
    r = irk.fgmres(np.eye(4), np.zeros(4))
    assert r.iterations == 0 and np.all(r.x == 0)
    r = irk.fgmres(np.diag([2.0, 4.0]), np.array([2.0, 4.0]), x0=np.array([1.0, 1.0]))
    assert r.iterations == 0
    with pytest.raises(ValueError):
        irk.fgmres(np.eye(2), np.array([1.0, np.nan]))
    rng = np.random.default_rng(6)
    A = rng.standard_normal((40, 40)) + 2 * np.eye(40)
    with pytest.raises(irk.NonConvergenceError) as err:
        irk.fgmres(A, rng.standard_normal(40), settings=irk.KrylovSettings(rtol=1e-14, maxit=3, restart=2))
    assert len(err.value.residuals) >= 3
    # exact inverse as a (host callable) preconditioner -> 1 iteration
    A = rng.standard_normal((8, 8)) + 8 * np.eye(8)
    Ainv = np.linalg.inv(A)
    assert irk.fgmres(A, rng.standard_normal(8), pc=lambda v: Ainv @ v).iterations == 1
    # left preconditioning and restarts
    A = rng.standard_normal((25, 25)) + 12 * np.eye(25)
    b = rng.standard_normal(25)
    r = irk.fgmres(A, b, settings=irk.KrylovSettings(rtol=1e-10, restart=4, maxit=500))
    assert np.linalg.norm(b - A @ r.x) <= 1e-9 * np.linalg.norm(b)
    P = np.diag(1 / np.diag(A))
    r = irk.fgmres(A, b, pc=lambda v: P @ v, settings=irk.KrylovSettings(rtol=1e-12, right_pc=False))
    np.testing.assert_allclose(A @ r.x, b, atol=1e-9)
    r2 = irk.fgmres(A, b, settings=irk.KrylovSettings(rtol=1e-12, reorth=True))
    np.testing.assert_allclose(A @ r2.x, b, atol=1e-10)


def test_fgmres_residual_history_monotone(irk):
    rng = np.random.default_rng(4)
    A = rng.standard_normal((30, 30)) + 10 * np.eye(30)
    res = irk.fgmres(A, rng.standard_normal(30), settings=irk.KrylovSettings(rtol=1e-10))
    h = np.array(res.residuals)
    assert np.all(np.diff(h) <= 1e-13 * h[0])


# ------------------------------------------------------------- block solves


@pytest.mark.parametrize("dim,n", [(2, 33), (3, 9)])
def test_batched_pcg_vs_oracle(irk, oracle, dim, n):
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(dim, n))
    Mo, Ko = oracle.p1_matrices(dim, n)
    m = M.nrows
    alphas, betas = [1.0, 1.0, 0.7], [0.01, 0.2, 1e-3]
    nb = 3
    rng = np.random.default_rng(7)
    B = rng.standard_normal((m, nb))
    rhs = la.to_dev(B.ravel())
    x = la.dev_empty(m * nb)
    mask = la.dof_mask(m, bd)
    its = np.zeros(8, dtype=np.int32)
    relres = np.zeros(8)
    st = _lib.load().irk_pcg(_lib.ctx(), nb, _lib.hptr(np.array(alphas)), _lib.hptr(np.array(betas)),
                             M.device().eliminated(mask).handle, K.device().eliminated(mask).handle,
                             _lib.ptr(None), _lib.ptr(mask),
                             _lib.ptr(rhs), nb, _lib.ptr(x), nb, 1e-12, 0.0, 5000, _lib.hptr(its),
                             _lib.hptr(relres))
    assert st == 0
    X = x.cpu().numpy().reshape(m, nb)
    for k in range(nb):
        C = oracle.dirichlet_identity((alphas[k] * Mo + betas[k] * Ko).tocsr(), bd)
        exact = sp.linalg.spsolve(C.tocsc(), B[:, k])
        assert rel(X[:, k], exact) < 1e-9
        assert relres[k] <= 1e-12 and its[k] > 0


def test_cocg_complex_symmetric(irk, oracle):
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    n = 25
    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    Mo, Ko = oracle.p1_matrices(2, n)
    m = M.nrows
    coefs = [(1.0 + 0j, 0.01 + 0.004j), (0.5 + 0.2j, 0.003 + 0j)]
    rng = np.random.default_rng(9)
    Bc = rng.standard_normal((m, 2)) + 1j * rng.standard_normal((m, 2))
    il = np.zeros((m, 4))
    il[:, 0::2], il[:, 1::2] = Bc.real, Bc.imag
    rhs = la.to_dev(il.ravel())
    x = la.dev_empty(4 * m)
    mask = la.dof_mask(m, bd)
    its = np.zeros(8, dtype=np.int32)
    rr = np.zeros(8)
    arr = lambda f: _lib.hptr(np.array([f(c) for c in coefs] + [0.0] * 6))  # noqa: E731
    st = _lib.load().irk_cocg(_lib.ctx(), 2, arr(lambda c: c[0].real), arr(lambda c: c[0].imag),
                              arr(lambda c: c[1].real), arr(lambda c: c[1].imag),
                              M.device().eliminated(mask).handle, K.device().eliminated(mask).handle,
                              _lib.ptr(mask), _lib.ptr(rhs), 4, _lib.ptr(x), 4,
                              1e-12, 0.0, 5000, _lib.hptr(its), _lib.hptr(rr))
    assert st == 0
    X = x.cpu().numpy().reshape(m, 4)
    for k, (a, b) in enumerate(coefs):
        Z = oracle.dirichlet_identity((a * Mo + b * Ko).tocsr(), bd)
        exact = sp.linalg.spsolve(Z.tocsc(), Bc[:, k])
        got = X[:, 2 * k] + 1j * X[:, 2 * k + 1]
        assert np.linalg.norm(got - exact) / np.linalg.norm(exact) < 1e-9


def test_factorize_block(irk):
    M, K, bd = irk.assemble_heat(irk.StructuredGrid(1, 9))
    fac = irk.factorize_block(M, K, 2.5, 0.1)
    rng = np.random.default_rng(1)
    for _ in range(3):
        b = rng.standard_normal(10)
        assert np.linalg.norm(fac.matvec(fac.solve(b)) - b) < 1e-10 * np.linalg.norm(b)
    dense = M.to_dense() + 0.25 * K.to_dense()
    b = rng.standard_normal(10)
    np.testing.assert_allclose(irk.factorize_block(M, K, 1.0, 0.25).solve(b),
                               np.linalg.solve(dense, b), atol=1e-11)
    with pytest.raises(irk.FactorizationError):
        irk.factorize_block(K, K, 0.0, 1.0)  # pure Neumann stiffness is singular
    with pytest.raises(ValueError):
        irk.factorize_block(M, irk.assemble_heat(irk.StructuredGrid(1, 4))[1], 1.0, 1.0)


# ----------------------------------------------------------- preconditioners


@pytest.mark.parametrize("tname", ["radau3", "lobatto3"])
@pytest.mark.parametrize("kind", ["jacobi", "gs-lower", "gs-upper", "rana-ld", "rana-du"])
@pytest.mark.parametrize("form", ["ai", "ia"])
def test_preconditioner_vs_reference(irk, golden, tname, kind, form):
    key = f"pc_{tname}_{kind}_{form}"
    if key not in golden.files:
        pytest.skip("reference rejects this kind/form/tableau")
    M, K, bd = irk.assemble_heat(irk.StructuredGrid(1, 10))
    tab = irk.radau_iia(3) if tname == "radau3" else irk.lobatto_iiic(3)
    pc = irk.build_preconditioner(irk.PreconditionerKind(kind), tab, M, K, 0.05,
                                  irk.Splitting(form), bd,
                                  settings=irk.BlockSolveSettings(rtol=1e-14, maxit=1000))
    assert rel(pc.apply(golden[f"pc_{tname}_v"]), golden[key]) < 1e-10


@pytest.mark.parametrize("tab_name", ["gauss-legendre:4", "radau-iia:3", "gauss-legendre:3"])
@pytest.mark.parametrize("form", ["ai", "ia"])
def test_schur_preconditioner_vs_oracle(irk, oracle, tab_name, form):
    n = 5
    M, K, bd = irk.assemble_p1(irk.CubeGrid(3, n))
    Mo, Ko = oracle.p1_matrices(3, n)
    tab = irk.from_spec(tab_name)
    pc = irk.build_preconditioner(irk.PreconditionerKind.SCHUR, tab, M, K, 5e-3,
                                  irk.Splitting(form), bd,
                                  settings=irk.BlockSolveSettings(rtol=1e-14, maxit=2000))
    v = np.random.default_rng(2).standard_normal(tab.s * M.nrows)
    # dense reference: (Q (x) I) blockdiag(P_b (x) M + Q_b (x) K)^-1 (Q^T (x) I), constrained
    At = pc.A_tilde
    s, m = tab.s, M.nrows
    if form == "ai":
        S = np.kron(np.eye(s), Mo.toarray()) + 5e-3 * np.kron(At, Ko.toarray())
    else:
        S = np.kron(np.linalg.inv(At), Mo.toarray()) + 5e-3 * np.kron(np.eye(s), Ko.toarray())
    idx = oracle.stage_index(s, m, bd)
    keep = np.ones(s * m, bool)
    keep[idx] = False
    S[~keep, :] = 0
    S[:, ~keep] = 0
    S[idx, idx] = 1.0
    assert rel(pc.apply(v), np.linalg.solve(S, v)) < 1e-9


# ------------------------------------------------------- geometric multigrid


def _p1_block(irk, dim, n, alpha, beta):
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(dim, n))
    st = la.BlockSolveSettings(method="mg", rtol=1e-12, raise_on_maxit=True)
    fac = la.BlockFactorization(M, K, alpha, beta, bd, st)
    return M, K, bd, fac


@pytest.mark.gpu
def test_direct_small_blocks(cuda, irk, oracle):
    """Blocks of at most DIRECT_MAX rows are solved exactly through the
    device-resident inverse (one dense matrix-vector kernel): equal to a
    sparse direct solve, one 'iteration', nothing logged when deferred."""
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, 32))
    fac = la.BlockFactorization(M, K, 1.0, 5e-3, bd, la.BlockSolveSettings(rtol=1e-6))
    assert fac.direct and fac._mg is None
    Mo, Ko = oracle.p1_matrices(2, 32)
    B = oracle.dirichlet_identity((Mo + 5e-3 * Ko).tocsr(), bd)
    rhs = np.random.default_rng(9).standard_normal(M.nrows)
    x = fac.solve(rhs)
    assert rel(x, spla.spsolve(B.tocsc(), rhs)) < 1e-12
    assert fac.last_iterations == 1
    rd, xd = la.to_dev(rhs), la.dev_empty(3 * M.nrows)
    with _lib.deferred_solves() as log:
        assert fac.dev_solve(rd, xd[1:], ld_x=3, defer=True) == 1
    assert log.entries.shape[0] == 0
    assert rel(la.to_host(xd).reshape(-1, 3)[:, 1], x) < 1e-14
    assert fac._inv is not None


@pytest.mark.gpu
@pytest.mark.parametrize("n", [32, 1024])
def test_chebyshev_block_solver(cuda, irk, oracle, n):
    """method="chebyshev" runs irk_chebyshev (Gershgorin bounds, sweep count
    from rtol) and meets the tolerance against a sparse direct solve -- at
    the config-2 block (n = 1024: M + dt a_ii K, RadauIIA-3) too."""
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    beta = 1e-3 * 0.1550510257216822  # dt * a_11 of RadauIIA-3
    st = la.BlockSolveSettings(method="chebyshev", rtol=1e-10)
    fac = la.BlockFactorization(M, K, 1.0, beta, bd, st)
    lmin, lmax = fac._cheb
    assert 0 < lmin < 1 < lmax <= 2
    Mo, Ko = oracle.p1_matrices(2, n)
    B = oracle.dirichlet_identity((Mo + beta * Ko).tocsr(), bd)
    rhs = np.random.default_rng(4).standard_normal(M.nrows)
    x = fac.solve(rhs)
    k = fac.last_iterations
    assert k == fac.chebyshev_iterations() and k > 1
    ref = spla.spsolve(B.tocsc(), rhs)
    # the bound 2/T_k is on the D^-1/2 B D^-1/2-energy norm of the error;
    # the 2-norm error stays within a condition-number factor of it
    assert rel(x, ref) < 1e-7
    # fixed sweep count: cheb_iters overrides the bound
    fac2 = la.BlockFactorization(M, K, 1.0, beta, bd,
                                 la.BlockSolveSettings(method="chebyshev", cheb_iters=7))
    fac2.solve(rhs)
    assert fac2.last_iterations == 7


@pytest.mark.gpu
def test_chebyshev_rejects_indefinite_bounds(cuda, irk):
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, 8))
    with pytest.raises(ValueError):  # pure stiffness: Gershgorin lower bound 0
        la.BlockFactorization(M, K, 0.0, 1.0, bd, la.BlockSolveSettings(method="chebyshev"))


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["direct", "chebyshev"])
def test_block_diagonal_pc_honours_block_method(cuda, irk, method):
    """BLOCK_DIAGONAL with method="direct"/"chebyshev" solves through the
    block factors the user asked for (not the batched Jacobi-PCG)."""
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, 16))
    tab = irk.radau_iia(3)
    st = la.BlockSolveSettings(method=method, rtol=1e-10)
    pc = irk.build_preconditioner(irk.PreconditionerKind.BLOCK_DIAGONAL, tab, M, K, 1e-2,
                                  irk.Splitting.AI, bd, st)
    v = np.random.default_rng(2).standard_normal(3 * M.nrows)
    y = pc.apply(v)
    assert pc._mg_blocks()
    its = [r[0] for r in pc.inner_iterations]
    if method == "direct":
        assert its == [1, 1, 1]
    else:
        assert its == [pc.block_factors[i].chebyshev_iterations() for i in range(3)]
    ref = irk.build_preconditioner(irk.PreconditionerKind.BLOCK_DIAGONAL, tab, M, K, 1e-2,
                                   irk.Splitting.AI, bd,
                                   la.BlockSolveSettings(method="pcg", rtol=1e-13)).apply(v)
    assert rel(y, ref) < 1e-6


@pytest.mark.gpu
def test_deferred_log_grows(cuda, irk):
    """More than 4096 deferred solves in one log: every entry is kept, in
    order, and the status codes stay deferred (no synchronous fallback)."""
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(1, 64))
    fac = la.BlockFactorization(M, K, 1.0, 1e-2, bd,
                                la.BlockSolveSettings(method="pcg", rtol=1e-8))
    rhs = la.to_dev(np.random.default_rng(1).standard_normal(M.nrows))
    x = la.dev_empty(M.nrows)
    with _lib.deferred_solves() as log:
        for _ in range(5000):
            assert fac.dev_solve(rhs, x, defer=True) is None
    assert log.entries.shape == (5000, 4)
    assert np.all(log.entries[:, 1] == 0)
    assert len(set(log.entries[:, 0].tolist())) == 1


@pytest.mark.gpu
def test_mg_vcycle_is_symmetric(cuda, irk):
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd, fac = _p1_block(irk, 2, 64, 1.0, 2e-3)
    assert fac._mg is not None and fac._mg.levels >= 3
    rng = np.random.default_rng(3)
    a = la.to_dev(rng.standard_normal(M.nrows))
    b = la.to_dev(rng.standard_normal(M.nrows))
    va, vb = la.dev_empty(M.nrows), la.dev_empty(M.nrows)
    lib = _lib.load()
    assert lib.irk_mg_vcycle(_lib.ctx(), fac._mg.handle, _lib.ptr(a), _lib.ptr(va)) == 0
    assert lib.irk_mg_vcycle(_lib.ctx(), fac._mg.handle, _lib.ptr(b), _lib.ptr(vb)) == 0
    x, y = float((va * b).sum()), float((a * vb).sum())
    assert abs(x - y) <= 1e-12 * max(abs(x), 1.0)
    assert float((va * a).sum()) > 0  # positive


@pytest.mark.gpu
@pytest.mark.parametrize("n,beta", [(64, 2e-3), (128, 1e-3), (1024, 4e-4)])
def test_mg_structured_vcycle_matches_generic(cuda, irk, n, beta):
    """The matrix-free 2D stencil V-cycle (k_mg2_*) computes the generic
    gather V-cycle (k_mg_*) up to summation order, stays symmetric, and the
    MG-PCG solve converges in the same number of iterations."""
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd, fac = _p1_block(irk, 2, n, 1.0, beta)
    mg = fac._mg
    assert mg is not None and mg.structured
    rng = np.random.default_rng(5)
    a = la.to_dev(rng.standard_normal(M.nrows))
    b = la.to_dev(rng.standard_normal(M.nrows))
    lib = _lib.load()

    def vc(v):
        out = la.dev_empty(M.nrows)
        assert lib.irk_mg_vcycle(_lib.ctx(), mg.handle, _lib.ptr(v), _lib.ptr(out)) == 0
        return out

    za, zb = vc(a), vc(b)
    mg.structured = False
    ga = vc(a)
    rhs = rng.standard_normal(M.nrows)
    x_gen = fac.solve(rhs)
    its_gen = fac.last_iterations
    mg.structured = True
    x_st = fac.solve(rhs)
    assert float(torch_norm(za - ga)) <= 1e-12 * float(torch_norm(ga))
    x, y = float((za * b).sum()), float((a * zb).sum())
    assert abs(x - y) <= 1e-12 * max(abs(x), 1.0)
    assert rel(x_st, x_gen) < 1e-10
    assert abs(fac.last_iterations - its_gen) <= 1


def torch_norm(t):
    return t.double().norm()


@pytest.mark.gpu
@pytest.mark.parametrize("nu", [3, 4])
def test_mg_structured_smoothing_degree(cuda, irk, nu):
    """Temporally blocked pre/post smoothers with nu = 3, 4 Chebyshev steps
    (halo nu shared-memory tiles) equal the generic per-step kernels and keep
    the V-cycle symmetric; more smoothing never needs more CG iterations."""
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, 256))
    fac2 = la.BlockFactorization(M, K, 1.0, 1e-3, bd, la.BlockSolveSettings(rtol=1e-10))
    st = la.BlockSolveSettings(rtol=1e-10, mg_nu=nu)
    fac = la.BlockFactorization(M, K, 1.0, 1e-3, bd, st)
    mg = fac._mg
    assert mg is not None and mg.structured
    rng = np.random.default_rng(nu)
    a = la.to_dev(rng.standard_normal(M.nrows))
    b = la.to_dev(rng.standard_normal(M.nrows))
    lib = _lib.load()

    def vc(v):
        out = la.dev_empty(M.nrows)
        assert lib.irk_mg_vcycle(_lib.ctx(), mg.handle, _lib.ptr(v), _lib.ptr(out)) == 0
        return out

    za, zb = vc(a), vc(b)
    mg.structured = False
    ga = vc(a)
    mg.structured = True
    assert float(torch_norm(za - ga)) <= 1e-12 * float(torch_norm(ga))
    x, y = float((za * b).sum()), float((a * zb).sum())
    assert abs(x - y) <= 1e-12 * max(abs(x), 1.0)
    rhs = rng.standard_normal(M.nrows)
    fac2.solve(rhs)
    fac.solve(rhs)
    assert fac.last_iterations <= fac2.last_iterations


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 64), (3, 16)])
def test_mgc_cocg_schur_pair(cuda, irk, oracle, dim, n):
    """Complex multigrid-preconditioned COCG (irk_mgc_cocg) on a Gauss-
    Legendre Schur-pair block alpha M + beta K (complex beta, Dirichlet
    identity rows / eliminated columns) against a sparse direct solve, and
    in far fewer iterations than Jacobi-COCG."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(dim, n))
    m = M.nrows
    mask = la.dof_mask(m, bd)
    Md, Kd = la.shared_pattern([M.device(), K.device()])
    Md, Kd = Md.eliminated(mask), Kd.eliminated(mask)
    alpha, beta = 1.0 + 0.0j, 0.05 * (0.0916 + 0.1157j) * (n / 16) ** 2
    h = la._MgcHierarchy.build(M, K, Md, Kd, alpha, beta, mask,
                               la.BlockSolveSettings(method="mg", rtol=1e-10))
    assert h is not None and h.levels >= 2 and not h.dst
    rng = np.random.default_rng(7)
    rhs = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    b = la.to_dev(np.ascontiguousarray(np.stack([rhs.real, rhs.imag], axis=1)).reshape(-1))
    x = la.dev_zeros(2 * m)
    its = np.zeros(1, dtype=np.int32)
    rel_ = np.zeros(1)
    st = _lib.load().irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(b), 2, _lib.ptr(x), 2, 1e-10,
                                  0.0, 500, _lib.hptr(its), _lib.hptr(rel_))
    assert st == 0, _lib.last_error()
    xh = la.to_host(x).reshape(m, 2)
    xc = xh[:, 0] + 1j * xh[:, 1]
    Mo, Ko = oracle.p1_matrices(dim, n)
    keep = np.ones(m)
    keep[bd] = 0.0
    D, I = sp.diags(keep), sp.diags(1.0 - keep)
    A = (D @ (alpha * Mo + beta * Ko) @ D + I).tocsc()
    ref = spla.spsolve(A, rhs)
    assert np.linalg.norm(xc - ref) / np.linalg.norm(ref) < 1e-8
    # Jacobi-COCG on the same block needs several times more iterations
    itj = np.zeros(8, dtype=np.int32)
    relj = np.zeros(8)
    one = np.zeros(8)
    one[0] = 1.0
    bi = np.zeros(8)
    bi[0], bi_im = beta.real, np.zeros(8)
    bi_im[0] = beta.imag
    xj = la.dev_zeros(2 * m)
    st = _lib.load().irk_cocg(_lib.ctx(), 1, _lib.hptr(one), _lib.hptr(np.zeros(8)),
                              _lib.hptr(bi), _lib.hptr(bi_im), Md.handle, Kd.handle,
                              _lib.ptr(mask), _lib.ptr(b), 2, _lib.ptr(xj), 2, 1e-10, 0.0, 5000,
                              _lib.hptr(itj), _lib.hptr(relj))
    assert st == 0
    assert its[0] * 2 < itj[0], (its[0], itj[0])
    if dim == 3:
        # the structured 3D kernels (k_mg3_*) and the generic ones give the
        # same preconditioner: same iterations, same solution
        assert h.structured
        h.structured = False
        xg = la.dev_zeros(2 * m)
        itg = np.zeros(1, dtype=np.int32)
        st = _lib.load().irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(b), 2, _lib.ptr(xg), 2,
                                      1e-10, 0.0, 500, _lib.hptr(itg), _lib.hptr(rel_))
        h.structured = True
        assert st == 0 and itg[0] == its[0]
        assert float((xg - x).norm()) <= 1e-9 * float(x.norm())


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n,beta", [(2, 32, 5e-3), (2, 64, 1e-2), (3, 16, 5e-3)])
def test_mg_pcg_solves_block(cuda, irk, oracle, dim, n, beta):
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import sparsela as la

    M, K, bd, fac = _p1_block(irk, dim, n, 1.0, beta)
    assert fac._mg is not None
    Mo, Ko = oracle.p1_matrices(dim, n)
    B = oracle.dirichlet_identity((Mo + beta * Ko).tocsr(), bd)
    rhs = np.random.default_rng(11).standard_normal(M.nrows)
    x = fac.solve(rhs)
    ref = spla.spsolve(B.tocsc(), rhs)
    assert rel(x, ref) < 1e-9
    its_mg = fac.last_iterations
    jac = la.BlockFactorization(M, K, 1.0, beta, bd,
                                la.BlockSolveSettings(method="pcg", rtol=1e-12,
                                                      raise_on_maxit=True))
    jac.solve(rhs)
    assert its_mg < jac.last_iterations / 3, (its_mg, jac.last_iterations)


@pytest.mark.gpu
def test_mg_pcg_cap_and_deferred_log(cuda, irk):
    """Iteration cap inside the graph-resident loop raises / reports like the
    host loop; deferred solves log (iterations, code) in call order."""
    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd, fac = _p1_block(irk, 2, 32, 1.0, 5e-3)
    rhs = la.to_dev(np.random.default_rng(2).standard_normal(M.nrows))
    x = la.dev_empty(M.nrows)
    capped = la.BlockSolveSettings(rtol=1e-14, maxit=2, raise_on_maxit=True)
    with pytest.raises(la.NonConvergenceError):
        fac.dev_solve(rhs, x, settings=capped)
    assert fac.last_iterations == 2
    soft = la.BlockSolveSettings(rtol=1e-6)
    ref_its = fac.dev_solve(rhs, x, settings=soft)
    capped_soft = la.BlockSolveSettings(rtol=1e-14, maxit=3)
    with _lib.deferred_solves() as log:
        assert fac.dev_solve(rhs, x, settings=soft, defer=True) is None
        assert fac.dev_solve(rhs, x, settings=capped_soft, defer=True) is None
    assert log.entries.shape == (2, 4)
    assert log.entries[0, 0] == ref_its and log.entries[0, 1] == 0
    assert log.entries[1, 0] == 3 and log.entries[1, 1] == 1


@pytest.mark.gpu
def test_forked_block_and_pair_solves_match_sequential(cuda, irk):
    """irk_mg_pcg_multi / irk_mgc_cocg_multi: deferred independent solves
    run concurrently on auxiliary streams and give bit-identical solutions,
    iteration counts and log order to the one-by-one synchronous solves."""
    import ctypes as C

    import torch

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    lib = _lib.load()
    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, 128))
    m, s = M.nrows, 3
    st = la.BlockSolveSettings(method="mg", rtol=1e-8)
    facs = [la.BlockFactorization(M, K, 1.0, b, bd, st) for b in (2e-3, 5e-3, 1e-2)]
    assert all(f._mg is not None for f in facs)
    R = la.to_dev(np.random.default_rng(5).standard_normal(s * m))
    X_seq = la.dev_zeros(s * m)
    its_seq = []
    for k, f in enumerate(facs):
        its_seq.append(f.dev_solve(R[k:], X_seq[k:], ld_rhs=s, ld_x=s, settings=st))
    hs = (C.c_void_p * s)(*[f._mg.handle.value for f in facs])
    X_par = la.dev_zeros(s * m)
    with _lib.deferred_solves() as log:
        assert lib.irk_mg_pcg_multi(_lib.ctx(), s, hs, _lib.ptr(R), s, 1, _lib.ptr(X_par), s, 1,
                                    1e-8, 0.0, 500, None, None) == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert log.entries.shape == (s, 4)
    assert list(log.entries[:, 0]) == its_seq and not log.entries[:, 1].any()
    assert torch.equal(X_par, X_seq)

    # complex Schur-pair blocks (two pairs, interleaved with ld 4)
    M3, K3, bd3 = irk.assemble_p1(irk.structured_grid(3, 16))
    m3 = M3.nrows
    mask = la.dof_mask(m3, bd3)
    Md, Kd = la.shared_pattern([M3.device(), K3.device()])
    Md, Kd = Md.eliminated(mask), Kd.eliminated(mask)
    hs3 = [la._MgcHierarchy.build(M3, K3, Md, Kd, 1.0 + 0j, b, mask,
                                  la.BlockSolveSettings(rtol=1e-10))
           for b in (0.01 * (0.09 + 0.12j), 0.01 * (0.2 + 0.05j))]
    assert all(h is not None for h in hs3)
    W = la.to_dev(np.random.default_rng(6).standard_normal(4 * m3))
    Z_seq = la.dev_zeros(4 * m3)
    its_c = []
    for k, h in enumerate(hs3):
        its = np.zeros(1, dtype=np.int32)
        rel_ = np.zeros(1)
        assert lib.irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(W[2 * k:]), 4,
                                _lib.ptr(Z_seq[2 * k:]), 4, 1e-10, 0.0, 500, _lib.hptr(its),
                                _lib.hptr(rel_)) == 0
        its_c.append(int(its[0]))
    Z_par = la.dev_zeros(4 * m3)
    hh = (C.c_void_p * 2)(*[h.handle.value for h in hs3])
    with _lib.deferred_solves() as log:
        assert lib.irk_mgc_cocg_multi(_lib.ctx(), 2, hh, _lib.ptr(W), 4, 2, _lib.ptr(Z_par), 4,
                                      2, 1e-10, 0.0, 500, None, None) == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert list(log.entries[:, 0]) == its_c and not log.entries[:, 1].any()
    assert torch.equal(Z_par, Z_seq)


def _dst_prec_host(B, N, r):
    """Host restatement of the sine-transform preconditioner (irk_dst.cuh):
    the reflection-symmetrised interior stencil of B inverted by 2D DST-I,
    boundary rows identity."""
    from scipy.fft import dst

    n1 = N + 1
    c = (N // 2) * n1 + N // 2
    st = {(dx, dy): B[c, c + dx + dy * n1] for dx in (-1, 0, 1) for dy in (-1, 0, 1)}
    s00 = st[(0, 0)]
    s10 = (st[(1, 0)] + st[(-1, 0)]) / 2
    s01 = (st[(0, 1)] + st[(0, -1)]) / 2
    s11 = (st[(1, 1)] + st[(-1, -1)] + st[(1, -1)] + st[(-1, 1)]) / 4
    cs = np.cos(np.pi * np.arange(1, N) / N)
    lam = s00 + 2 * s10 * cs[None, :] + 2 * s01 * cs[:, None] + 4 * s11 * np.outer(cs, cs)
    R = r.reshape(n1, n1)
    T = dst(dst(R[1:N, 1:N], type=1, axis=1), type=1, axis=0) / 4  # scipy DST-I = 2 sum
    Z = R.copy()
    Z[1:N, 1:N] = dst(dst(T / lam, type=1, axis=1), type=1, axis=0) / 4 * (2.0 / N) ** 2
    return Z.reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("n,beta", [(32, 2e-2), (64, 5e-3), (256, 3e-4), (512, 1e-3),
                                    (1024, 2e-4), (2048, 4.4e-4)])
def test_dst_preconditioner(cuda, irk, oracle, n, beta):
    """Fast sine-transform preconditioner (k_dst_rows / k_dst_cols below N = 256,
    the half-length k_dsth_rows / k_dsth_cols from there: N / 8 = 32 .. 256
    threads per transform, the fused-CG block sizes 128 and 256 included) against
    its scipy DST-I restatement, and the sine-transform-preconditioned CG
    block solve against a sparse direct solve, in a handful of iterations."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    m = M.nrows
    fac = la.BlockFactorization(M, K, 1.0, beta, bd,
                                la.BlockSolveSettings(method="dst", rtol=1e-10,
                                                      raise_on_maxit=True))
    assert fac._mg is not None and fac._mg.dst
    Mo, Ko = oracle.p1_matrices(2, n)
    keep = np.ones(m)
    keep[bd] = 0.0
    D, I = sp.diags(keep), sp.diags(1.0 - keep)
    A = (D @ (Mo + beta * Ko) @ D + I).tocsr()
    rng = np.random.default_rng(n)
    r = rng.standard_normal(m)
    z = la.dev_empty(m)
    assert _lib.load().irk_mg_vcycle(_lib.ctx(), fac._mg.handle, _lib.ptr(la.to_dev(r)),
                                     _lib.ptr(z)) == 0, _lib.last_error()
    z_ref = _dst_prec_host(A, n, r)
    assert np.linalg.norm(la.to_host(z) - z_ref) <= 1e-12 * np.linalg.norm(z_ref)
    if n > 256:
        return
    x = fac.solve(r)
    ref = spla.spsolve(A.tocsc(), r)
    assert np.linalg.norm(x - ref) <= 1e-8 * np.linalg.norm(ref)
    assert fac.last_iterations <= (12 if n <= 64 else 5), fac.last_iterations
    if m <= la.DIRECT_MAX:
        return  # "auto" solves small blocks directly
    # "auto" picks it, "mg" keeps the V-cycle
    assert la.BlockFactorization(M, K, 1.0, beta, bd)._mg.dst
    assert not la.BlockFactorization(M, K, 1.0, beta, bd,
                                     la.BlockSolveSettings(method="mg"))._mg.dst


def _dst3_prec_host(A, N, r):
    """scipy restatement of irk_dst3.cu: the centre row's 3x3x3 stencil of the
    complex block A averaged over the reflections of every offset, inverted
    by DST-I along the three axes on the interior; boundary rows identity."""
    from scipy.fft import dstn

    n1 = N + 1
    c = N // 2
    ctr = (c * n1 + c) * n1 + c
    row = A.getrow(ctr)
    s = np.zeros((2, 2, 2), dtype=complex)
    for col, v in zip(row.indices, row.data):
        d = int(col) - ctr
        dz = int(np.round(d / (n1 * n1)))
        d -= dz * n1 * n1
        dy = int(np.round(d / n1))
        dx = d - dy * n1
        k = (abs(dx), abs(dy), abs(dz))
        s[k] += v / 2 ** sum(k)
    t = 2 * np.cos(np.pi * np.arange(1, N) / N)
    tx, ty, tz = t[None, None, :], t[None, :, None], t[:, None, None]
    lam = sum(s[a, b, e] * tx ** a * ty ** b * tz ** e
              for a in (0, 1) for b in (0, 1) for e in (0, 1))
    R = r.reshape(n1, n1, n1)
    Ri = R[1:N, 1:N, 1:N]
    T = (dstn(Ri.real, type=1) + 1j * dstn(Ri.imag, type=1)) / lam
    Z = R.copy()
    Z[1:N, 1:N, 1:N] = (dstn(T.real, type=1) + 1j * dstn(T.imag, type=1)) / (2.0 * N) ** 3
    return Z.reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("n,bscale", [(12, 1.0), (16, 0.5), (24, 0.3), (32, 0.2), (48, 0.1),
                                      (96, 0.05)])
def test_dst3_preconditioner(cuda, irk, oracle, n, bscale):
    """3D complex fast sine-transform preconditioner (k_dst3, mixed-radix
    shared-memory FFTs) against its scipy DST-I restatement, and the
    sine-transform-preconditioned COCG pair-block solve against a sparse
    direct solve, in fewer iterations than the complex V-cycle."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(3, n))
    m = M.nrows
    mask = la.dof_mask(m, bd)
    Md, Kd = la.shared_pattern([M.device(), K.device()])
    Md, Kd = Md.eliminated(mask), Kd.eliminated(mask)
    alpha, beta = 1.0 + 0.0j, bscale * (0.0916 + 0.1157j)
    h = la._MgcHierarchy.build(M, K, Md, Kd, alpha, beta, mask,
                               la.BlockSolveSettings(method="dst", rtol=1e-10))
    assert h is not None and h.dst_available and h.dst
    Mo, Ko = oracle.p1_matrices(3, n)
    keep = np.ones(m)
    keep[bd] = 0.0
    D, I = sp.diags(keep), sp.diags(1.0 - keep)
    A = (D @ (alpha * Mo + beta * Ko) @ D + I).tocsr()
    rng = np.random.default_rng(n)
    rhs = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    b = la.to_dev(np.ascontiguousarray(np.stack([rhs.real, rhs.imag], axis=1)).reshape(-1))
    z = la.dev_empty(2 * m)
    assert _lib.load().irk_mgc_vcycle(_lib.ctx(), h.handle, _lib.ptr(b), _lib.ptr(z)) == 0, \
        _lib.last_error()
    zh = la.to_host(z).reshape(m, 2)
    z_ref = _dst3_prec_host(A, n, rhs)
    assert np.linalg.norm(zh[:, 0] + 1j * zh[:, 1] - z_ref) <= 1e-12 * np.linalg.norm(z_ref)
    x = la.dev_zeros(2 * m)
    its = np.zeros(1, dtype=np.int32)
    rel_ = np.zeros(1)
    st = _lib.load().irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(b), 2, _lib.ptr(x), 2, 1e-10,
                                  0.0, 500, _lib.hptr(its), _lib.hptr(rel_))
    assert st == 0, _lib.last_error()
    if n <= 48:
        xh = la.to_host(x).reshape(m, 2)
        ref = spla.spsolve(A.tocsc(), rhs)
        assert np.linalg.norm(xh[:, 0] + 1j * xh[:, 1] - ref) <= 1e-8 * np.linalg.norm(ref)
    else:
        xh = la.to_host(x).reshape(m, 2)
        res = rhs - A @ (xh[:, 0] + 1j * xh[:, 1])
        assert np.linalg.norm(res) <= 2e-10 * np.linalg.norm(rhs)
    # the V-cycle on the same block needs more iterations
    h.dst = False
    xv = la.dev_zeros(2 * m)
    itv = np.zeros(1, dtype=np.int32)
    st = _lib.load().irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(b), 2, _lib.ptr(xv), 2, 1e-10,
                                  0.0, 500, _lib.hptr(itv), _lib.hptr(rel_))
    assert st == 0 and float((xv - x).norm()) <= 1e-8 * float(x.norm())
    assert its[0] <= itv[0] + 2, (its[0], itv[0])
    # "auto" picks the sine transform, "mg" keeps the V-cycle, "pcg" has no hierarchy
    assert la._MgcHierarchy.build(M, K, Md, Kd, alpha, beta, mask, la.BlockSolveSettings()).dst
    if n == 12:
        # N = 20 has no transform plan (2N = 40): "dst" is refused, "auto" keeps the V-cycle
        M2, K2, bd2 = irk.assemble_p1(irk.structured_grid(3, 20))
        mask2 = la.dof_mask(M2.nrows, bd2)
        Md2, Kd2 = la.shared_pattern([M2.device(), K2.device()])
        Md2, Kd2 = Md2.eliminated(mask2), Kd2.eliminated(mask2)
        with pytest.raises(ValueError):
            la._MgcHierarchy.build(M2, K2, Md2, Kd2, alpha, beta, mask2,
                                   la.BlockSolveSettings(method="dst"))
        assert not la._MgcHierarchy.build(M2, K2, Md2, Kd2, alpha, beta, mask2,
                                          la.BlockSolveSettings()).dst


@pytest.mark.gpu
def test_mg_hierarchy_1d_and_masks(cuda, irk, oracle):
    """1D P1 blocks get a hierarchy; a non-boundary Dirichlet set or a
    missing grid tag falls back to Jacobi-PCG; the mask cache returns one
    object per dof set."""
    import scipy.sparse.linalg as spla

    from paper_2403_08084_b200 import sparsela as la

    M, K, bd, fac = _p1_block(irk, 1, 256, 1.0, 1e-3)
    assert fac._mg is not None and fac._mg.levels >= 3
    rhs = np.random.default_rng(4).standard_normal(M.nrows)
    Mo, Ko = oracle.p1_matrices(1, 256)
    B = oracle.dirichlet_identity((Mo + 1e-3 * Ko).tocsr(), bd)
    assert rel(fac.solve(rhs), spla.spsolve(B.tocsc(), rhs)) < 1e-9
    inner = la.BlockFactorization(M, K, 1.0, 1e-3, np.array([5, 9]),
                                  la.BlockSolveSettings(rtol=1e-12, raise_on_maxit=True))
    assert inner._mg is None
    untagged = la.SparseMatrix.from_scipy(Mo)
    assert la.BlockFactorization(untagged, la.SparseMatrix.from_scipy(Ko), 1.0, 1e-3, bd)._mg is None
    assert la.dof_mask(M.nrows, bd) is la.dof_mask(M.nrows, np.array(bd))


@pytest.mark.gpu
@pytest.mark.parametrize("restart,reorth,pc", [(50, False, False), (4, False, True),
                                               (7, True, True), (50, False, True)])
def test_fgmres_device_cycle_matches_host_loop(cuda, irk, restart, reorth, pc):
    """The device-resident FGMRES cycle (one CUDA graph per restart cycle:
    Arnoldi, Givens rotations and stop tests on the device) reproduces the
    host Givens loop: same iteration count, residual history and solution.
    A recurring (operator, preconditioner) key is captured on its second
    use; the first solve runs the host loop."""
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(2, 24))
    op = irk.KroneckerStageOperator(np.eye(2), irk.radau_iia(2).A, M, [K], 0.01)
    P = None
    if pc:
        fac = la.BlockFactorization(M, K, 1.0, 0.01 * 0.4, None, la.BlockSolveSettings())
        assert fac.direct and fac.graph_safe()

        class _BlockJacobi(la._DevOp):  # one direct solve per stage (interleaved)
            n = op.n

            def dev_apply(self, x, out):
                for i in range(2):
                    fac.dev_solve(x[i:], out[i:], ld_rhs=2, ld_x=2)

            def graph_key(self):
                return ("bj", fac._serial)

        P = _BlockJacobi()
    A = op._dev_op()
    assert A.graph_key() is not None
    b = la.to_dev(np.random.default_rng(11).standard_normal(op.n))
    st = la.KrylovSettings(rtol=1e-12, restart=restart, reorth=reorth, maxit=400)
    la._FG_CACHE.clear()
    la._FG_SEEN.clear()
    host = la.fgmres_device(A, b, P, st)
    assert not la._FG_CACHE  # first use: host loop
    dev = la.fgmres_device(A, b, P, st)
    assert len(la._FG_CACHE) == 1  # second use: captured and replayed
    assert dev.iterations == host.iterations
    h, d = np.array(host.residuals), np.array(dev.residuals)
    assert h.shape == d.shape
    np.testing.assert_allclose(d, h, rtol=1e-8, atol=1e-14 * h[0])
    x_h, x_d = host.x.cpu().numpy(), dev.x.cpu().numpy()
    assert np.linalg.norm(x_d - x_h) <= 1e-11 * np.linalg.norm(x_h)
    # a third solve replays the cached graph again
    again = la.fgmres_device(A, b, P, st)
    assert again.iterations == dev.iterations
    assert np.array_equal(again.x.cpu().numpy(), x_d)  # deterministic


@pytest.mark.gpu
def test_fgmres_device_cycle_lucky_breakdown(cuda, irk):
    """An exact preconditioner ends the device cycle after one step (lucky
    breakdown / converged), as the host loop does."""
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.structured_grid(2, 12))
    fac = la.BlockFactorization(M, K, 1.0, 0.05, None, la.BlockSolveSettings())
    A = la._SpmvOp(fac.matrix)
    P = fac._dev_op()
    b = la.to_dev(np.random.default_rng(2).standard_normal(M.nrows))
    st = la.KrylovSettings(rtol=1e-12)
    la._FG_CACHE.clear()
    la._FG_SEEN.clear()
    r1 = la.fgmres_device(A, b, P, st)
    r2 = la.fgmres_device(A, b, P, st)
    assert len(la._FG_CACHE) == 1
    assert r1.iterations == r2.iterations == 1
    np.testing.assert_allclose(r2.x.cpu().numpy(), r1.x.cpu().numpy(), rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("s,shift", [(3, 0), (3, 1), (2, 0), (4, 0), (1, 1)])
def test_stage_apply_bulk_tiles_vs_oracle(cuda, irk, oracle, s, shift):
    """K2 on a 2D stencil grid large enough for the bulk-asynchronous tiles
    (k_stage_apply_bulk: interior tiles by cp.async.bulk, the first / last
    tiles by gathers), masked and unmasked, with the stage vector 16-byte
    aligned or 8 bytes off (shift = 1: a Krylov basis row of odd length)."""
    from paper_2403_08084_b200 import sparsela as la

    n = 160
    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    Mo, Ko = oracle.p1_matrices(2, n)
    tab = irk.radau_iia(s)
    m = M.nrows
    op = irk.KroneckerStageOperator(np.eye(s), tab.A, M, [K], 1e-3)
    rng = np.random.default_rng(40 + s)
    v = rng.standard_normal(s * m)
    ref = oracle.kron_apply(np.eye(s), tab.A, Mo, [Ko], 1e-3, v)
    idx = oracle.stage_index(s, m, bd)
    refc = oracle.constrained(lambda w: oracle.kron_apply(np.eye(s), tab.A, Mo, [Ko], 1e-3, w),
                              idx)(v)
    import torch

    for masked, want in ((False, ref), (True, refc)):
        dev = (irk.ConstrainedStageOperator(op, bd) if masked else op)._dev_op()
        buf = la.dev_zeros(s * m + 2)
        Y = buf[shift: shift + s * m]
        Y.copy_(la.to_dev(_to_il(v, m, s)))
        out = la.dev_empty(s * m)
        dev.dev_apply(Y, out)
        got = out.cpu().numpy().reshape(m, s).T.reshape(-1)
        assert rel(got, want) < 1e-14, (masked, shift)
    torch.cuda.synchronize()


def _to_il(v, m, s):
    return np.ascontiguousarray(np.asarray(v).reshape(s, m).T).reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("gs-lower", 256), ("jacobi", 128)])
def test_fgmres_device_cycle_with_captured_dst_blocks(cuda, irk, kind, n):
    """Sweeps over sine-transform-preconditioned blocks are capturable: a
    captured block solve is a straight-line sequence of a fixed number of CG
    iterations (run_cg's captured branch; the count comes from a probe
    solve), so the device-resident FGMRES cycle holds the whole
    preconditioner application.  It reproduces the host loop (whose block
    solves stop on their tolerance) to the outer tolerance, in the same
    number of outer iterations (+-1).  dt / h^2 as in config 2 (there the
    probe finds 2 iterations); n = 256 is above DEVFG_MAX_N unknowns."""
    from paper_2403_08084_b200 import bcs
    from paper_2403_08084_b200 import sparsela as la

    M, K, bd = irk.assemble_p1(irk.StructuredGrid(2, n))
    tab = irk.radau_iia(3)
    dt = 1000.0 / n ** 2
    s = tab.s
    Ainv = np.linalg.inv(tab.A)
    op = bcs.ConstrainedStageOperator(irk.KroneckerStageOperator(Ainv, np.eye(s), M, [K], dt),
                                      bd)
    pc = irk.build_preconditioner(irk.PreconditionerKind(kind), tab, M, K, dt, irk.Splitting.IA, bd,
                                  la.BlockSolveSettings(rtol=1e-6))
    fac = pc.block_factors[0]
    assert fac._mg is not None and fac._mg.dst and not fac.direct
    ks = [f._fixed_iterations(pc.settings) for f in pc.block_factors]
    assert all(k is not None and 1 <= k <= 4 for k in ks), ks
    assert fac.graph_safe(pc.settings) and pc._graph_key() is not None
    # strict settings are never captured (a capped solve must raise)
    assert fac._fixed_iterations(la.BlockSolveSettings(rtol=1e-6, raise_on_maxit=True)) is None
    A, P = op._dev_op(), pc._dev_op()
    assert P.fixed_solves()
    b = la.to_dev(np.random.default_rng(n).standard_normal(op.n))
    st = la.KrylovSettings(rtol=1e-12, maxit=200)
    la._FG_CACHE.clear()
    la._FG_SEEN.clear()
    host = la.fgmres_device(A, b, P, st)
    assert not la._FG_CACHE
    n0 = len(pc.inner_iterations)
    dev = la.fgmres_device(A, b, P, st)
    assert len(la._FG_CACHE) == 1
    assert abs(dev.iterations - host.iterations) <= 1
    assert dev.residuals[-1] <= 1e-12 * dev.residuals[0]
    x_h, x_d = host.x.cpu().numpy(), dev.x.cpu().numpy()
    assert np.linalg.norm(x_d - x_h) <= 1e-9 * np.linalg.norm(x_h)
    # the book-keeping records the fixed count per block solve and application
    rec = pc.inner_iterations[n0:]
    assert rec == [[k] for k in ks] * dev.iterations
    again = la.fgmres_device(A, b, P, st)
    assert np.array_equal(again.x.cpu().numpy(), x_d)  # deterministic replay
