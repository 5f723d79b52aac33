"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's stage-coupled solve path
(implicitrk, /root/reference/pkg/src/implicitrk/), used as the CHECKER of the
CUDA product path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference arm may import it; the product package never
does (and fails loudly when its CUDA library is missing).

Every function cites the reference file:line it restates.  Pieces the
reference does not have (P1 triangle/Kuhn-tetrahedron assembly,
Gauss-Legendre tableaux, the real-Schur stage preconditioner, Jacobi-PCG /
COCG inner block solves, Allen-Cahn) are written here from their published
definitions and pinned by known-answer tests.

Parity pinning: tests/golden/*.npz are produced by oracle/make_golden.py,
which imports the unmodified reference from /root/reference in the build
container and runs it on the same seeded inputs; tests/test_oracle.py checks
this module against those fixtures.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

# ------------------------------------------------------------------ tableaux


@dataclass
class Tab:
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    name: str

    @property
    def s(self):
        return len(self.b)

    @property
    def stiffly_accurate(self):  # tableaux.py:315-316
        return bool(np.max(np.abs(self.b - self.A[-1])) <= 1e-12)

    @property
    def lower_triangular(self):  # tableaux.py:319-320
        return self.s == 1 or bool(np.max(np.abs(np.triu(self.A, 1))) <= 1e-12)


def _lagrange_tableau(c):
    """a_ij = int_0^{c_i} l_j, b_j = int_0^1 l_j with (s+1)-point Gauss
    quadrature (tableaux.py:146-170)."""
    s = len(c)
    xg, wg = np.polynomial.legendre.leggauss(s + 1)

    def basis(x):
        out = np.ones((s, len(x)))
        for j in range(s):
            for k in range(s):
                if k != j:
                    out[j] *= (x - c[k]) / (c[j] - c[k])
        return out

    A = np.array([basis(0.5 * ci * (xg + 1)) @ (0.5 * ci * wg) for ci in c])
    b = basis(0.5 * (xg + 1)) @ (0.5 * wg)
    return A, b


def radau(s):
    """RadauIIA (tableaux.py:125-188): nodes = roots of d^{s-1}/dx^{s-1}
    [x^{s-1}(x-1)^s], last node snapped to 1."""
    if s == 1:
        return Tab(np.array([[1.0]]), np.array([1.0]), np.array([1.0]), "radau-iia:1")
    P = np.polynomial.Polynomial
    p = (P([0.0, 1.0]) ** (s - 1) * P([-1.0, 1.0]) ** s).deriv(s - 1)
    p = p / np.max(np.abs(p.coef))
    c = np.sort(p.roots().real)
    for _ in range(50):
        r = p(c)
        if np.max(np.abs(r)) < 1e-14:
            break
        c = c - r / p.deriv()(c)
    c[-1] = 1.0
    A, b = _lagrange_tableau(c)
    return Tab(A, b, c, f"radau-iia:{s}")


def gauss(s):
    """Gauss-Legendre collocation (nodes = shifted Legendre roots)."""
    x, _ = np.polynomial.legendre.leggauss(s)
    c = 0.5 * (x + 1.0)
    A, b = _lagrange_tableau(c)
    return Tab(A, b, c, f"gauss-legendre:{s}")


def alexander():
    """Alexander SDIRK (tableaux.py:215-254)."""
    p = lambda x: x**3 - 3 * x**2 + 1.5 * x - 1 / 6  # noqa: E731
    lo, hi = 1 / 6, 0.5
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if p(lo) * p(mid) <= 0:
            hi = mid
        else:
            lo = mid
        if hi - lo < 1e-12:
            break
    x = 0.5 * (lo + hi)
    for _ in range(50):
        if abs(p(x)) < 1e-14:
            break
        x -= p(x) / (3 * x**2 - 6 * x + 1.5)
    y = -1.5 * x * x + 4 * x - 0.25
    z = 1.0 - x - y
    A = np.array([[x, 0, 0], [(1 - x) / 2, x, 0], [y, z, x]])
    return Tab(A, np.array([y, z, x]), np.array([x, (1 + x) / 2, 1.0]), "alexander")


# ------------------------------------------------------------------ assembly


def grid_coords(dim, n):
    """Vertex coordinates, lexicographic with x fastest (problems.py:47-53)."""
    x = np.linspace(0.0, 1.0, n + 1)
    mesh = np.meshgrid(*([x] * dim), indexing="ij")
    return np.column_stack([g.transpose(tuple(range(dim))[::-1]).ravel() for g in mesh])


def grid_boundary(dim, n):
    """Sorted boundary vertex ids (problems.py:55-64, extended to 3D)."""
    idx = np.arange((n + 1) ** dim)
    on = np.zeros(len(idx), dtype=bool)
    for d in range(dim):
        k = (idx // (n + 1) ** d) % (n + 1)
        on |= (k == 0) | (k == n)
    return np.nonzero(on)[0].astype(np.int64)


def _simplices(dim, n):
    """Element vertex lists in the global element order: cells ascending
    lexicographically (x fastest), then the fixed simplex order in a cell."""
    n1 = n + 1
    if dim == 1:
        e = np.arange(n)
        return np.stack([e, e + 1], axis=1)
    if dim == 2:
        cj, ci = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        v00 = (cj * n1 + ci).ravel()
        v10, v01, v11 = v00 + 1, v00 + n1, v00 + n1 + 1
        t1 = np.stack([v00, v10, v11], axis=1)  # right angle at v10
        t2 = np.stack([v00, v11, v01], axis=1)  # right angle at v01
        return np.stack([t1, t2], axis=1).reshape(-1, 3)
    ck, cj, ci = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = (ck * n1 * n1 + cj * n1 + ci).ravel()
    stride = np.array([1, n1, n1 * n1])
    tets = []
    for perm in itertools.permutations(range(3)):
        e0, e1 = stride[perm[0]], stride[perm[1]]
        tets.append(np.stack([base, base + e0, base + e0 + e1, base + stride.sum()], axis=1))
    return np.stack(tets, axis=1).reshape(-1, 4)


def p1_matrices(dim, n):
    """P1 mass and stiffness on the simplicial split, assembled element by
    element (COO in element order -> CSR, duplicates summed, explicit zeros
    kept, M and K on one pattern).  Element matrices: mass |T|/((d+1)(d+2))
    (1 + delta_ab); stiffness |T| grad(phi_a).grad(phi_b)."""
    h = 1.0 / n
    el = _simplices(dim, n)
    X = grid_coords(dim, n)
    nv, m = el.shape[1], X.shape[0]
    if dim == 1:
        mloc = np.array([[2 * h / 6, h / 6], [h / 6, 2 * h / 6]])
        kloc = np.array([[1.0 / h, -1.0 / h], [-1.0 / h, 1.0 / h]])
        Mv = np.broadcast_to(mloc, (len(el), 2, 2))
        Kv = np.broadcast_to(kloc, (len(el), 2, 2))
    else:
        mf = (h * h / 24.0) if dim == 2 else (h * h * h / 120.0)
        Mv = mf * (np.ones((nv, nv)) + np.eye(nv))[None].repeat(len(el), axis=0)
        if dim == 2:
            # exact local stiffness of the two right triangles (no round-off)
            k1 = np.array([[0.5, -0.5, 0.0], [-0.5, 1.0, -0.5], [0.0, -0.5, 0.5]])
            k2 = np.array([[0.5, 0.0, -0.5], [0.0, 0.5, -0.5], [-0.5, -0.5, 1.0]])
            Kv = np.stack([k1, k2])[None].repeat(len(el) // 2, axis=0).reshape(-1, 3, 3)
        else:
            g = np.array([[1, -1, 0, 0], [-1, 2, -1, 0], [0, -1, 2, -1], [0, 0, -1, 1]], float)
            Kv = (h / 6.0) * np.broadcast_to(g, (len(el), 4, 4))
    rows = np.repeat(el, nv, axis=1).ravel()
    cols = np.tile(el, (1, nv)).ravel()
    M = sp.coo_matrix((np.asarray(Mv).ravel(), (rows, cols)), shape=(m, m)).tocsr()
    K = sp.coo_matrix((np.asarray(Kv).ravel(), (rows, cols)), shape=(m, m)).tocsr()
    for A in (M, K):
        A.sort_indices()
    return M, K


def q1_matrices(n):
    """Reference 2D Q1 operators (problems.py:67-99)."""
    h = 1.0 / n
    mm = np.full(n + 1, 4 * h / 6)
    mm[0] = mm[-1] = 2 * h / 6
    km = np.full(n + 1, 2.0 / h)
    km[0] = km[-1] = 1.0 / h
    M1 = sp.diags([np.full(n, h / 6), mm, np.full(n, h / 6)], [-1, 0, 1], format="csr")
    K1 = sp.diags([np.full(n, -1.0 / h), km, np.full(n, -1.0 / h)], [-1, 0, 1], format="csr")
    M = sp.kron(M1, M1, format="csr")
    K = (sp.kron(K1, M1) + sp.kron(M1, K1)).tocsr()
    M.sort_indices()
    K.sort_indices()
    return M, K


# ------------------------------------------------------------ stage operator


def kron_apply(C1, C2, M, Ks, dt, v):
    """(C1 (x) M + dt C2 (x) K) v, stage-major (sparsela.py:222-235)."""
    s = C1.shape[0]
    m = M.shape[0]
    V = v.reshape(s, m)
    U1, U2 = C1 @ V, C2 @ V
    out = (M @ U1.T).T
    if len(Ks) == 1:
        out = out + dt * (Ks[0] @ U2.T).T
    else:
        out = out.copy()
        for i in range(s):
            out[i] += dt * (Ks[i] @ U2[i])
    return out.ravel()


def stage_index(s, m, dofs):
    return (np.arange(s)[:, None] * m + np.asarray(dofs)[None, :]).ravel()


def constrained(op, idx):
    """Row identity / column elimination wrapper (bcs.py:114-120)."""

    def apply(v):
        w = v.copy()
        w[idx] = 0.0
        y = op(w)
        y[idx] = v[idx]
        return y

    return apply


# --------------------------------------------------------------- Krylov


class NoConvergence(RuntimeError):
    def __init__(self, msg, residuals):
        super().__init__(msg)
        self.residuals = residuals


def fgmres(A, b, P=None, rtol=1e-8, atol=1e-50, restart=50, maxit=500, right_pc=True, x0=None):
    """Restarted flexible GMRES with MGS Arnoldi and Givens rotations
    (sparsela.py:299-403).  Returns (x, iterations, residuals)."""
    n = len(b)
    left = P is not None and not right_pc
    rhs = P(b) if left else b
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)

    def resid(xv):
        r_ = b - A(xv)
        return P(r_) if left else r_

    r = rhs.copy() if x0 is None else resid(x)
    nb = np.linalg.norm(rhs)
    target = max(rtol * nb, atol)
    hist = [float(np.linalg.norm(r))]
    its = 0
    if hist[0] <= target:
        return x, 0, hist
    brk = 1e-14 * nb
    while True:
        cyc = min(restart, maxit - its)
        if cyc <= 0:
            raise NoConvergence("fgmres cap", hist)
        beta = np.linalg.norm(r)
        V = np.empty((cyc + 1, n))
        Z = np.empty((cyc, n))
        V[0] = r / beta
        H = np.zeros((cyc + 1, cyc))
        cs, sn, g = np.zeros(cyc), np.zeros(cyc), np.zeros(cyc + 1)
        g[0] = beta
        done = False
        for j in range(cyc):
            if left:
                z = V[j]
                w = P(A(z))
            else:
                z = V[j] if P is None else P(V[j])
                w = A(z)
            Z[j] = z
            its += 1
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            lucky = H[j + 1, j] < brk
            if not lucky:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            if d == 0.0:
                cs[j], sn[j], d = 1.0, 0.0, 1e-300
            else:
                cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j], H[j + 1, j] = d, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            hist.append(abs(float(g[j + 1])))
            if hist[-1] <= target or lucky:
                done = True
                break
        k = j + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + Z[:k].T @ y
        if done or hist[-1] <= target:
            return x, its, hist
        if its >= maxit:
            raise NoConvergence("fgmres cap", hist)
        r = resid(x)


def jacobi_pcg(B, b, rtol, atol=0.0, maxit=100000):
    """Jacobi-preconditioned CG from x = 0, stop on ||r|| <= max(rtol||b||, atol)."""
    dinv = 1.0 / B.diagonal()
    x = np.zeros_like(b)
    r = b.copy()
    bb = float(r @ r)
    tol2 = max(rtol * rtol * bb, atol * atol)
    if bb <= tol2:
        return x, 0
    z = dinv * r
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, maxit + 1):
        q = B @ p
        a = rz / float(p @ q)
        x += a * p
        r -= a * q
        if float(r @ r) <= tol2:
            return x, it
        z = dinv * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit


def jacobi_cocg(B, b, rtol, maxit=100000):
    """Jacobi-preconditioned conjugate orthogonal CG for complex-symmetric B."""
    dinv = 1.0 / B.diagonal()
    x = np.zeros_like(b)
    r = b.copy()
    bb = float(np.vdot(r, r).real)
    tol2 = rtol * rtol * bb
    if bb <= tol2:
        return x, 0
    z = dinv * r
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = B @ p
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if float(np.vdot(r, r).real) <= tol2:
            return x, it
        z = dinv * r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit


def dirichlet_identity(C, dofs):
    """Identity rows/columns on dofs (sparsela.py:126-146)."""
    if len(dofs) == 0:
        return C.tocsr()
    keep = np.ones(C.shape[0], dtype=bool)
    keep[dofs] = False
    D = sp.diags(keep.astype(float))
    out = (D @ C @ D).tolil()
    out[dofs, dofs] = 1.0
    return out.tocsr()


class Block:
    """alpha*M + dt*K with Dirichlet identity rows/cols, solved by SuperLU
    ('lu', the reference's factorize_block, sparsela.py:171-191) or by
    Jacobi-PCG ('pcg', north_star)."""

    def __init__(self, M, K, alpha, beta, dofs, method="lu", rtol=1e-6):
        self.C = dirichlet_identity((alpha * M + beta * K).tocsr(), dofs)
        self.method, self.rtol = method, rtol
        self.lu = spla.splu(self.C.tocsc()) if method == "lu" else None
        self.its = []

    def solve(self, b):
        if self.lu is not None:
            return self.lu.solve(b)
        x, it = jacobi_pcg(self.C, b, self.rtol)
        self.its.append(it)
        return x


# ---------------------------------------------------------- preconditioners


def surrogate(kind, A):
    """A~ per kind (precond.py:43-57) plus SCHUR = Q blockdiag(T) Q^T."""
    if kind == "jacobi":
        return np.diag(np.diag(A))
    if kind == "gs-lower":
        return np.tril(A)
    if kind == "gs-upper":
        return np.triu(A)
    if kind in ("rana-ld", "rana-du"):
        s = A.shape[0]
        U = A.copy()
        L = np.eye(s)
        for k in range(s):
            for i in range(k + 1, s):
                L[i, k] = U[i, k] / U[k, k]
                U[i, k:] -= L[i, k] * U[k, k:]
        D = np.diag(U).copy()
        return L * D[None, :] if kind == "rana-ld" else U
    if kind == "schur":
        Q, T, blocks = schur_blocks(A)
        Tb = np.zeros_like(A)
        for st, sz in blocks:
            Tb[st:st + sz, st:st + sz] = T[st:st + sz, st:st + sz]
        return Q @ Tb @ Q.T
    raise ValueError(kind)


def schur_blocks(A):
    T, Q = sla.schur(A, output="real")
    s = A.shape[0]
    blocks, i = [], 0
    while i < s:
        if i + 1 < s and abs(T[i + 1, i]) > 1e-14:
            blocks.append((i, 2))
            i += 2
        else:
            blocks.append((i, 1))
            i += 1
    return Q, T, blocks


class StagePC:
    """Block preconditioner apply on stage-major vectors (precond.py:60-117);
    kind 'schur' solves the blocks of I (x) M + dt T_bb (x) K (AI form) after
    the (Q^T (x) I) transform, complex pairs as one complex-symmetric system."""

    def __init__(self, kind, tab, M, Ks, dt, form, dofs, block="lu", rtol=1e-6):
        self.kind, self.form, self.M, self.Ks, self.dt = kind, form, M, Ks, dt
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self.s, self.m = tab.s, M.shape[0]
        self.At = surrogate(kind, np.asarray(tab.A))
        self.Ati = np.linalg.inv(self.At)
        self.coef = self.Ati if form == "ia" else dt * self.At
        self.block, self.rtol = block, rtol
        if kind == "schur":
            self._schur_setup(np.asarray(tab.A))
            return
        self.blocks = []
        for i in range(self.s):
            Ki = Ks[0] if len(Ks) == 1 else Ks[i]
            if form == "ia":
                self.blocks.append(Block(M, Ki, self.Ati[i, i], dt, self.dofs, block, rtol))
            else:
                self.blocks.append(Block(M, Ki, 1.0, dt * self.At[i, i], self.dofs, block, rtol))

    def _schur_setup(self, A):
        Q, T, blocks = schur_blocks(A)
        self.Q, self.T, self.sblocks = Q, T, blocks
        M, K = self.M, self.Ks[0]
        self.sol = []
        for st, sz in blocks:
            Tb = T[st:st + sz, st:st + sz]
            if sz == 1:
                self.sol.append(Block(M, K, 1.0, self.dt * Tb[0, 0], self.dofs, self.block, self.rtol))
            else:
                big = sp.bmat([[M + self.dt * Tb[0, 0] * K, self.dt * Tb[0, 1] * K],
                               [self.dt * Tb[1, 0] * K, M + self.dt * Tb[1, 1] * K]]).tocsr()
                dd = np.concatenate([self.dofs, self.dofs + self.m])
                self.sol.append(_PairSolver(big, dd, self.m, self.block, self.rtol, Tb, self.dt,
                                            M, K, self.dofs))

    def apply(self, r):
        s, m = self.s, self.m
        R = r.reshape(s, m)
        if self.kind == "schur":
            W = self.Q.T @ R
            X = np.zeros_like(W)
            for (st, sz), sol in zip(self.sblocks, self.sol):
                X[st:st + sz] = sol.solve(W[st:st + sz].ravel()).reshape(sz, m)
            return (self.Q @ X).ravel()
        X = np.zeros_like(R)
        if self.kind == "jacobi":
            order, deps = range(s), lambda i: ()
        elif self.kind in ("gs-lower", "rana-ld"):
            order, deps = range(s), lambda i: range(i)
        else:
            order, deps = range(s - 1, -1, -1), lambda i: range(i + 1, s)
        for i in order:
            acc = R[i].copy()
            for j in deps(i):
                if self.coef[i, j] != 0.0:
                    xj = X[j].copy()
                    xj[self.dofs] = 0.0
                    C = self.M if self.form == "ia" else (self.Ks[0] if len(self.Ks) == 1 else self.Ks[i])
                    c = self.coef[i, j] * (C @ xj)
                    c[self.dofs] = 0.0
                    acc -= c
            X[i] = self.blocks[i].solve(acc)
        return X.ravel()


class _PairSolver:
    """2x2 Schur block: exact (SuperLU on the real 2m system) or complex
    Jacobi-COCG on (M + dt(a + i w) K) after the standard scaling."""

    def __init__(self, big, dd, m, method, rtol, Tb, dt, M, K, dofs):
        self.m, self.method, self.rtol = m, method, rtol
        if method == "lu":
            self.lu = spla.splu(dirichlet_identity(big, dd).tocsc())
            return
        a = 0.5 * (Tb[0, 0] + Tb[1, 1])
        b, c = Tb[0, 1], Tb[1, 0]
        self.w = np.sqrt(-b * c)
        self.dd, self.cc = self.w / c, -self.w / b
        Z = (M + dt * (a + 1j * self.w) * K).tocsr()
        self.Z = dirichlet_identity(Z, dofs)

    def solve(self, rhs):
        m = self.m
        if self.method == "lu":
            return self.lu.solve(rhs)
        r1, r2 = rhs[:m], rhs[m:]
        z, _ = jacobi_cocg(self.Z, r1 + 1j * self.dd * r2, self.rtol)
        return np.concatenate([z.real, self.cc * z.imag])


# ---------------------------------------------------------------- stepping


@dataclass
class Problem:
    """M u' + K u = 0 with Dirichlet g at dofs, or a semilinear residual
    M u' + kscale K u + M g(u) (g polynomial, ascending coefficients)."""

    M: object
    K: object
    u0: np.ndarray
    dofs: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    g: object = None          # g(t) -> values at dofs
    kscale: float = 1.0
    poly: tuple | None = None  # semilinear reaction coefficients


def stage_values(tab, u_b, G, dt, unknown):
    """DAE boundary stage values (bcs.py:58-96)."""
    if unknown == "value":
        return G
    W = (G - u_b[None, :]) / dt
    return W if unknown == "w" else np.linalg.solve(tab.A, W)


class Stepper:
    """Fully coupled / DIRK / Newton steps with the reference's control flow
    (stepper.py:144-605).  form in {'ai', 'ia', 'value', 'dirk'}."""

    def __init__(self, prob: Problem, tab: Tab, dt, form="ai", pc="jacobi", block="lu",
                 inner_rtol=1e-6, rtol=1e-8, atol=1e-50, restart=50, maxit=500,
                 newton_rtol=1e-10, newton_atol=1e-12, newton_maxit=50):
        self.p, self.tab, self.dt, self.form = prob, tab, dt, form
        self.pc_kind, self.block, self.inner_rtol = pc, block, inner_rtol
        self.kry = dict(rtol=rtol, atol=atol, restart=restart, maxit=maxit)
        self.newton = (newton_rtol, newton_atol, newton_maxit)
        self.u = np.array(prob.u0, dtype=float)
        self.t = 0.0
        self._pc = None
        self._dirk_blocks = {}
        self.stages = []
        self.reports = []

    # linear fully coupled step (stepper.py:341-364)
    def _linear(self):
        tab, dt, p, u, s, m = self.tab, self.dt, self.p, self.u, self.tab.s, self.p.M.shape[0]
        A = np.asarray(tab.A)
        if self.form == "value":
            C1, C2, unknown = np.eye(s), A, "value"
            rhs = np.tile(p.M @ u, s)
        elif self.form == "ai":
            C1, C2, unknown = np.eye(s), A, "derivative"
            rhs = np.tile(-(p.K @ u), s)
        else:
            C1, C2, unknown = np.linalg.inv(A), np.eye(s), "w"
            rhs = np.tile(-(p.K @ u), s)
        op = lambda v: kron_apply(C1, C2, p.M, [p.K], dt, v)  # noqa: E731
        idx = None
        if len(p.dofs):
            G = np.stack([np.broadcast_to(p.g(self.t + ci * dt), (len(p.dofs),)) for ci in tab.c])
            sv = stage_values(tab, u[p.dofs], G, dt, unknown)
            idx = stage_index(s, m, p.dofs)
            gext = np.zeros(s * m)
            gext[idx] = sv.ravel()
            rhs = rhs - op(gext)
            rhs[idx] = gext[idx]
            sop = constrained(op, idx)
        else:
            sop = op
        if self._pc is None and self.pc_kind is not None:
            self._pc = StagePC(self.pc_kind, tab, p.M, [p.K], dt, "ia" if self.form == "ia" else "ai",
                               p.dofs, self.block, self.inner_rtol)
        x, its, hist = fgmres(sop, rhs, self._pc.apply if self._pc else None, **self.kry)
        if idx is not None:
            x[idx] = gext[idx]
        self.stages.append(x.copy())
        X = x.reshape(s, m)
        if self.form == "value":
            if tab.stiffly_accurate:
                un = X[-1].copy()
            else:
                w = np.linalg.solve(A.T, tab.b)
                un = u + w @ (X - u[None, :])
        else:
            Kst = X if self.form == "ai" else np.linalg.solve(A, X)
            un = u + dt * (tab.b @ Kst)
        return un, (0, its, hist[-1])

    # sequential DIRK (stepper.py:367-424); stage solver exact LU or PCG
    def _dirk(self):
        tab, dt, p, u = self.tab, self.dt, self.p, self.u
        s, m = tab.s, p.M.shape[0]
        A = np.asarray(tab.A)
        sv = None
        if len(p.dofs):
            G = np.stack([np.broadcast_to(p.g(self.t + ci * dt), (len(p.dofs),)) for ci in tab.c])
            sv = stage_values(tab, u[p.dofs], G, dt, "derivative")
        Kst = np.zeros((s, m))
        tot = 0
        for i in range(s):
            acc = u + dt * (A[i, :i] @ Kst[:i]) if i else u.copy()
            rhs = -(p.K @ acc)
            op = lambda v, a=A[i, i]: p.M @ v + dt * a * (p.K @ v)  # noqa: E731
            if sv is not None:
                gext = np.zeros(m)
                gext[p.dofs] = sv[i]
                rhs = rhs - op(gext)
                rhs[p.dofs] = sv[i]
                sop = constrained(op, p.dofs)
            else:
                sop = op
            key = A[i, i]
            if key not in self._dirk_blocks:
                self._dirk_blocks[key] = Block(p.M, p.K, 1.0, dt * key, p.dofs,
                                               "lu" if self.block == "lu" else "pcg",
                                               self.kry["rtol"])
            blk = self._dirk_blocks[key]
            if self.block == "lu":
                ki, its, _ = fgmres(sop, rhs, blk.solve, **self.kry)
            else:
                ki, its = jacobi_pcg(blk.C, rhs, self.kry["rtol"], self.kry["atol"])
            tot += its
            if sv is not None:
                ki[p.dofs] = sv[i]
            Kst[i] = ki
        self.stages.append(Kst.ravel().copy())
        return u + dt * (tab.b @ Kst), (0, tot, 0.0)

    # Newton on stage derivatives for the semilinear form (stepper.py:474-569)
    def _newton(self):
        tab, dt, p, u = self.tab, self.dt, self.p, self.u
        s, m = tab.s, p.M.shape[0]
        A = np.asarray(tab.A)
        c = np.asarray(p.poly, dtype=float)
        dc = np.polynomial.polynomial.polyder(c)
        x = np.zeros(s * m)
        rt, at, mx = self.newton
        hist, ktot = [], 0
        for it in range(mx + 1):
            X = x.reshape(s, m)
            U = u[None, :] + dt * (A @ X)
            R = np.stack([p.M @ X[i] + p.kscale * (p.K @ U[i])
                          + p.M @ np.polynomial.polynomial.polyval(U[i], c) for i in range(s)]).ravel()
            nr = float(np.linalg.norm(R))
            hist.append(nr)
            if nr <= max(rt * hist[0], at):
                break
            if it == mx:
                raise RuntimeError("oracle Newton did not converge")
            Ds = [np.polynomial.polynomial.polyval(U[i], dc) for i in range(s)]
            Ks = [(p.kscale * p.K + p.M @ sp.diags(Ds[i])).tocsr() for i in range(s)]
            op = lambda v: kron_apply(np.eye(s), A, p.M, Ks, dt, v)  # noqa: E731
            if self.block == "lu":
                pc = StagePC(self.pc_kind, tab, p.M, Ks, dt, "ai", p.dofs, "lu")
            else:  # SPD lumped-reaction surrogate blocks with Jacobi-PCG
                lump = np.asarray(p.M.sum(axis=1)).ravel()
                surr = [(p.kscale * p.K + sp.diags(lump * Ds[i])).tocsr() for i in range(s)]
                pc = StagePC(self.pc_kind, tab, p.M, surr, dt, "ai", p.dofs, "pcg", self.inner_rtol)
            dx, its, _ = fgmres(op, -R, pc.apply, **self.kry)
            ktot += its
            x = x + dx
        self.stages.append(x.copy())
        X = x.reshape(s, m)
        return u + dt * (tab.b @ X), (len(hist) - 1, ktot, hist[-1])

    def setup(self):
        """Build the preconditioner / DIRK stage block now (the reference's
        cli.run_precond_bench forces setup before timing, cli.py:224-242)."""
        tab, p, dt = self.tab, self.p, self.dt
        if self.form == "dirk":
            A = np.asarray(tab.A)
            for key in sorted(set(np.diag(A).tolist())):
                if key not in self._dirk_blocks:
                    self._dirk_blocks[key] = Block(p.M, p.K, 1.0, dt * key, p.dofs,
                                                   "lu" if self.block == "lu" else "pcg",
                                                   self.kry["rtol"])
        elif self.p.poly is None and self._pc is None and self.pc_kind is not None:
            self._pc = StagePC(self.pc_kind, tab, p.M, [p.K], dt, "ia" if self.form == "ia" else "ai",
                               p.dofs, self.block, self.inner_rtol)

    def reset(self, u0=None):
        """Back to the initial state (caches kept)."""
        self.u = np.array(self.p.u0 if u0 is None else u0, dtype=float)
        self.t = 0.0
        self.stages.clear()
        self.reports.clear()

    def step(self):
        if self.form == "dirk":
            un, rep = self._dirk()
        elif self.p.poly is not None:
            un, rep = self._newton()
        else:
            un, rep = self._linear()
        self.u = un
        self.t += self.dt
        self.reports.append(rep)
        return un


# ------------------------------------------------------------ config recipes

RADAU3_DT = 1e-3


def config(k, n=None, block="pcg"):
    """Problem + stepper settings of BASELINE.json configs 1..5 (optionally
    at a reduced grid size n).  Recipe fixed in SURVEY.md section 8(d)."""
    if k == 1:
        n = n or 32
        dim, tab, dt, steps, form, pc, rtol, seed = 2, radau(2), 1.0 / 32, 10, "ai", "jacobi", 1e-12, 0
    elif k == 2:
        n = n or 1024
        dim, tab, dt, steps, form, pc, rtol, seed = 2, radau(3), 1e-3, 20, "value", "gs-lower", 1e-12, 1
    elif k == 3:
        n = n or 96
        dim, tab, dt, steps, form, pc, rtol, seed = 3, gauss(4), 5e-3, 10, "ai", "schur", 1e-12, 2
    elif k == 4:
        n = n or 2048
        dim, tab, dt, steps, form, pc, rtol, seed = 2, alexander(), 1e-3, 50, "dirk", None, 1e-12, 3
    elif k == 5:
        n = n or 1024
        dim, tab, dt, steps, form, pc, rtol, seed = 2, radau(3), 1e-3, 20, "ai", "jacobi", 1e-10, 4
    else:
        raise ValueError(k)
    M, K = p1_matrices(dim, n)
    X = grid_coords(dim, n)
    m = X.shape[0]
    noise = np.random.default_rng(seed).uniform(-1.0, 1.0, size=m)
    prod = np.prod(np.sin(np.pi * X), axis=1)
    if k in (1, 2):
        u0 = prod + 0.01 * noise
    elif k == 3:
        u0 = prod + 0.01 * noise
    elif k == 4:
        u0 = noise.copy()
    else:
        u0 = 0.1 * noise
    dofs = grid_boundary(dim, n) if k != 5 else np.empty(0, dtype=np.int64)
    g = None
    if k == 3:
        xb = X[dofs, 0]
        g = lambda t: np.exp(-t) * np.sin(np.pi * xb)  # noqa: E731
        u0[dofs] = g(0.0)
    elif k != 5:
        zb = np.zeros(len(dofs))
        g = lambda t: zb  # noqa: E731
        u0[dofs] = 0.0
    prob = Problem(M=M, K=K, u0=u0, dofs=dofs, g=g)
    if k == 5:
        prob.kscale = 0.02 ** 2
        prob.poly = (0.0, -1.0, 0.0, 1.0)
    settings = dict(form=form, pc=pc, block=block, inner_rtol=1e-6 if k != 4 else rtol, rtol=rtol)
    if k == 5:
        settings.update(newton_rtol=1e-10, newton_atol=1e-10)
    return dict(problem=prob, tab=tab, dt=dt, steps=steps, dim=dim, n=n, settings=settings)


def run_config(k, n=None, steps=None, block="pcg", keep_stages=True):
    cfg = config(k, n, block)
    st = Stepper(cfg["problem"], cfg["tab"], cfg["dt"], **cfg["settings"])
    for _ in range(steps if steps is not None else cfg["steps"]):
        st.step()
        if not keep_stages:
            st.stages.clear()
    return st


# ------------------------------------------------------------------ sketches


def sketch_rows(m, nproj=32, seed=20240313):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((nproj, m))


def sketch(v, P=None, nsamp=4096):
    """Size-independent fingerprint of a long vector: norm, sum, a strided
    sample and Gaussian projections (relative L2 of a difference is read
    off the projections)."""
    v = np.asarray(v, dtype=float)
    m = len(v)
    step = max(1, m // nsamp)
    P = sketch_rows(m) if P is None else P
    return dict(norm=float(np.linalg.norm(v)), sum=float(v.sum()),
                idx=np.arange(0, m, step), sample=v[::step].copy(), proj=P @ v)


def sketch_rel_err(a: dict, b: dict):
    """Relative L2 differences read off two sketches (projection and sample)."""
    pa, pb = np.asarray(a["proj"]), np.asarray(b["proj"])
    proj = float(np.linalg.norm(pa - pb) / max(np.linalg.norm(pb), 1e-300))
    sa, sb = np.asarray(a["sample"]), np.asarray(b["sample"])
    samp = float(np.linalg.norm(sa - sb) / max(np.linalg.norm(sb), 1e-300))
    return proj, samp
