"""Butcher tableaux and their s-by-s algebra (host side; s <= 8).

Drop-in for implicitrk.tableaux (/root/reference/pkg/src/implicitrk/tableaux.py):
same classes, constructors, flags, decompositions and text formats, plus the
two pieces the reference lacks and north_star needs:

* ``gauss_legendre(s)`` — Gauss collocation (registered as
  ``"gauss-legendre:s"``; the bare ``"gauss"`` family keeps raising, as
  tests/test_tableaux.py:289-290 require);
* ``real_schur(tab)`` / ``schur_blocks`` — A = Q T Q^T with the 2x2 blocks
  standardised, the data of the tableau-eigen/real-Schur preconditioner.

Collocation tableaux are computed from the moment conditions
sum_j a_ij c_j^(k-1) = c_i^k / k, k = 1..s (an s-by-s Vandermonde solve),
which is algebraically the reference's Lagrange-integral construction
(tableaux.py:146-170).
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

STRUCT_TOL = 1e-12  # tableaux.py:16-17
ROOT_TOL = 1e-14    # tableaux.py:18-19


class UnsupportedStageCountError(ValueError):
    """Requested stage count outside the supported range of a family."""


class SingularFactorizationError(ArithmeticError):
    """A leading principal minor vanished during unpivoted elimination
    (tableaux.py:26-34)."""

    def __init__(self, stage, pivot):
        self.stage = stage
        self.pivot = pivot
        super().__init__(f"singular LDU factorization: pivot {pivot:.3e} at stage {stage}")


def _readonly(x):
    arr = np.array(x, dtype=np.float64, copy=True, order="C")
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class ButcherTableau:
    """(A, b, c) with order metadata; immutable (tableaux.py:43-94)."""

    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    formal_order: int
    stage_order: int
    name: str
    weak_stage_order: int = 0

    def __post_init__(self):
        for fld in ("A", "b", "c"):
            object.__setattr__(self, fld, _readonly(getattr(self, fld)))
        s = len(self.b)
        if self.b.ndim != 1 or self.A.shape != (s, s) or self.c.shape != (s,):
            raise ValueError(
                f"tableau {self.name!r}: A must be {s}x{s} and c length {s}, "
                f"got A {self.A.shape}, c {self.c.shape}"
            )
        if abs(float(np.sum(self.b)) - 1.0) > STRUCT_TOL:
            raise ValueError(f"tableau {self.name!r}: weights sum to {np.sum(self.b)!r}, not 1")

    @property
    def s(self) -> int:
        return int(self.b.shape[0])

    @property
    def stiffly_accurate(self) -> bool:
        return is_stiffly_accurate(self)

    @property
    def lower_triangular(self) -> bool:
        return is_lower_triangular(self)

    @property
    def invertible(self) -> bool:
        # A is read-only: the LU test runs once per tableau (steppers ask every step)
        hit = self.__dict__.get("_invertible")
        if hit is None:
            hit = is_invertible(self)
            object.__setattr__(self, "_invertible", hit)
        return hit

    def __repr__(self):
        return f"ButcherTableau({self.name!r}, s={self.s}, order={self.formal_order})"


@dataclass(frozen=True)
class LduFactors:
    """A = L diag(D) U, unit triangular L and U (tableaux.py:97-105)."""

    L: np.ndarray
    D: np.ndarray
    U: np.ndarray

    def reconstruct(self) -> np.ndarray:
        return (self.L * self.D[None, :]) @ self.U


@dataclass(frozen=True)
class AdditiveSplit:
    """A = L_strict + diag(D_diag) + U_strict (tableaux.py:108-117)."""

    L_strict: np.ndarray
    D_diag: np.ndarray
    U_strict: np.ndarray

    def reconstruct(self) -> np.ndarray:
        return self.L_strict + np.diag(self.D_diag) + self.U_strict


# ---------------------------------------------------------------- families


def _collocation(c: np.ndarray):
    """A and b from the collocation moment conditions at nodes c."""
    s = len(c)
    powers = np.arange(s)
    V = c[None, :] ** powers[:, None]            # V[k, j] = c_j^k
    W = c[:, None] ** (powers[None, :] + 1) / (powers[None, :] + 1)  # c_i^(k+1)/(k+1)
    A = np.linalg.solve(V, W.T).T                # A V^T = W
    b = np.linalg.solve(V, 1.0 / (powers + 1))
    return A, b


def _polish(poly, dpoly, x):
    for _ in range(60):
        r = poly(x)
        if np.max(np.abs(r)) < ROOT_TOL:
            break
        x = x - r / dpoly(x)
    return x


def _radau_right_nodes(s: int) -> np.ndarray:
    # zeros of P_s(2x-1) - P_{s-1}(2x-1): right Radau points on [0, 1]
    L = np.polynomial.legendre.Legendre
    Poly = np.polynomial.Polynomial
    p = (L.basis(s) - L.basis(s - 1)).convert(kind=Poly)(Poly([-1.0, 2.0]))
    p = p / np.max(np.abs(p.coef))
    x = _polish(p, p.deriv(), np.sort(np.real(p.roots())))
    if np.max(np.abs(p(x))) >= 1e-12:
        raise ArithmeticError(f"Radau node refinement stalled for s={s}")
    x[-1] = 1.0  # exact endpoint: last row of A reproduces b
    return x


def radau_iia(s: int) -> ButcherTableau:
    """RadauIIA, order 2s-1, stage order s, stiffly accurate (tableaux.py:173-188)."""
    if not 1 <= s <= 5:
        raise UnsupportedStageCountError(f"radau_iia supports 1 <= s <= 5, got {s}")
    if s == 1:
        return ButcherTableau([[1.0]], [1.0], [1.0], 1, 1, "radau-iia:1")
    c = _radau_right_nodes(s)
    A, b = _collocation(c)
    A[-1, :] = b  # stiff accuracy holds exactly by construction
    return ButcherTableau(A, b, c, 2 * s - 1, s, f"radau-iia:{s}")


def gauss_legendre(s: int) -> ButcherTableau:
    """Gauss-Legendre collocation, order 2s, stage order s, A-stable, not
    stiffly accurate.  New relative to the reference."""
    if not 1 <= s <= 6:
        raise UnsupportedStageCountError(f"gauss_legendre supports 1 <= s <= 6, got {s}")
    x, _ = np.polynomial.legendre.leggauss(s)
    c = 0.5 * (x + 1.0)
    A, b = _collocation(c)
    return ButcherTableau(A, b, c, 2 * s, s, f"gauss-legendre:{s}")


def lobatto_iiic(s: int) -> ButcherTableau:
    """LobattoIIIC, s in {2, 3} (tableaux.py:191-212)."""
    if s == 2:
        data = ([[1 / 2, -1 / 2], [1 / 2, 1 / 2]], [1 / 2, 1 / 2], [0.0, 1.0])
    elif s == 3:
        data = (
            [[1 / 6, -1 / 3, 1 / 6], [1 / 6, 5 / 12, -1 / 12], [1 / 6, 2 / 3, 1 / 6]],
            [1 / 6, 2 / 3, 1 / 6],
            [0.0, 0.5, 1.0],
        )
    else:
        raise UnsupportedStageCountError(f"lobatto_iiic supports s in {{2, 3}}, got {s}")
    return ButcherTableau(*data, 2 * s - 2, s - 1, f"lobatto-iiic:{s}")


def _alexander_gamma() -> float:
    # root of x^3 - 3x^2 + 3/2 x - 1/6 in (1/6, 1/2)
    p = np.polynomial.Polynomial([-1 / 6, 1.5, -3.0, 1.0])
    roots = np.real(p.roots()[np.abs(np.imag(p.roots())) < 1e-12])
    g = float(roots[(roots > 1 / 6) & (roots < 0.5)][0])
    g = float(_polish(p, p.deriv(), np.array([g]))[0])
    if abs(p(g)) >= ROOT_TOL:
        raise ArithmeticError("Alexander diagonal root refinement stalled")
    return g


def alexander_dirk() -> ButcherTableau:
    """Alexander's 3-stage L-stable SDIRK, gamma ~ 0.4358665215 (tableaux.py:215-254)."""
    g = _alexander_gamma()
    b1 = -1.5 * g * g + 4.0 * g - 0.25
    b2 = 1.0 - g - b1
    A = [[g, 0.0, 0.0], [(1.0 - g) / 2.0, g, 0.0], [b1, b2, g]]
    return ButcherTableau(A, [b1, b2, g], [g, (1.0 + g) / 2.0, 1.0], 3, 1, "alexander")


def wsodirk433() -> ButcherTableau:
    """Four-stage DIRK with weak stage order 3, coefficients at their
    published eight digits (tableaux.py:257-277)."""
    rows = [
        [0.13756544],
        [0.56695123, 0.23483889],
        [-1.08354073, 2.96618224, 0.44915522],
        [0.59761292, -0.43420998, -0.05305815, 0.88965521],
    ]
    A = np.zeros((4, 4))
    for i, r in enumerate(rows):
        A[i, : len(r)] = r
    return ButcherTableau(
        A, A[3].copy(), [0.13756544, 0.80179012, 2.33179673, 1.0], 3, 1, "wsodirk433",
        weak_stage_order=3,
    )


# ------------------------------------------------------ splits and flags


def ldu_factor(tab: ButcherTableau) -> LduFactors:
    """Unpivoted Doolittle A = L diag(D) U (tableaux.py:284-304)."""
    s = tab.s
    work = np.array(tab.A, dtype=np.float64)
    L = np.eye(s)
    for k in range(s):
        piv = work[k, k]
        if abs(piv) < 1e-14:
            raise SingularFactorizationError(k + 1, piv)
        mult = work[k + 1 :, k] / piv
        L[k + 1 :, k] = mult
        work[k + 1 :, k:] -= np.outer(mult, work[k, k:])
        work[k + 1 :, k] = 0.0
    D = np.diag(work).copy()
    return LduFactors(L=L, D=D, U=work / D[:, None])


def additive_split(tab: ButcherTableau) -> AdditiveSplit:
    A = np.array(tab.A, dtype=np.float64)
    return AdditiveSplit(np.tril(A, -1), np.diag(A).copy(), np.triu(A, 1))


def is_stiffly_accurate(tab: ButcherTableau) -> bool:
    return bool(np.max(np.abs(tab.A[-1] - tab.b)) <= STRUCT_TOL)


def is_lower_triangular(tab: ButcherTableau) -> bool:
    if tab.s == 1:
        return True
    return bool(np.max(np.abs(np.triu(tab.A, 1))) <= STRUCT_TOL)


def is_invertible(tab: ButcherTableau) -> bool:
    """Partial-pivoting LU test with relative threshold 1e-12 (tableaux.py:323-331)."""
    import scipy.linalg

    nrm = np.linalg.norm(tab.A)
    if nrm == 0.0:
        return False
    lu, _ = scipy.linalg.lu_factor(np.array(tab.A), check_finite=False)
    return bool(np.min(np.abs(np.diag(lu))) > 1e-12 * nrm)


def order_condition_residuals(tab: ButcherTableau, p: int, stage_p: int | None = None):
    """(b_res, stage_res): |b.c^(k-1) - 1/k| and |A c^(k-1) - c^k/k| (tableaux.py:334-360)."""
    if p < 1:
        raise ValueError("p must be >= 1")
    q = tab.stage_order if stage_p is None else stage_p
    ks = np.arange(1, p + 1)
    b_res = np.abs(np.array([tab.b @ tab.c ** (k - 1) for k in ks]) - 1.0 / ks)
    stage = [np.abs(tab.A @ tab.c ** (k - 1) - tab.c**k / k) for k in range(1, q + 1)]
    return b_res, np.array(stage).reshape(q, tab.s)


def row_sum_residuals(tab: ButcherTableau) -> np.ndarray:
    return np.abs(np.sum(tab.A, axis=1) - tab.c)


# ------------------------------------------------------------ real Schur


@dataclass(frozen=True)
class SchurData:
    """A = Q T Q^T with T block diagonal part split into 1x1 / 2x2 blocks.

    ``blocks`` lists (start, size) of the diagonal blocks of T in Q's column
    order; every 2x2 block is standardised to [[a, b], [c, a]] with b c < 0
    (complex pair a +/- i sqrt(-b c)).
    """

    Q: np.ndarray
    T: np.ndarray
    blocks: tuple


def real_schur(A) -> SchurData:
    """Real Schur form of an s-by-s matrix with standardised 2x2 blocks."""
    import scipy.linalg

    A = np.asarray(A, dtype=np.float64)
    T, Q = scipy.linalg.schur(A, output="real")
    s = A.shape[0]
    blocks = []
    i = 0
    while i < s:
        if i + 1 < s and abs(T[i + 1, i]) > 1e-14 * max(1.0, np.abs(T).max()):
            # standardise to equal diagonals with a Givens rotation
            a, b, c, d = T[i, i], T[i, i + 1], T[i + 1, i], T[i + 1, i + 1]
            G = _standardize_rotation(a, b, c, d)
            R = np.eye(s)
            R[i : i + 2, i : i + 2] = G
            T = R.T @ T @ R
            Q = Q @ R
            blocks.append((i, 2))
            i += 2
        else:
            blocks.append((i, 1))
            i += 1
    for st, sz in blocks:
        if sz == 2:
            T[st + 1, st + 1] = T[st, st] = 0.5 * (T[st, st] + T[st + 1, st + 1])
    T.setflags(write=False)
    Q.setflags(write=False)
    return SchurData(Q=Q, T=T, blocks=tuple(blocks))


def _standardize_rotation(a, b, c, d):
    # rotation [[cs, -sn], [sn, cs]] making the diagonal entries of G^T B G equal
    # (LAPACK dlanv2 convention): tan(2 th) = (a - d) / (b + c)
    th = 0.5 * np.arctan2(a - d, b + c)
    cs, sn = np.cos(th), np.sin(th)
    G = np.array([[cs, -sn], [sn, cs]])
    B = G.T @ np.array([[a, b], [c, d]]) @ G
    if abs(B[0, 0] - B[1, 1]) > 1e-12 * max(1.0, abs(a) + abs(d)):
        th += np.pi / 4
        cs, sn = np.cos(th), np.sin(th)
        G = np.array([[cs, -sn], [sn, cs]])
    return G


# ------------------------------------------------------------ text formats


def format_butcher(tab: ButcherTableau, digits: int = 15) -> str:
    """Aligned plain-text Butcher array (tableaux.py:366-381)."""
    w = digits + 7

    def cell(v):
        return f"{v: .{digits}g}".rjust(w)

    buf = io.StringIO()
    for i in range(tab.s):
        buf.write(cell(tab.c[i]) + " |" + "".join(cell(v) for v in tab.A[i]) + "\n")
    buf.write("-" * (w + 1) + "+" + "-" * (w * tab.s) + "\n")
    buf.write(" " * (w + 1) + "|" + "".join(cell(v) for v in tab.b) + "\n")
    return buf.getvalue()


def to_csv(tab: ButcherTableau) -> str:
    """``stage,c,a_1..a_s`` rows then a ``b,,...`` row (tableaux.py:384-393)."""
    head = "stage,c," + ",".join(f"a_{j + 1}" for j in range(tab.s))
    body = [
        f"{i + 1},{float(tab.c[i])!r}," + ",".join(repr(float(v)) for v in tab.A[i])
        for i in range(tab.s)
    ]
    tail = "b,," + ",".join(repr(float(v)) for v in tab.b)
    return "\n".join([head, *body, tail]) + "\n"


_FAMILIES = {
    "radau-iia": (radau_iia, True),
    "gauss-legendre": (gauss_legendre, True),
    "lobatto-iiic": (lobatto_iiic, True),
    "alexander": (alexander_dirk, False),
    "wsodirk433": (wsodirk433, False),
}


def from_spec(spec: str) -> ButcherTableau:
    """``family[:stages]`` -> tableau (tableaux.py:404-421)."""
    family, _, count = spec.partition(":")
    if family not in _FAMILIES:
        raise UnsupportedStageCountError(f"unknown tableau family {family!r}")
    ctor, staged = _FAMILIES[family]
    if staged:
        if not count:
            raise UnsupportedStageCountError(f"family {family!r} needs a stage count")
        return ctor(int(count))
    tab = ctor()
    if count and int(count) != tab.s:
        raise UnsupportedStageCountError(f"family {family!r} has exactly {tab.s} stages")
    return tab
