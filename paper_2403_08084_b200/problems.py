"""Structured grids, on-device P1/Q1 assembly and model problems
(drop-in for the assembly part of implicitrk.problems,
/root/reference/pkg/src/implicitrk/problems.py).

* ``StructuredGrid(dim, n)``: dim 1, 2 (as the reference) and 3 (new);
  vertices lexicographic with x fastest (problems.py:25-64).
* ``assemble_heat(grid)``: the reference's operators (1D P1, 2D Q1 Kronecker
  form, problems.py:80-99), assembled by libirk on the device; dim 3 gives
  the P1 Kuhn-tetrahedra operators.
* ``assemble_p1(grid)``: P1 on right triangles (2D, diagonal
  (i,j)-(i+1,j+1)) or Kuhn tetrahedra (3D) — the north_star configs.
* model problems used by the bench configs: ``heat_problem`` and
  ``allen_cahn_problem``; the scalar ODE test set of the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import ctypes as C
import numpy as np

from . import sparsela as la
from ._lib import call, ctx
from .bcs import DirichletBC
from .sparsela import SparseMatrix
from .stepper import SemidiscreteProblem, SemilinearForm, zero_load


@dataclass(frozen=True)
class StructuredGrid:
    """Uniform grid on [0,1]^dim, vertices lexicographic with x fastest."""

    dim: int
    n: int

    def __post_init__(self):
        if self.dim not in (1, 2, 3):
            raise ValueError("dim must be 1, 2 or 3")
        if self.n < 2:
            raise ValueError("need at least 2 cells per direction")

    @property
    def h(self) -> float:
        return 1.0 / self.n

    @property
    def npoints(self) -> int:
        return (self.n + 1) ** self.dim

    def coords(self) -> np.ndarray:
        """(npoints, dim) vertex coordinates, x fastest."""
        x = np.linspace(0.0, 1.0, self.n + 1)
        grids = np.meshgrid(*([x] * self.dim), indexing="ij")
        # meshgrid 'ij' makes the first axis slowest; reverse so x is fastest
        cols = [g.transpose(tuple(range(self.dim))[::-1]).ravel() for g in grids]
        return np.column_stack(cols)

    def boundary_dofs(self) -> np.ndarray:
        n1 = self.n + 1
        idx = np.arange(self.npoints)
        on = np.zeros(self.npoints, dtype=bool)
        for d in range(self.dim):
            k = (idx // n1**d) % n1
            on |= (k == 0) | (k == self.n)
        return np.nonzero(on)[0].astype(np.int64)


def _assemble(kind: str, grid: StructuredGrid):
    hM, hK = C.c_void_p(), C.c_void_p()
    if kind == "q1":
        call("irk_mat_assemble_q1", ctx(), grid.n, C.byref(hM), C.byref(hK))
    else:
        call("irk_mat_assemble_p1", ctx(), grid.dim, grid.n, C.byref(hM), C.byref(hK))
    return (SparseMatrix._from_device(la.DeviceMatrix(hM)),
            SparseMatrix._from_device(la.DeviceMatrix(hK)))


def assemble_heat(grid: StructuredGrid):
    """(M, K, boundary dofs) with the reference's elements (problems.py:80-99):
    1D P1, 2D Q1 (M1 (x) M1, K1 (x) M1 + M1 (x) K1); 3D P1 Kuhn tetrahedra."""
    kind = "q1" if grid.dim == 2 else "p1"
    M, K = _assemble(kind, grid)
    return M, K, grid.boundary_dofs()


def assemble_p1(grid: StructuredGrid):
    """(M, K, boundary dofs) for P1 on the simplicial split of the grid:
    intervals (1D), right triangles along (i,j)-(i+1,j+1) (2D), Kuhn
    tetrahedra along (0,0,0)-(1,1,1) (3D).  M and K share one pattern,
    K's exact zeros stay stored."""
    M, K = _assemble("p1", grid)
    return M, K, grid.boundary_dofs()


def interpolate(grid: StructuredGrid, fn: Callable, t: float) -> np.ndarray:
    """Vertex interpolant of fn(t, x[, y[, z]])."""
    X = grid.coords()
    return np.asarray(fn(t, *(X[:, d] for d in range(grid.dim))), dtype=float)


# ------------------------------------------------------- bench problems


def seeded_noise(m: int, seed: int) -> np.ndarray:
    """U[-1, 1] nodal noise over all m vertices in numbering order."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=m)


def heat_problem(grid: StructuredGrid, u0: np.ndarray, g: Optional[Callable] = None,
                 element: str = "p1", dirichlet: bool = True, name: str = "") -> SemidiscreteProblem:
    """Heat equation M u' + K u = 0 with Dirichlet data g(t, x..) on every
    boundary vertex (homogeneous when g is None).  Boundary entries of u0
    are set to g(0)."""
    M, K, bd = assemble_p1(grid) if element == "p1" else assemble_heat(grid)
    m = grid.npoints
    u0 = np.array(u0, dtype=float)
    bc = None
    if dirichlet:
        if g is None:
            zeros = np.zeros(len(bd))
            gfun = lambda t: zeros  # noqa: E731
            gdot = lambda t: zeros  # noqa: E731
        else:
            Xb = grid.coords()[bd]
            args = tuple(Xb[:, d] for d in range(grid.dim))
            gfun = lambda t: np.asarray(g(t, *args), dtype=float)  # noqa: E731
            gdot = None
        bc = DirichletBC(dofs=bd, g=gfun, g_dot=gdot)
        u0[bd] = gfun(0.0)
    return SemidiscreteProblem(m=m, mass=M, stiffness=K, load=zero_load(m), dirichlet=bc,
                               u0=u0, grid=grid, name=name or f"heat-p1-{grid.dim}d-n{grid.n}")


def allen_cahn_problem(grid: StructuredGrid, eps: float, u0: np.ndarray,
                       name: str = "") -> SemidiscreteProblem:
    """Allen-Cahn u_t = eps^2 Lap u + u - u^3, homogeneous Neumann, P1:
    M u' + eps^2 K u + M (u^3 - u) = 0 (consistent-mass reaction)."""
    M, K, _ = assemble_p1(grid)
    return SemidiscreteProblem(
        m=grid.npoints, mass=M, stiffness=K, u0=np.array(u0, dtype=float), grid=grid,
        semilinear=SemilinearForm(kscale=eps * eps, coef=(0.0, -1.0, 0.0, 1.0)),
        name=name or f"allen-cahn-{grid.dim}d-n{grid.n}")


# ------------------------------------------------------ scalar ODE set


@dataclass
class OdeTestProblem:
    name: str
    problem: SemidiscreteProblem
    exact: Callable[[float], float]


def _scalar(v):
    return SparseMatrix.from_dense([[float(v)]])


def dahlquist(lam: float = -1.0) -> OdeTestProblem:
    """y' = lam y, y(0) = 1 (problems.py:304-318)."""
    p = SemidiscreteProblem(m=1, mass=_scalar(1.0), stiffness=_scalar(-lam),
                            load=lambda t: np.zeros(1), u0=np.ones(1), name="dahlquist")
    return OdeTestProblem("dahlquist", p, lambda t: float(np.exp(lam * t)))


def prothero_robinson(lam: float = -1e4) -> OdeTestProblem:
    """y' = lam (y - sin t) + cos t (problems.py:321-340)."""
    p = SemidiscreteProblem(m=1, mass=_scalar(1.0), stiffness=_scalar(-lam),
                            load=lambda t: np.array([np.cos(t) - lam * np.sin(t)]),
                            u0=np.zeros(1), name="prothero-robinson")
    return OdeTestProblem("prothero-robinson", p, lambda t: float(np.sin(t)))


def riccati() -> OdeTestProblem:
    """y' = y^2, y(0) = 1 (problems.py:343-353)."""
    p = SemidiscreteProblem(m=1, mass=_scalar(1.0), residual=lambda t, u, udot: udot - u**2,
                            jacobian_u=lambda t, u: _scalar(-2.0 * u[0]), u0=np.ones(1),
                            name="riccati")
    return OdeTestProblem("riccati", p, lambda t: float(1.0 / (1.0 - t)))


def ode_suite():
    return [dahlquist(), prothero_robinson(), riccati()]
