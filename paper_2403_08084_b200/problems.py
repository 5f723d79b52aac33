"""Structured grids, on-device P1/Q1 assembly and model problems
(drop-in for the assembly part of implicitrk.problems,
/root/reference/pkg/src/implicitrk/problems.py).

* ``StructuredGrid(dim, n)``: dim 1, 2, validated exactly as the reference
  (problems.py:25-64; dim 3 raises ValueError there, so it does here);
  ``CubeGrid(n)`` / ``structured_grid(3, n)``: the unit cube (new, config 3).
  Vertices lexicographic with x fastest.
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
from ._lib import call, ctx, ptr
from .bcs import DirichletBC
from .sparsela import SparseMatrix
from .stepper import SemidiscreteProblem, SemilinearForm, zero_load


@dataclass(frozen=True)
class StructuredGrid:
    """Uniform grid on [0,1]^dim, vertices lexicographic with x fastest."""

    dim: int
    n: int

    _DIMS = (1, 2)  # the reference's grids (problems.py:33-37)

    def __post_init__(self):
        if self.dim not in self._DIMS:
            raise ValueError("dim must be 1 or 2" if self._DIMS == (1, 2)
                             else f"dim must be one of {self._DIMS}")
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



@dataclass(frozen=True)
class CubeGrid(StructuredGrid):
    """The unit cube [0,1]^3 (new: the reference's grids are 1D/2D only and
    reject dim 3), for the P1 Kuhn-tetrahedra workloads (config 3)."""

    _DIMS = (1, 2, 3)


def structured_grid(dim: int, n: int) -> StructuredGrid:
    """StructuredGrid for dim 1, 2; CubeGrid for dim 3."""
    return CubeGrid(dim, n) if dim == 3 else StructuredGrid(dim, n)


def _assemble(kind: str, grid: StructuredGrid):
    hM, hK = C.c_void_p(), C.c_void_p()
    if kind == "q1":
        call("irk_mat_assemble_q1", ctx(), grid.n, C.byref(hM), C.byref(hK))
    else:
        call("irk_mat_assemble_p1", ctx(), grid.dim, grid.n, C.byref(hM), C.byref(hK))
    M = SparseMatrix._from_device(la.DeviceMatrix(hM))
    K = SparseMatrix._from_device(la.DeviceMatrix(hK))
    if kind == "p1":
        # nested P1 grids: blocks built from this pair get the geometric
        # multigrid inner solver (sparsela.BlockFactorization)
        M._p1_grid = K._p1_grid = (grid.dim, grid.n)
    return M, K


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


# ------------------------------------------- manufactured solutions (MMS)
# SURVEY §8 f row 3: load vectors and error norms of the forced heat
# problems, assembled / reduced on the device (libirk irk_fe_*).

_GAUSS2 = ((0.5 - 0.5 / np.sqrt(3.0), 0.5), (0.5 + 0.5 / np.sqrt(3.0), 0.5))


@dataclass(frozen=True)
class ManufacturedSolution:
    """Exact solution with its time derivative, gradient and forcing
    f = u_t - Lap u (problems.py:102-111)."""

    dim: int
    u: Callable
    u_t: Callable
    grad: tuple
    f: Callable


def _device_forcing(fn, kind):
    fn._irk_mms_kind = kind  # evaluated by irk_fe_mms_forcing on the device
    return fn


def heat_mms_2d() -> ManufacturedSolution:
    """u(t, x, y) = exp(-0.1 t) sin(pi x) cos(pi y) (problems.py:113-129)."""

    def u(t, x, y):
        return np.exp(-0.1 * t) * np.sin(np.pi * x) * np.cos(np.pi * y)

    def gx(t, x, y):
        return np.pi * np.exp(-0.1 * t) * np.cos(np.pi * x) * np.cos(np.pi * y)

    def gy(t, x, y):
        return -np.pi * np.exp(-0.1 * t) * np.sin(np.pi * x) * np.sin(np.pi * y)

    def f(t, x, y):
        return (2 * np.pi**2 - 0.1) * u(t, x, y)

    return ManufacturedSolution(dim=2, u=u, u_t=lambda t, x, y: -0.1 * u(t, x, y),
                                grad=(gx, gy), f=_device_forcing(f, 2))


def heat_mms_1d() -> ManufacturedSolution:
    """u(t, x) = exp(-0.1 t) sin(pi x) (problems.py:132-149)."""

    def u(t, x):
        return np.exp(-0.1 * t) * np.sin(np.pi * x)

    def f(t, x):
        return (np.pi**2 - 0.1) * u(t, x)

    return ManufacturedSolution(
        dim=1, u=u, u_t=lambda t, x: -0.1 * u(t, x),
        grad=(lambda t, x: np.pi * np.exp(-0.1 * t) * np.cos(np.pi * x),),
        f=_device_forcing(f, 1))


def _fe_grid(grid: StructuredGrid):
    if grid.dim not in (1, 2):
        raise ValueError("the manufactured-solution problems are 1D (P1) or 2D (Q1)")
    return grid.n ** grid.dim


def _quad_points(grid: StructuredGrid):
    """Physical quadrature points, one tuple of per-element coordinate arrays
    per point of the 2-point Gauss rule (xi outer, eta inner;
    problems.py:171-191)."""
    h, n = grid.h, grid.n
    if grid.dim == 1:
        xl = np.arange(n) * h
        return [(xl + xi * h,) for xi, _ in _GAUSS2]
    ex, ey = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    xl, yl = (ex * h).ravel(), (ey * h).ravel()
    return [(xl + xi * h, yl + eta * h) for xi, _ in _GAUSS2 for eta, _ in _GAUSS2]


def _qdata(grid, fns, t):
    """Device tensor of fn(t, x_q) for every quadrature point q (outer), the
    functions in `fns` (middle) and elements (inner)."""
    ne = _fe_grid(grid)
    cols = []
    for xq in _quad_points(grid):
        for fn in fns:
            v = np.asarray(fn(t, *xq), dtype=np.float64)
            cols.append(np.broadcast_to(v, (ne,)))
    return la.to_dev(np.concatenate(cols))


def assemble_load_device(grid: StructuredGrid, f: Callable, t: float):
    """Load vector (f(t, .), phi_j) as a CUDA tensor: the built-in forcings
    are evaluated on the device, any other callable on the host at the
    quadrature points; the element accumulation runs on the device in the
    reference's order (problems.py:194-202)."""
    ne = _fe_grid(grid)
    kind = getattr(f, "_irk_mms_kind", 0)
    if kind == grid.dim:
        fq = la.dev_empty(ne * 2 ** grid.dim)
        call("irk_fe_mms_forcing", ctx(), kind, grid.n, float(t), ptr(fq))
    else:
        fq = _qdata(grid, (f,), t)
    out = la.dev_empty(grid.npoints)
    call("irk_fe_load", ctx(), grid.dim, grid.n, ptr(fq), ptr(out))
    return out


def assemble_load(grid: StructuredGrid, f: Callable, t: float) -> np.ndarray:
    """Load vector (f(t, .), phi_j) (problems.py:194-202), numpy out."""
    return la.to_host(assemble_load_device(grid, f, t))


def _err_sq(grid, u_h, uex, grads, t):
    _fe_grid(grid)
    u = la.to_dev(u_h)
    ue = _qdata(grid, (uex,), t) if uex is not None else None
    ge = _qdata(grid, grads, t) if grads is not None else None
    out = C.c_double()
    call("irk_fe_error_sq", ctx(), grid.dim, grid.n, ptr(u),
         ptr(ue) if ue is not None else None, ptr(ge) if ge is not None else None,
         C.byref(out))
    return out.value


def l2_error(grid: StructuredGrid, u_h, u_exact: Callable, t: float) -> float:
    """Quadrature L2 norm of u_h - u_exact(t, .) (problems.py:205-212)."""
    return float(np.sqrt(_err_sq(grid, u_h, u_exact, None, t)))


def h1_error(grid: StructuredGrid, u_h, u_exact: Callable, grad_exact: tuple, t: float) -> float:
    """Full H1 norm of the error, L2 plus gradient part (problems.py:215-232)."""
    return float(np.sqrt(_err_sq(grid, u_h, u_exact, tuple(grad_exact), t)))


def fe_l2_norm(grid: StructuredGrid, u_h) -> float:
    """L2 norm of a finite-element function (problems.py:235-239)."""
    return float(np.sqrt(_err_sq(grid, u_h, None, None, 0.0)))


def mms_heat_problem(grid: StructuredGrid,
                     mms: Optional[ManufacturedSolution] = None) -> SemidiscreteProblem:
    """Heat equation with manufactured forcing (device load assembly) and
    Dirichlet data from the exact solution on every boundary vertex
    (problems.py:250-272)."""
    if mms is None:
        mms = heat_mms_2d() if grid.dim == 2 else heat_mms_1d()
    if mms.dim != grid.dim:
        raise ValueError("manufactured solution dimension mismatch")
    M, K, bd = assemble_heat(grid)
    Xb = grid.coords()[bd]
    args = tuple(Xb[:, d] for d in range(grid.dim))
    bc = DirichletBC(dofs=bd, g=lambda t: mms.u(t, *args), g_dot=lambda t: mms.u_t(t, *args))
    return SemidiscreteProblem(
        m=grid.npoints, mass=M, stiffness=K,
        load=lambda t: assemble_load_device(grid, mms.f, t),
        dirichlet=bc, u0=interpolate(grid, mms.u, 0.0), grid=grid,
        name=f"heat-mms-{grid.dim}d-n{grid.n}")


def incompatible_heat_1d(n: int = 10) -> SemidiscreteProblem:
    """1D heat problem, zero initial data, g = 1 at both ends: the DAE
    boundary treatment sees the incompatibility, the ODE one (g' = 0) never
    does (problems.py:275-295)."""
    grid = StructuredGrid(1, n)
    M, K, bd = assemble_heat(grid)
    ones, zeros = np.ones(len(bd)), np.zeros(len(bd))
    bc = DirichletBC(dofs=bd, g=lambda t: ones, g_dot=lambda t: zeros)
    return SemidiscreteProblem(m=grid.npoints, mass=M, stiffness=K, load=zero_load(grid.npoints),
                               dirichlet=bc, u0=np.zeros(grid.npoints), grid=grid,
                               name=f"heat-incompatible-1d-n{n}")


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
