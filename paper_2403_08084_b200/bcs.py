"""Dirichlet data as algebraic stage equations (drop-in for implicitrk.bcs,
/root/reference/pkg/src/implicitrk/bcs.py).

The s-by-|Gamma| stage boundary values are host algebra (one dense s-by-s
solve shared by all constrained dofs, bcs.py:58-96); everything that touches
length-m data — the constrained operator (row identity + column
elimination), the right-hand-side lifting and the stage-value scatter — runs
on the device on the stage-interleaved layout.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Optional

import numpy as np

from . import sparsela as la
from ._lib import call, ctx, hptr, ptr


class BcMethod(Enum):
    DAE = "dae"
    ODE = "ode"


class StageUnknown(Enum):
    """What a stage solve solves for (bcs.py:30-36)."""

    DERIVATIVE = "derivative"
    W = "w"
    VALUE = "value"


@dataclass
class DirichletBC:
    """Constrained dofs with data g(t) (and g'(t) for the ODE method) (bcs.py:39-55)."""

    dofs: np.ndarray
    g: Callable[[float], np.ndarray]
    g_dot: Optional[Callable[[float], np.ndarray]] = None
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        self.dofs = np.asarray(self.dofs, dtype=np.int64)
        if len(self.dofs) and self.dofs.min() < 0:
            raise ValueError("negative dof index in DirichletBC")

    def dofs_dev(self):
        import torch

        d = self._dev.get("dofs")
        if d is None:
            d = self._dev["dofs"] = la.to_dev(self.dofs, dtype=torch.int64)
        return d

    def mask_dev(self, m: int):
        key = ("mask", int(m))
        mk = self._dev.get(key)
        if mk is None:
            mk = self._dev[key] = la.dof_mask(m, self.dofs)
        return mk


_INV_CACHE: dict = {}


def _tableau_inverse(tab):
    key = id(tab)
    hit = _INV_CACHE.get(key)
    if hit is None or hit[0] is not tab:
        hit = _INV_CACHE[key] = (tab, np.linalg.inv(np.asarray(tab.A, dtype=np.float64)))
    return hit[1]


def _values_at(fn, t, shape):
    return np.broadcast_to(np.asarray(fn(t), dtype=np.float64), shape)


def stage_fn_values(fn, times, shape) -> np.ndarray:
    """fn at the stage times, stacked: shape (s, |Gamma|)."""
    return np.stack([_values_at(fn, ti, shape) for ti in times])


class BoundaryPrefetch:
    """Boundary data of the NEXT step evaluated on a helper thread while the
    GPU runs the current step's solve.

    The reference evaluates ``bc.g`` / ``bc.g_dot`` at the s stage times on the
    host at the start of every step (bcs.py:76-93).  At config 3 that is four
    numpy evaluations over 55 298 boundary vertices, ~2 ms during which the
    GPU idles (a third of the step).  ``schedule`` submits the evaluation for
    the stage times the next step will ask for; ``take`` returns it if the key
    (function, times, shape) matches exactly and evaluates inline otherwise,
    so results never depend on the prediction.  User callbacks never run
    concurrently with each other: ``join`` (called at the start of every
    step and before any inline evaluation) waits for a pending evaluation,
    and only linear problems (no user callbacks inside the solve) schedule.
    ``IRK_BC_PREFETCH=0`` or ``TimeStepper.bc_prefetch = False`` disables it.
    """

    MIN_DOFS = 1024

    def __init__(self):
        self._pool = None
        self._key = None
        self._fut = None

    def join(self):
        if self._fut is not None:
            try:
                self._fut.result()
            except Exception:  # re-raised by the inline evaluation of the same call
                pass

    def take(self, fn, times, shape) -> np.ndarray:
        key = (id(fn), tuple(float(t) for t in times), tuple(shape))
        fut, k = self._fut, self._key
        self._fut = self._key = None
        if fut is not None:
            try:
                val = fut.result()
            except Exception:
                val = None
            if k == key and val is not None:
                return val
        return stage_fn_values(fn, times, shape)

    def schedule(self, fn, times, shape):
        from concurrent.futures import ThreadPoolExecutor

        self.join()
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="irk-bc")
        times = [float(t) for t in times]
        self._key = (id(fn), tuple(times), tuple(shape))
        self._fut = self._pool.submit(stage_fn_values, fn, times, tuple(shape))


def _boundary_state(u_n, dofs):
    if la.is_torch(u_n):
        if u_n.device.type == "cuda":
            import torch

            out = la.dev_empty(len(dofs))
            idx = la.to_dev(dofs, dtype=torch.int64)
            call("irk_bc_gather", ctx(), len(dofs), ptr(idx), ptr(u_n), ptr(out))
            return la.to_host(out)
        return u_n.numpy()[dofs]
    return np.asarray(u_n, dtype=np.float64)[dofs]


def stage_bc_values(method: BcMethod, tab, bc: DirichletBC, u_n, t: float, dt: float,
                    unknown: StageUnknown = StageUnknown.DERIVATIVE,
                    fn_values: np.ndarray | None = None) -> np.ndarray:
    """Boundary values of the stage unknowns, shape (s, |Gamma|) (bcs.py:58-96).
    ``fn_values``: bc.g (DAE) / bc.g_dot (ODE) at the stage times, already
    evaluated (BoundaryPrefetch)."""
    shape = (len(bc.dofs),)
    stage_t = [t + ci * dt for ci in tab.c]
    if method is BcMethod.DAE:
        G = fn_values if fn_values is not None else stage_fn_values(bc.g, stage_t, shape)
        if unknown is StageUnknown.VALUE:
            return G  # independent of u_n: no device read-back
        if la.is_torch(u_n) and u_n.device.type == "cuda":
            # from the device state without a host round trip: (s, |Gamma|)
            # device array, consumed by stage_values_dev
            if unknown is not StageUnknown.W and not tab.invertible:
                raise ValueError(
                    "DAE boundary conditions on stage derivatives need an invertible "
                    f"tableau, got {tab.name!r}")
            out = la.dev_empty(G.size)
            ainv = (None if unknown is StageUnknown.W
                    else np.ascontiguousarray(_tableau_inverse(tab), dtype=np.float64))
            call("irk_bc_dae_values", ctx(), tab.s, shape[0], ptr(bc.dofs_dev()),
                 ptr(la.to_dev(np.ascontiguousarray(G).reshape(-1))), ptr(u_n), float(dt),
                 hptr(ainv) if ainv is not None else None, ptr(out))
            return out.reshape(tab.s, -1)
        ub = _boundary_state(u_n, bc.dofs)
        W = (G - ub[None, :]) / dt
        if unknown is StageUnknown.W:
            return W
        if not tab.invertible:
            raise ValueError(
                "DAE boundary conditions on stage derivatives need an invertible "
                f"tableau, got {tab.name!r}")
        # A^-1 W with the s x s inverse formed once per tableau (a many-rhs
        # LAPACK solve over |Gamma| columns costs ~1 ms per step at config 3)
        return _tableau_inverse(tab) @ W
    if bc.g_dot is None:
        raise ValueError("ODE boundary conditions require g_dot")
    Gd = fn_values if fn_values is not None else stage_fn_values(bc.g_dot, stage_t, shape)
    if unknown is StageUnknown.DERIVATIVE:
        return Gd
    W = tab.A @ Gd
    if unknown is StageUnknown.W:
        return W
    return _boundary_state(u_n, bc.dofs)[None, :] + dt * W


class ConstrainedStageOperator:
    """Row replacement + column elimination of a stage operator (bcs.py:99-120),
    applied by the masked variant of the fused stage kernel."""

    def __init__(self, op, dofs):
        self.op = op
        self.dofs = np.asarray(dofs, dtype=np.int64)
        if len(self.dofs) and self.dofs.max() >= op.m:
            raise ValueError("constrained dof index out of range")
        self.n = op.n
        self.s, self.m = op.s, op.m
        self._idx = (np.arange(op.s)[:, None] * op.m + self.dofs[None, :]).ravel()
        self._mask = None

    def mask(self):
        if self._mask is None:
            self._mask = la.dof_mask(self.m, self.dofs)
        return self._mask

    def dev_apply(self, Y, Out):
        return self.op.dev_apply(Y, Out, self.mask())

    def _dev_op(self):
        return self.op._dev_op(self.mask())

    def apply(self, v):
        vd = la.to_dev(v)
        if tuple(vd.shape) != (self.n,):
            raise ValueError(f"operator expects length {self.n}, got {tuple(vd.shape)}")
        out = la.stage_major_apply(self._dev_op(), vd, self.m, self.s)
        return la._like_input(out, v)


def stage_values_dev(svals):
    """The (s, |Gamma|) stage values as one flat device array (upload once,
    scatter several times)."""
    if la.is_torch(svals) and svals.device.type == "cuda":
        return svals.reshape(-1)
    return la.to_dev(np.ascontiguousarray(svals, dtype=np.float64).reshape(-1))


def scatter_stage_values(X_il, dofs_dev, svals, s: int):
    """X[dof*s + i] = svals[i, k] on an interleaved device block (svals:
    numpy, or the device array of stage_values_dev)."""
    sv = stage_values_dev(svals)
    call("irk_bc_scatter", ctx(), s, int(dofs_dev.numel()), ptr(dofs_dev), ptr(sv), ptr(X_il))


def constrain_stage_system_dev(op, rhs_il, bc: DirichletBC, svals):
    """Device form of constrain_stage_system on interleaved data:
    srhs = rhs - op(g_ext); srhs[Gamma] = g_ext[Gamma] (bcs.py:137-142)."""
    s, m = op.s, op.m
    dofs = bc.dofs_dev()
    svals = stage_values_dev(svals)
    g_ext = la.dev_zeros(m * s)
    scatter_stage_values(g_ext, dofs, svals, s)
    lifted = la.dev_empty(m * s)
    op.dev_apply(g_ext, lifted)
    srhs = rhs_il.clone()
    call("irk_axpby", ctx(), m * s, -1.0, ptr(lifted), 1.0, ptr(srhs))
    scatter_stage_values(srhs, dofs, svals, s)
    return ConstrainedStageOperator(op, bc.dofs), srhs


def constrain_stage_system(op, rhs, bc: DirichletBC, stage_values):
    """Impose stage boundary values on the coupled system (bcs.py:123-142).

    Public form on the reference's stage-major vectors."""
    if len(bc.dofs) == 0:
        return op, rhs
    s, m = op.s, op.m
    rd = la.to_dev(rhs)
    ril = la.dev_empty(m * s)
    call("irk_to_interleaved", ctx(), m, s, ptr(rd), ptr(ril))
    sop, srhs_il = constrain_stage_system_dev(op, ril, bc, np.asarray(stage_values))
    out = la.dev_empty(m * s)
    call("irk_to_stage_major", ctx(), m, s, ptr(srhs_il), ptr(out))
    return sop, la._like_input(out, rhs)
