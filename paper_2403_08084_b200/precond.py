"""Stage preconditioners on the device (drop-in for implicitrk.precond,
/root/reference/pkg/src/implicitrk/precond.py).

Every kind replaces A by a surrogate A~ and inverts the surrogate stage
system block by block (precond.py:43-57, :92-117):

* block diagonal ("jacobi"): all s blocks independent -> ONE batched
  Jacobi-PCG over the interleaved m-by-s block (one pass over M, K per
  iteration advances every stage);
* block lower/upper and the Rana LD/DU kinds: sequential blocks; the
  Gauss-Seidel coupling R_i - sum_j c_ij C x_j is one fused kernel, each
  block a Jacobi-PCG on the pre-combined block matrix;
* SCHUR (new; the reference declines it): A = Q T Q^T (real
  Schur), A~ = Q blockdiag(T) Q^T.  After the (Q^T (x) I) transform every
  1x1 block is a real SPD system (batched PCG) and every 2x2 block
  [[a, b], [c, a]] is the real form of one complex-symmetric system
  (D + i w X) z = r1 + i d r2, solved by batched Jacobi-COCG.

Inner block solves follow ``BlockSolveSettings`` (Jacobi-PCG, rtol 1e-6 by
default, as north_star's config 2 specifies); FGMRES being flexible, an
inexact block solve only changes the outer iteration count.
"""

from __future__ import annotations

from enum import Enum

import ctypes as C
import numpy as np

from . import _lib
from . import sparsela as la
from ._lib import call, ctx, hptr, ptr
from .sparsela import BlockFactorization, BlockSolveSettings, FactorizationError, SparseMatrix, Splitting
from .tableaux import ButcherTableau, additive_split, ldu_factor, real_schur


class PreconditionerKind(Enum):
    BLOCK_DIAGONAL = "jacobi"
    BLOCK_LOWER = "gs-lower"
    BLOCK_UPPER = "gs-upper"
    RANA_LD = "rana-ld"
    RANA_DU = "rana-du"
    SCHUR = "schur"


_LOWER_KINDS = (PreconditionerKind.BLOCK_LOWER, PreconditionerKind.RANA_LD)
_UPPER_KINDS = (PreconditionerKind.BLOCK_UPPER, PreconditionerKind.RANA_DU)


def _surrogate(kind: PreconditionerKind, tab: ButcherTableau) -> np.ndarray:
    """A~ for each kind (precond.py:43-57; SCHUR: Q blockdiag(T) Q^T)."""
    A = np.array(tab.A, dtype=np.float64)
    if kind is PreconditionerKind.BLOCK_DIAGONAL:
        return np.diag(np.diag(A))
    if kind is PreconditionerKind.BLOCK_LOWER:
        sp_ = additive_split(tab)
        return sp_.L_strict + np.diag(sp_.D_diag)
    if kind is PreconditionerKind.BLOCK_UPPER:
        sp_ = additive_split(tab)
        return np.diag(sp_.D_diag) + sp_.U_strict
    if kind is PreconditionerKind.SCHUR:
        sd = real_schur(A)
        Tb = np.zeros_like(A)
        for st, sz in sd.blocks:
            Tb[st:st + sz, st:st + sz] = sd.T[st:st + sz, st:st + sz]
        return sd.Q @ Tb @ sd.Q.T
    fac = ldu_factor(tab)
    if kind is PreconditionerKind.RANA_LD:
        return fac.L * fac.D[None, :]
    if kind is PreconditionerKind.RANA_DU:
        return fac.D[:, None] * fac.U
    raise ValueError(f"unknown preconditioner kind {kind!r}")


class _LazyBlocks:
    """block_factors[i] built on first access (the batched paths never need
    the pre-combined block matrices)."""

    def __init__(self, builders):
        self._builders = builders
        self._made = [None] * len(builders)

    def __len__(self):
        return len(self._builders)

    def __getitem__(self, i):
        if self._made[i] is None:
            self._made[i] = self._builders[i]()
        return self._made[i]

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class StagePreconditioner:
    """Application of the surrogate stage system's inverse (precond.py:60-117).

    Attributes mirror the reference (kind, A_tilde, A_tilde_inv,
    block_factors, form, M, Ks, dt, dofs, s, m, n).  ``apply`` takes the
    reference's stage-major vectors; ``dev_apply`` works on interleaved
    device blocks."""

    def __init__(self, kind, A_tilde, A_tilde_inv, block_factors, form, M, Ks, dt, dofs,
                 settings: BlockSolveSettings | None = None, tab=None, shift=None):
        self.kind = kind
        self.A_tilde = A_tilde
        self.A_tilde_inv = A_tilde_inv
        self.block_factors = block_factors
        self.form = form
        self.M = M
        self.Ks = Ks
        self.dt = dt
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self.s = A_tilde.shape[0]
        self.m = M.nrows
        self.n = self.s * self.m
        self.settings = settings or BlockSolveSettings()
        self._coef = A_tilde_inv if form is Splitting.IA else dt * A_tilde
        self._tab = tab
        self._shift = shift  # optional m-by-s diagonal shifts (semilinear surrogate)
        self._mask = None
        self._mats = None
        self._schur = None
        self.inner_iterations = []
        self.defer_solves = False  # set by the stepper around deferred_solves
        self._serial = next(la._SERIAL)
        self._last_apply = []  # inner_iterations entries of the latest apply

    # ------------------------------------------------------------ helpers
    def mask(self):
        if self._mask is None and len(self.dofs):
            self._mask = la.dof_mask(self.m, self.dofs)
        return self._mask

    def _device_mats(self):
        if self._mats is None:
            self._mats = la.shared_pattern([self.M.device()] + [K.device() for K in self.Ks])
        return self._mats

    def _sweep_plan(self):
        """(block order, per-block coupling coefficients or None) of the
        sequential sweep, built once."""
        plan = getattr(self, "_sweep", None)
        if plan is None:
            s, kind = self.s, self.kind
            if kind is PreconditionerKind.BLOCK_DIAGONAL:
                order, deps = list(range(s)), (lambda i: ())
            elif kind in _LOWER_KINDS:
                order, deps = list(range(s)), (lambda i: range(i))
            else:
                order, deps = list(range(s - 1, -1, -1)), (lambda i: range(i + 1, s))
            coefs = []
            for i in range(s):
                coef = np.zeros(s)
                for j in deps(i):
                    coef[j] = self._coef[i, j]
                coefs.append(np.ascontiguousarray(coef) if np.any(coef != 0.0) else None)
            plan = self._sweep = (order, coefs)
        return plan

    def _mg_blocks(self) -> bool:
        """Blocks are solved one by one through their factors when the user
        asked for a per-block method ("direct", "chebyshev"), when every
        block is direct (small blocks, any pattern), or when each has a
        multigrid hierarchy or a direct inverse (P1 grid operators, no
        diagonal shift: ~5 instead of O(100) batched Jacobi iterations)."""
        meth = self.settings.method
        if self._shift is not None:
            return False
        if meth in ("direct", "chebyshev"):
            return True
        if meth not in ("auto", "mg", "dst"):
            return False
        facs = list(self.block_factors)
        if all(f.direct for f in facs):
            return True
        if getattr(self.M, "_p1_grid", None) is None:
            return False
        if getattr(self.Ks[0], "_p1_grid", None) != self.M._p1_grid:
            return False
        return all(f._mg is not None or f.direct for f in facs)

    def _concurrent_blocks(self, coefs) -> bool:
        """Independent multigrid block solves that may overlap: no coupling
        terms, deferred status, every block on its hierarchy."""
        if not self.defer_solves or self.settings.raise_on_maxit or self.s < 2:
            return False
        if any(c is not None for c in coefs) or self.settings.method not in ("auto", "mg", "dst"):
            return False
        return all(f._mg is not None and not f.direct for f in self.block_factors)

    def _block_coefs(self):
        s = self.s
        if self.form is Splitting.IA:
            return [float(self.A_tilde_inv[i, i]) for i in range(s)], [self.dt] * s
        return [1.0] * s, [self.dt * float(self.A_tilde[i, i]) for i in range(s)]

    def _pcg(self, nb, alpha, beta, A, Bm, shift, rhs, ld_rhs, x, ld_x):
        st = self.settings
        its = np.zeros(8, dtype=np.int32)
        rel = np.zeros(8)
        al = np.ascontiguousarray(alpha + [0.0] * (8 - nb), dtype=np.float64)
        be = np.ascontiguousarray(beta + [0.0] * (8 - nb), dtype=np.float64)
        status = _lib.load().irk_pcg(
            ctx(), nb, hptr(al), hptr(be), A.handle, Bm.handle if Bm is not None else C.c_void_p(),
            ptr(shift), ptr(self.mask()), ptr(rhs), int(ld_rhs), ptr(x), int(ld_x),
            float(st.rtol), float(st.atol), int(st.maxit), hptr(its), hptr(rel))
        self._inner_status(status, its[:nb])
        return its[:nb]

    def _inner_status(self, status, its):
        self.inner_iterations.append([int(v) for v in its])
        if status in (_lib.IRK_OK,):
            return
        if status == _lib.IRK_ENOCONV and not self.settings.raise_on_maxit:
            return
        if status == _lib.IRK_ESINGULAR and not self.settings.raise_on_maxit:
            return
        _lib.check(status, "stage preconditioner block solve")

    # ------------------------------------------------------------- apply
    def dev_apply(self, R, X):
        """X = P^-1 R on interleaved device blocks (R, X distinct)."""
        kind = self.kind
        s, m = self.s, self.m
        if kind is PreconditionerKind.SCHUR:
            return self._apply_schur(R, X)
        mk = self.mask()
        mats = [d.eliminated(mk) for d in self._device_mats()]
        Md, Ks = mats[0], mats[1:]
        if kind is PreconditionerKind.BLOCK_DIAGONAL and len(Ks) == 1 and not self._mg_blocks():
            # independent blocks without a multigrid hierarchy: one batched
            # Jacobi-PCG advances all s systems per pass
            a, b = self._block_coefs()
            self._pcg(s, a, b, Md, Ks[0], self._shift, R, s, X, s)
            return X
        # sequential Gauss-Seidel sweep (precond.py:97-117); every block
        # solve writes its whole stage column of X before a later block reads
        # it, so X needs no zeroing
        order, coefs = self._sweep_plan()
        n0 = len(self.inner_iterations)
        if self._concurrent_blocks(coefs) and not la._torch().cuda.is_current_stream_capturing():
            # block Jacobi on multigrid blocks, deferred: the s independent
            # solves read their stage columns of R in place and run
            # concurrently (one auxiliary stream per block after the first)
            st = self.settings
            hs = (C.c_void_p * s)(*[f._mg.handle.value for f in self.block_factors])
            status = _lib.load().irk_mg_pcg_multi(
                ctx(), s, hs, ptr(R), s, 1, ptr(X), s, 1, float(st.rtol), float(st.atol),
                int(st.maxit), None, None)
            _lib.check(status, "deferred block solves")
            self.inner_iterations.extend([[None]] * s)
            self._last_apply = self.inner_iterations[n0:]
            return X
        tmp = la.dev_empty(m)
        for i in order:
            coef = coefs[i]
            if coef is not None:
                C_ = Md if self.form is Splitting.IA else (Ks[0] if len(Ks) == 1 else Ks[i])
                call("irk_stage_couple", ctx(), s, i, hptr(coef), C_.handle,
                     ptr(self.mask()), ptr(R), ptr(X), ptr(tmp), 1)
            fac = self.block_factors[i]
            xi = X[i:]
            # a block without coupling terms reads its stage column of R in
            # place (stride s): no staging copy
            rhs_i, ld_i = (tmp, 1) if coef is not None else (R[i:], s)
            # deferred (no host round trip) when the caller collects the log
            st = fac.dev_solve(rhs_i, xi, ld_rhs=ld_i, ld_x=s, settings=self.settings,
                               defer=self.defer_solves)
            self.inner_iterations.append([st])
        self._last_apply = self.inner_iterations[n0:]
        return X

    def _graph_key(self):
        """Identity of a capturable application (graph-replayed inside the
        device FGMRES cycles): the sequential sweep over blocks solved by a
        fixed kernel sequence (direct inverses, fixed-sweep Chebyshev, a fixed
        number of sine-transform-preconditioned CG iterations)."""
        if self.kind is PreconditionerKind.SCHUR or self._shift is not None:
            return None
        if not self._mg_blocks():
            return None
        if not all(f.graph_safe(self.settings) for f in self.block_factors):
            return None
        return ("pc", self._serial)
    def _schur_plan(self):
        if self._schur is not None:
            return self._schur
        s = self.s
        sd = real_schur(self._tab.A)
        pairs = [(st, sz) for st, sz in sd.blocks if sz == 2]
        reals = [(st, sz) for st, sz in sd.blocks if sz == 1]
        order = [c for st, _ in pairs for c in (st, st + 1)] + [st for st, _ in reals]
        Qp = sd.Q[:, order]
        sl = np.ones(s)
        sr = np.ones(s)
        ca_re, ca_im, cb_re, cb_im = [], [], [], []
        for k, (st, _) in enumerate(pairs):
            Tb = sd.T[st:st + 2, st:st + 2]
            if self.form is Splitting.IA:
                P_, Q_ = np.linalg.inv(Tb), self.dt * np.eye(2)
                a, b, c = P_[0, 0], P_[0, 1], P_[1, 0]
                w = np.sqrt(-b * c)
                ca_re.append(a), ca_im.append(w), cb_re.append(self.dt), cb_im.append(0.0)
            else:
                a, b, c = self.dt * Tb[0, 0], self.dt * Tb[0, 1], self.dt * Tb[1, 0]
                w = np.sqrt(-b * c)
                ca_re.append(1.0), ca_im.append(0.0), cb_re.append(a), cb_im.append(w)
            sl[2 * k + 1] = w / c     # scale of equation 2
            sr[2 * k + 1] = -w / b    # x2 = (-w/b) y2
        real_a, real_b = [], []
        for st, _ in reals:
            t = sd.T[st, st]
            if self.form is Splitting.IA:
                real_a.append(1.0 / t), real_b.append(self.dt)
            else:
                real_a.append(1.0), real_b.append(self.dt * t)
        s_pad = s + (s % 2)
        L = np.zeros((s_pad, s))
        L[:s] = sl[:, None] * Qp.T
        Rb = np.zeros((s, s_pad))
        Rb[:, :s] = Qp * sr[None, :]
        self._schur = dict(np=len(pairs), nr=len(reals), s_pad=s_pad,
                           L=np.ascontiguousarray(L), R=np.ascontiguousarray(Rb),
                           ca=(ca_re, ca_im), cb=(cb_re, cb_im), ra=real_a, rb=real_b)
        return self._schur

    def _schur_mg(self, plan, Md, Kd):
        """Complex multigrid hierarchies of the pair blocks (None when the
        blocks are not P1 grid operators with a full-boundary mask)."""
        if "mgc" not in plan:
            hs = []
            for k in range(plan["np"]):
                a = complex(plan["ca"][0][k], plan["ca"][1][k])
                b = complex(plan["cb"][0][k], plan["cb"][1][k])
                h = la._MgcHierarchy.build(self.M, self.Ks[0], Md, Kd, a, b, self.mask(),
                                           self.settings)
                if h is None:
                    hs = None
                    break
                hs.append(h)
            plan["mgc"] = hs
        return plan["mgc"]

    def _apply_schur(self, R, X):
        plan = self._schur_plan()
        mats = [d.eliminated(self.mask()) for d in self._device_mats()]
        if len(mats) != 2:
            raise ValueError("the Schur preconditioner needs one shared stiffness matrix")
        Md, Kd = mats
        s, m, sp_ = self.s, self.m, plan["s_pad"]
        W = la.dev_empty(m * sp_)
        Z = la.dev_zeros(m * sp_)
        call("irk_stage_mix", ctx(), m, sp_, s, hptr(plan["L"]), ptr(R), ptr(W))
        st = self.settings
        npairs, nr = plan["np"], plan["nr"]
        mgc = self._schur_mg(plan, Md, Kd) if npairs else None
        if mgc is not None:
            # one multigrid-preconditioned COCG per pair block (complex V-cycle)
            defer = self.defer_solves and not st.raise_on_maxit
            if defer:
                # the pair solves are independent: concurrent on auxiliary
                # streams, status to the deferred log
                hs = (C.c_void_p * npairs)(*[h.handle.value for h in mgc])
                status = _lib.load().irk_mgc_cocg_multi(
                    ctx(), npairs, hs, ptr(W), sp_, 2, ptr(Z), sp_, 2, float(st.rtol),
                    float(st.atol), int(st.maxit), None, None)
                _lib.check(status, "deferred pair solves")
                self.inner_iterations.extend([[None]] * npairs)
            for k in range(0 if defer else npairs):
                its = np.zeros(1, dtype=np.int32)
                rel = np.zeros(1)
                status = _lib.load().irk_mgc_cocg(
                    ctx(), mgc[k].handle, ptr(W[2 * k:]), sp_, ptr(Z[2 * k:]), sp_,
                    float(st.rtol), float(st.atol), int(st.maxit),
                    None if defer else hptr(its), None if defer else hptr(rel))
                if defer:
                    _lib.check(status, "deferred pair solve")
                    self.inner_iterations.append([None])
                else:
                    self._inner_status(status, its[:1])
        elif npairs:
            its = np.zeros(8, dtype=np.int32)
            rel = np.zeros(8)
            arrs = [np.ascontiguousarray(v + [0.0] * (8 - npairs), dtype=np.float64)
                    for v in (*plan["ca"], *plan["cb"])]
            status = _lib.load().irk_cocg(
                ctx(), npairs, hptr(arrs[0]), hptr(arrs[1]), hptr(arrs[2]), hptr(arrs[3]),
                Md.handle, Kd.handle, ptr(self.mask()), ptr(W), sp_, ptr(Z), sp_,
                float(st.rtol), float(st.atol), int(st.maxit), hptr(its), hptr(rel))
            self._inner_status(status, its[:npairs])
        if nr:
            off = 2 * npairs
            self._pcg(nr, plan["ra"], plan["rb"], Md, Kd, None, W[off:], sp_, Z[off:], sp_)
        call("irk_stage_mix", ctx(), m, s, sp_, hptr(plan["R"]), ptr(Z), ptr(X))
        return X

    def _dev_op(self):
        pc = self

        class _Op(la._DevOp):
            n = pc.n
            layout = (pc.m, pc.s) if pc.s > 1 else None

            def dev_apply(self, x, out):
                pc.dev_apply(x, out)

            def graph_key(self):
                return pc._graph_key()

            def account(self, applications):
                pc.inner_iterations.extend(list(pc._last_apply) * applications)

            def discard(self, applications):
                k = len(pc._last_apply) * applications
                if k:
                    del pc.inner_iterations[-k:]

            def fixed_solves(self):
                return all(f._fixed_iterations(pc.settings) is not None
                           for f in pc.block_factors)

        return _Op()

    def apply(self, r):
        rd = la.to_dev(r)
        if tuple(rd.shape) != (self.n,):
            raise ValueError(f"preconditioner expects length {self.n}, got {tuple(rd.shape)}")
        out = la.stage_major_apply(self._dev_op(), rd, self.m, self.s)
        return la._like_input(out, r)


def build_preconditioner(kind: PreconditionerKind, tab: ButcherTableau, M: SparseMatrix, K, dt: float,
                         form: Splitting = Splitting.IA, dirichlet=None,
                         settings: BlockSolveSettings | None = None, shift=None) -> StagePreconditioner:
    """Build a stage preconditioner (precond.py:120-157).

    ``K`` is one stiffness matrix or a per-stage list (Newton Jacobians);
    ``dirichlet`` lists constrained dofs (identity rows/columns in every
    block); ``settings`` selects the inner block solver; ``shift`` (m-by-s
    interleaved device block) adds diag(shift[:, i]) to block i (the lumped
    reaction surrogate of semilinear Jacobians)."""
    Ks = list(K) if isinstance(K, (list, tuple)) else [K]
    dofs = np.asarray(dirichlet if dirichlet is not None else [], dtype=np.int64)
    A_tilde = _surrogate(kind, tab)
    try:
        A_tilde_inv = np.linalg.inv(A_tilde)
    except np.linalg.LinAlgError as exc:
        raise FactorizationError(f"{kind.value} surrogate of {tab.name!r} is singular") from exc
    if form is Splitting.IA and not tab.invertible:
        raise FactorizationError(
            f"IA-form preconditioning needs an invertible tableau, got {tab.name!r}")
    if kind is PreconditionerKind.SCHUR and len(Ks) != 1:
        raise ValueError("the Schur preconditioner needs one shared stiffness matrix")
    st = settings or BlockSolveSettings()
    if kind is PreconditionerKind.SCHUR and st.method in ("direct", "chebyshev"):
        # the pair blocks are complex symmetric: COCG (multigrid or Jacobi)
        raise ValueError(f"block method {st.method!r} is not available for the Schur "
                         "preconditioner's complex pair blocks (use 'auto', 'mg' or 'pcg')")
    if shift is not None and st.method in ("direct", "chebyshev", "mg", "dst"):
        raise ValueError(f"block method {st.method!r} cannot include the diagonal shift of "
                         "the semilinear surrogate blocks (use 'auto' or 'pcg')")

    def builder(i):
        Ki = Ks[0] if len(Ks) == 1 else Ks[i]
        if form is Splitting.IA:
            return lambda: BlockFactorization(M, Ki, A_tilde_inv[i, i], dt, dofs, st)
        return lambda: BlockFactorization(M, Ki, 1.0, dt * A_tilde[i, i], dofs, st)

    blocks = _LazyBlocks([builder(i) for i in range(tab.s)])
    pc = StagePreconditioner(kind, A_tilde, A_tilde_inv, blocks, form, M, Ks, dt, dofs, st,
                             tab=tab, shift=shift)
    if kind not in (PreconditionerKind.BLOCK_DIAGONAL, PreconditionerKind.SCHUR) or len(Ks) > 1:
        for b in blocks:  # regularity checks up front, as the reference's factorisations do
            pass
    return pc


def apply_preconditioner(pc: StagePreconditioner, r):
    return pc.apply(r)
