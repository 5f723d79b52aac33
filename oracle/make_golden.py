"""Generate tests/golden/*.npz from the UNMODIFIED reference (test infrastructure).

Runs in the build container only: it imports implicitrk from
/root/reference/pkg/src (read-only, never copied) and records its outputs on
seeded inputs.  The fixtures pin both the CPU oracle (oracle/irk_oracle.py)
and, on the GPU box, the CUDA path.

  python oracle/make_golden.py small          # seconds: unit + small trajectories
  python oracle/make_golden.py mms            # seconds: MMS loads / norms / CLI sweeps
  python oracle/make_golden.py full K [K...]  # full-size config sketches (minutes-hours)

Pieces the reference lacks are fed to it from the oracle (P1 matrices,
Gauss-Legendre tableau, Allen-Cahn callables); configs whose full size the
reference cannot run (3: SuperLU infeasible in 3D; 5: hours of per-Newton
SuperLU) are produced by the oracle's PCG-block restatement and labelled so.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import irk_oracle as orc  # noqa: E402


def ref():
    if not REF_SRC.exists():
        raise SystemExit("the reference is only available in the build container")
    sys.path.insert(0, str(REF_SRC))
    import implicitrk  # noqa: F401

    return implicitrk


def csr_arrays(prefix, A):
    return {f"{prefix}_rowptr": np.asarray(A.row_offsets, dtype=np.int64),
            f"{prefix}_col": np.asarray(A.col_indices, dtype=np.int64),
            f"{prefix}_val": np.asarray(A.values, dtype=np.float64)}


def ref_sparse(irk, A):
    return irk.SparseMatrix.from_scipy(A)


def ref_tab(irk, t: orc.Tab):
    return irk.ButcherTableau(t.A, t.b, t.c, 2 * t.s, t.s, t.name)


def random_spd_pair(rng, m, density=0.4):
    B = rng.standard_normal((m, m)) * (rng.random((m, m)) < density)
    S = B @ B.T + m * np.eye(m)
    C = rng.standard_normal((m, m)) * (rng.random((m, m)) < density)
    T = C @ C.T
    return S, T


# ------------------------------------------------------------------ small


def make_small():
    irk = ref()
    out = {}
    # tableaux (tableaux.py)
    tabs = {f"radau{s}": irk.radau_iia(s) for s in range(1, 6)}
    tabs.update(lobatto2=irk.lobatto_iiic(2), lobatto3=irk.lobatto_iiic(3),
                alexander=irk.alexander_dirk(), wsodirk=irk.wsodirk433())
    for k, t in tabs.items():
        out[f"tab_{k}_A"], out[f"tab_{k}_b"], out[f"tab_{k}_c"] = t.A, t.b, t.c
    # reference assembly: 1D P1 and 2D Q1 (problems.py:80-99)
    for dim, n in ((1, 5), (1, 9), (2, 4), (2, 7)):
        M, K, bd = irk.assemble_heat(irk.StructuredGrid(dim, n))
        out.update(csr_arrays(f"asm{dim}d{n}_M", M))
        out.update(csr_arrays(f"asm{dim}d{n}_K", K))
        out[f"asm{dim}d{n}_bd"] = bd
    # Kronecker stage operator (sparsela.py:222-235), shared and per-stage K
    rng = np.random.default_rng(11)
    for s, m in ((1, 5), (2, 8), (3, 6), (4, 5)):
        S, T = random_spd_pair(rng, m)
        A = rng.standard_normal((s, s))
        C1 = rng.standard_normal((s, s))
        Ms, Ks = irk.SparseMatrix.from_dense(S), irk.SparseMatrix.from_dense(T)
        Kl = [irk.SparseMatrix.from_dense(random_spd_pair(rng, m)[1]) for _ in range(s)]
        v = rng.standard_normal(s * m)
        dt = 0.37
        key = f"kron_s{s}m{m}"
        out[f"{key}_M"], out[f"{key}_K"], out[f"{key}_C1"], out[f"{key}_C2"] = S, T, C1, A
        out[f"{key}_Kl"] = np.stack([k.to_dense() for k in Kl])
        out[f"{key}_v"] = v
        out[f"{key}_y"] = irk.KroneckerStageOperator(C1, A, Ms, [Ks], dt).apply(v)
        out[f"{key}_yl"] = irk.KroneckerStageOperator(C1, A, Ms, Kl, dt).apply(v)
        dofs = np.array([0, m - 1])
        from implicitrk.bcs import ConstrainedStageOperator
        cop = ConstrainedStageOperator(irk.KroneckerStageOperator(C1, A, Ms, [Ks], dt), dofs)
        out[f"{key}_yc"] = cop.apply(v)
    # FGMRES (sparsela.py:299-403)
    for n, seed in ((6, 1), (12, 2), (30, 3)):
        r = np.random.default_rng(seed)
        A = r.standard_normal((n, n)) + (n / 2) * np.eye(n)
        b = r.standard_normal(n)
        res = irk.fgmres(A, b, settings=irk.KrylovSettings(rtol=1e-12, restart=5, maxit=200))
        out[f"fgmres{n}_A"], out[f"fgmres{n}_b"], out[f"fgmres{n}_x"] = A, b, res.x
        out[f"fgmres{n}_its"] = np.array(res.iterations)
        out[f"fgmres{n}_res"] = np.array(res.residuals)
    # preconditioners: every kind x form on 1D heat with Dirichlet (precond.py)
    grid = irk.StructuredGrid(1, 10)
    M, K, bd = irk.assemble_heat(grid)
    r = np.random.default_rng(5)
    for tname, tab in (("radau3", irk.radau_iia(3)), ("lobatto3", irk.lobatto_iiic(3))):
        v = r.standard_normal(tab.s * grid.npoints)
        out[f"pc_{tname}_v"] = v
        for kind in irk.PreconditionerKind:
            for form in irk.Splitting:
                try:
                    pc = irk.build_preconditioner(kind, tab, M, K, 0.05, form, bd)
                except Exception:
                    continue
                out[f"pc_{tname}_{kind.value}_{form.value}"] = pc.apply(v)
    # DAE stage boundary values (bcs.py:58-96)
    tab = irk.radau_iia(3)
    bc = irk.DirichletBC(dofs=np.array([0, 4]), g=lambda t: np.array([np.sin(t), 1.0 + t]))
    u = np.array([0.3, 0.0, 0.0, 0.0, -0.2])
    for unk in irk.StageUnknown:
        out[f"bc_{unk.value}"] = irk.stage_bc_values(irk.BcMethod.DAE, tab, bc, u, 0.2, 0.1, unk)
    # small trajectories of the config recipes through the reference steppers
    out.update(trajectory(irk, 1, None))
    out.update(trajectory(irk, 2, 32))
    out.update(trajectory(irk, 3, 6))
    out.update(trajectory(irk, 4, 32))
    out.update(trajectory(irk, 5, 32))
    GOLDEN.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(GOLDEN / "reference_small.npz", **out)
    print("wrote", GOLDEN / "reference_small.npz", len(out), "arrays")


_FORMS = {"ai": "STAGE_DERIVATIVE_AI", "ia": "STAGE_DERIVATIVE_IA", "value": "STAGE_VALUE",
          "dirk": "DIRK"}
_PCS = {"jacobi": "BLOCK_DIAGONAL", "gs-lower": "BLOCK_LOWER", "rana-ld": "RANA_LD"}


def ref_problem(irk, cfg):
    p = cfg["problem"]
    M, K = ref_sparse(irk, p.M), ref_sparse(irk, p.K)
    m = M.nrows
    if p.poly is not None:
        c = np.asarray(p.poly)
        dc = np.polynomial.polynomial.polyder(c)
        import scipy.sparse as sp

        def residual(t, u, udot):
            return (M.to_scipy() @ udot + p.kscale * (K.to_scipy() @ u)
                    + M.to_scipy() @ np.polynomial.polynomial.polyval(u, c))

        def jac(t, u):
            return irk.SparseMatrix.from_scipy(
                p.kscale * K.to_scipy() + M.to_scipy() @ sp.diags(np.polynomial.polynomial.polyval(u, dc)))

        return irk.SemidiscreteProblem(m=m, mass=M, residual=residual, jacobian_u=jac, u0=p.u0)
    bc = irk.DirichletBC(dofs=p.dofs, g=p.g) if len(p.dofs) else None
    return irk.SemidiscreteProblem(m=m, mass=M, stiffness=K, load=lambda t: np.zeros(m),
                                   dirichlet=bc, u0=p.u0)


class StageRecorder:
    """Records the stage vectors the reference computes but does not keep.

    DIRK (stepper.py:391-421): every linear stage is ``res = fgmres(...)``
    and ``ki = res.x`` is then overwritten at the Dirichlet dofs in place, so
    the recorded ``res.x`` objects ARE the final K_stages rows.  The wrapper
    replaces the module attribute ``implicitrk.stepper.fgmres`` (the
    reference's source is untouched).  Newton (stepper.py:519-541): the last
    s residual evaluations of a step are at the converged iterate; their
    ``udot`` arguments are the stage derivatives (the AI unknown)."""

    def __init__(self, irk):
        import implicitrk.stepper as rst

        self.rst, self.orig, self.xs = rst, rst.fgmres, []

        def rec(*a, **kw):
            res = self.orig(*a, **kw)
            self.xs.append(res.x)
            return res

        rst.fgmres = rec
        self.udots = []

    def take_dirk(self, s):
        out = np.array([np.asarray(x, dtype=float).copy() for x in self.xs[-s:]])
        self.xs.clear()
        return out

    def take_newton(self, s):
        out = np.array(self.udots[-s:])
        self.udots.clear()
        return out

    def close(self):
        self.rst.fgmres = self.orig


def trajectory(irk, k, n, steps=None, full=False):
    cfg = orc.config(k, n)
    prob = ref_problem(irk, cfg)
    rec = StageRecorder(irk) if k in (4, 5) else None
    if k == 5:
        res0 = prob.residual

        def residual(t, u, udot):
            rec.udots.append(np.array(udot, dtype=float))
            return res0(t, u, udot)

        prob.residual = residual
    tab = cfg["tab"]
    rt = irk.ButcherTableau(tab.A, tab.b, tab.c, 1, 1, tab.name)
    st = cfg["settings"]
    pc = st["pc"]
    if pc == "schur":
        pc = "rana-ld"  # the reference has no Schur PC; the trajectory does not depend on it
    kw = dict(formulation=getattr(irk.StageFormulation, _FORMS[st["form"]]),
              krylov=irk.KrylovSettings(rtol=st["rtol"]),
              pc_kind=getattr(irk.PreconditionerKind, _PCS[pc]) if pc else None)
    if k == 5:
        kw["newton"] = irk.NewtonSettings(rtol=1e-10, atol=1e-10)
    stp = irk.TimeStepper(prob, rt, cfg["dt"], **kw)
    key = f"traj{k}_n{cfg['n']}"
    out = {} if full else {f"{key}_u0": np.asarray(prob.u0)}
    us, stages, its = [], [], []
    t0 = time.time()
    nsteps = steps if steps is not None else cfg["steps"]
    P = None
    for i in range(nsteps):
        u, rep = stp.step(prob)
        its.append((rep.newton_iters, rep.krylov_iters))
        xs = None
        if k == 4:
            xs = rec.take_dirk(tab.s).ravel()  # K_stages, stage-major
        elif k == 5:
            xs = rec.take_newton(tab.s).ravel()
        elif stp._last_stages is not None:
            xs = stp._last_stages
        if full:
            if P is None:
                P = orc.sketch_rows(len(u))
                # per-stage projections for DIRK (s*m Gaussian rows would be 3 GB)
                Ps = orc.sketch_rows(len(u) if k == 4 else len(u) * tab.s, seed=77)
            sk = orc.sketch(u, P)
            for f in ("proj", "sample", "norm", "sum"):
                out[f"{key}_u{i}_{f}"] = np.asarray(sk[f])
            if xs is not None:
                if k == 4:
                    X = xs.reshape(tab.s, -1)
                    out[f"{key}_x{i}_proj"] = np.stack([Ps @ X[j] for j in range(tab.s)])
                    out[f"{key}_x{i}_norm"] = np.asarray(np.linalg.norm(xs))
                    out[f"{key}_x{i}_sample"] = xs[:: max(1, len(xs) // 4096)].copy()
                else:
                    sks = orc.sketch(xs, Ps)
                    out[f"{key}_x{i}_proj"] = sks["proj"]
                    out[f"{key}_x{i}_norm"] = np.asarray(sks["norm"])
            print(f"  config {k} step {i + 1}/{nsteps} its {its[-1]} {time.time() - t0:.1f}s",
                  flush=True)
        else:
            us.append(u.copy())
            if xs is not None:
                stages.append(np.array(xs, dtype=float))
    if rec is not None:
        rec.close()
    if not full:
        out[f"{key}_u"] = np.array(us)
        if stages:
            out[f"{key}_x"] = np.array(stages)
    out[f"{key}_its"] = np.array(its)
    out[f"{key}_wall"] = np.array(time.time() - t0)
    return out


def make_full(k):
    """Full-size sketches: reference code (exact LU) for configs 1, 2, 4;
    oracle PCG restatement for 3 and 5 (reference infeasible)."""
    GOLDEN.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    if k in (1, 2, 4):
        irk = ref()
        out = trajectory(irk, k, None, full=True)
        out["source"] = np.array("reference (implicitrk, exact SuperLU blocks)")
    else:
        cfg = orc.config(k, None, block="pcg")
        st = orc.Stepper(cfg["problem"], cfg["tab"], cfg["dt"], **cfg["settings"])
        key = f"traj{k}_n{cfg['n']}"
        out = {}
        P = Ps = None
        for i in range(cfg["steps"]):
            u = st.step()
            if P is None:
                P = orc.sketch_rows(len(u))
                Ps = orc.sketch_rows(len(u) * cfg["tab"].s, seed=77)
            sk = orc.sketch(u, P)
            for f in ("proj", "sample", "norm", "sum"):
                out[f"{key}_u{i}_{f}"] = np.asarray(sk[f])
            sks = orc.sketch(st.stages[-1], Ps)
            out[f"{key}_x{i}_proj"] = sks["proj"]
            out[f"{key}_x{i}_norm"] = np.asarray(sks["norm"])
            st.stages.clear()
            print(f"  config {k} step {i + 1}/{cfg['steps']} {st.reports[-1]} "
                  f"{time.time() - t0:.1f}s", flush=True)
        out[f"{key}_its"] = np.array([r[:2] for r in st.reports])
        out["source"] = np.array("oracle restatement (Jacobi-PCG/COCG inner blocks)")
    out["wall"] = np.array(time.time() - t0)
    np.savez_compressed(GOLDEN / f"full_config{k}.npz", **out)
    print("wrote", GOLDEN / f"full_config{k}.npz", f"{time.time() - t0:.1f}s")


def make_mms():
    """Manufactured-solution layer (SURVEY §8 f rows 2-3): the reference's
    load vectors, error norms, an MMS trajectory and its CLI sweeps."""
    irk = ref()
    import tempfile

    from implicitrk import cli as rcli

    out = {}
    t = 0.3
    for dim, n in ((1, 10), (2, 8)):
        grid = irk.StructuredGrid(dim, n)
        mms = irk.heat_mms_2d() if dim == 2 else irk.heat_mms_1d()
        out[f"load{dim}d"] = irk.assemble_load(grid, mms.f, t)
        uh = irk.interpolate(grid, mms.u, t)
        uh = uh + 0.01 * np.random.default_rng(5 + dim).standard_normal(uh.shape)
        out[f"uh{dim}d"] = uh
        out[f"l2_{dim}d"] = irk.l2_error(grid, uh, mms.u, t)
        out[f"h1_{dim}d"] = irk.h1_error(grid, uh, mms.u, mms.grad, t)
        out[f"norm_{dim}d"] = irk.fe_l2_norm(grid, uh)
    # MMS trajectory through the reference stepper (2D Q1, RadauIIA(2), rana-ld)
    grid = irk.StructuredGrid(2, 8)
    prob = irk.mms_heat_problem(grid)
    st = irk.TimeStepper(prob, irk.radau_iia(2), 0.1, krylov=irk.KrylovSettings(rtol=1e-12),
                         pc_kind=irk.PreconditionerKind.RANA_LD)
    u, _ = irk.advance(st, prob, 0.5)
    out["mms_u"] = u
    mms = irk.heat_mms_2d()
    out["mms_l2"] = irk.l2_error(grid, u, mms.u, 0.5)
    out["mms_h1"] = irk.h1_error(grid, u, mms.u, mms.grad, 0.5)
    # CLI: spatial convergence sweep and the DAE/ODE boundary contrast
    with tempfile.TemporaryDirectory() as td:
        rc = rcli.main(["converge", "--mode", "spatial", "--n-list", "4", "8", "--tfinal", "0.2",
                        "--rtol", "1e-12", "--out", f"{td}/conv.csv"])
        assert rc == 0
        out["cli_converge"] = np.loadtxt(f"{td}/conv.csv", delimiter=",", skiprows=1)
        rc = rcli.main(["converge", "--mode", "temporal", "--problem", "dahlquist",
                        "--dt-list", "0.2", "0.1", "--tfinal", "1.0", "--out", f"{td}/temp.csv"])
        assert rc == 0
        out["cli_temporal"] = np.genfromtxt(f"{td}/temp.csv", delimiter=",", skip_header=1)
        rc = rcli.main(["bc-compare", "--nx", "6", "--dt", "0.1", "--tfinal", "0.3",
                        "--rtol", "1e-12", "--out", f"{td}/bc"])
        assert rc == 0
        out["cli_dae"] = np.loadtxt(f"{td}/bc/daenorm.csv", delimiter=",", skiprows=1)
        out["cli_ode"] = np.loadtxt(f"{td}/bc/odenorm.csv", delimiter=",", skiprows=1)
    GOLDEN.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(GOLDEN / "reference_mms.npz", **out)
    print("wrote", GOLDEN / "reference_mms.npz")


if __name__ == "__main__":
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        make_small()
    elif what == "mms":
        make_mms()
    else:
        for k in map(int, sys.argv[2:]):
            make_full(k)
