#!/usr/bin/env python
"""Benchmark: RadauIIA-3 heat at ~1M DOFs (BASELINE.json config 2) — time
steps/s on the B200, the fused stage-operator apply and the dominant inner
kernel against the HBM roofline, and the CPU port of the reference path timed
on the same host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One JSON line on rank 0.  For N > 1 (torchrun, one process per GPU) every
rank runs an independent replica of the workload (the path does not shard,
DESIGN.md "Multi-GPU"); value = all ranks' steps / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RadauIIA-3 heat 1M-DOF time steps/s; stage-operator apply HBM GB/s vs peak"
UNIT = "steps/s"
L2_BYTES = 126 * 2**20


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region, in-process through NVML (the fields of the profiling recipe's
    nvidia-smi line).  NVML is initialised before the warm-up; the timed loop
    calls sample() between time steps (a few per run, ~5 ms each, on the
    main thread).  Concurrent sampling from another thread or a looping
    nvidia-smi was measured to stall this workload's frequent stream syncs by
    100-400 ms per step (driver-lock contention), so it is not used."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []  # (time, sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.window = None

    def __enter__(self):
        if os.environ.get("IRK_BENCH_NOCLOCKS"):
            return self
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:  # no NVML: no samples (reported as such)
            self._h = None
        return self

    def sample(self):
        if getattr(self, "_h", None) is None:
            return
        nv, h = self._nv, self._h
        try:
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            self.samples.append((time.perf_counter(), sm, rs))
        except Exception:
            pass

    def mark(self, t0, t1):
        """Bracket the timed region; summary() keeps the samples inside it
        (the nearest one when the region is shorter than the period)."""
        self.window = (t0, t1)

    def __exit__(self, *exc):
        pass

    def summary(self):
        smp = self.samples
        if self.window is not None and smp:
            t0, t1 = self.window
            inside = [x for x in smp if t0 <= x[0] <= t1]
            smp = inside or [min(smp, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))]
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted({n for _, _, rs in smp for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median([x[1] for x in smp])), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(smp), "source": "nvml"}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(t_local: float, steps: int, world: int):
    """Whole-job steps/s of `world` independent replicas: every rank ran
    `steps` steps; the job takes the slowest rank's time (max over ranks)."""
    t_max = max_over_ranks(t_local, world)
    return t_max, world * steps / t_max


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ----------------------------------------------------------------- ours


def stage_apply_roofline(wl, reps=40):
    """Fused stage-operator apply (K2) at the workload size, masked (the
    constrained operator every FGMRES iteration applies), CUDA events on the
    launching stream; inputs (201 MB at config 2) exceed the 126 MB L2."""
    import torch

    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.bcs import ConstrainedStageOperator
    from paper_2403_08084_b200.stepper import _SPLIT

    st, prob = wl.stepper, wl.problem
    if st.formulation.name == "DIRK":
        # the DIRK stage operator M + dt a_ii K (one stage; a_ii shared)
        from paper_2403_08084_b200.sparsela import KroneckerStageOperator

        aii = float(st.tableau.A[0, 0])
        op = KroneckerStageOperator(np.eye(1), np.array([[aii]]), prob.mass, [prob.stiffness],
                                    st.dt)
    else:
        op = st._stage_operator(prob, _SPLIT[st.formulation])
    dev_op = (ConstrainedStageOperator(op, prob.dirichlet.dofs)._dev_op()
              if prob.dirichlet is not None else op._dev_op())
    s, m = op.s, op.m
    nnz = prob.mass.nnz
    Y = la.to_dev(np.random.default_rng(0).standard_normal(s * m))
    Out = la.dev_empty(s * m)
    for _ in range(3):
        dev_op.dev_apply(Y, Out)
    torch.cuda.synchronize()
    # the reps applies replayed from one captured CUDA graph: device time per
    # launch (an eager Python loop costs ~35 us of host time per call, about
    # the kernel's own duration), CUDA events on the replaying stream
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            dev_op.dev_apply(Y, Out)
    g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    if st.formulation.name == "DIRK":
        # the single-stage apply of the combined B = M + dt a_ii K
        algo = nnz * 12 + (m + 1) * 4 + 2 * m * 8
    else:
        algo = nnz * 20 + (m + 1) * 4 + 2 * s * m * 8
    return t, algo, dict(s=s, m=m, nnz=nnz)


def inner_solve_profile(wl, peak, reps=20):
    """The step's dominant cost: one inner block solve of the first
    preconditioner block (the DIRK stage block for config 4) to the
    workload's inner tolerance, timed with CUDA events over `reps` solves of
    a seeded right-hand side.  Newton workloads (config 5) solve batched
    surrogate blocks inside the Newton loop instead: None there.

    Algorithmic bytes per CG iteration:
      Jacobi-PCG:      nnz*12 + (m+1)*4 + 96*m   (SpMV with CSR values and
                       columns, the update's vectors)
      multigrid-PCG on the structured 2D path (matrix-free levels, stencil
      SpMV on slot-uniform values): 80*m for the CG vectors (SpMV reads z,
      p_old, writes p_new, q: 32 B; update reads p, q, x, r, writes x, r:
      48 B) + per V-cycle level 62*m_l (pre 16, restriction 20, post 26) and
      16*m_L on the single-CTA coarsest level.
      sine-transform-preconditioned CG (2D real): the 80*m of the CG vectors
      + 3 transform kernels reading and writing the grid once (48*m).
      sine-transform-preconditioned COCG (3D complex pair blocks, config 3):
      160*m for the complex CG vectors + 5 line-transform kernels reading
      and writing the complex grid once (160*m)."""
    import torch

    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    st, prob = wl.stepper, wl.problem
    if not prob.is_linear:
        return None
    if st.formulation.name == "DIRK":
        fac = st._dirk_factor(st.tableau.A[0, 0], prob)
        sett = fac.settings
    else:
        pc = st._preconditioner(_SPLIT[st.formulation], prob)
        if pc is None:
            return None
        if pc.kind.name == "SCHUR":
            return pair_solve_profile(pc, prob, peak, reps)
        fac = pc.block_factors[0]
        sett = pc.settings
    if fac.direct:
        return None
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    sett = la.BlockSolveSettings(**{**sett.__dict__, "raise_on_maxit": False})
    fac.dev_solve(b, x, settings=sett)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    its = sum(fac.dev_solve(b, x, settings=sett) for _ in range(reps))
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    per_it = t / max(its / reps, 1)
    mg = getattr(fac, "_mg", None)
    nnz = prob.mass.nnz
    if mg is not None and mg.dst:
        b_it = 80 * m + 48 * m
        kind = "sine-transform-preconditioned CG (2D DST-I of the symmetrised stencil)"
    elif mg is not None and mg.structured:
        dim, N = prob.mass._p1_grid
        ms = [((N >> l) + 1) ** dim for l in range(mg.levels)]
        b_it = 80 * m + sum(62 * v for v in ms[:-1]) + 16 * ms[-1]
        kind = "multigrid-PCG (structured 2D V-cycle)"
    elif mg is not None:
        b_it = None
        kind = "multigrid-PCG (generic V-cycle)"
    else:
        b_it = nnz * 12 + (m + 1) * 4 + 96 * m
        kind = "Jacobi-PCG"
    out = dict(m=m, iterations_per_solve=its / reps, rtol=sett.rtol, method=kind,
               mg_levels=mg.levels if mg is not None else 0, us_per_solve=t * 1e6,
               us_per_iteration=per_it * 1e6)
    if b_it is not None:
        out["roofline"] = {
            "bound": "hbm", "algorithmic_bytes_per_iteration": int(b_it),
            "achieved": b_it / per_it / 1e9, "peak": peak, "unit": "GB/s",
            "frac": b_it / per_it / 1e9 / peak,
            "note": "per CG iteration incl. one preconditioner application; the working set (<= 8 vectors of "
                    f"{m * 8 / 1e6:.1f} MB) is largely L2-resident, so HBM is an upper "
                    "bound on the traffic, not the binding limit"}
    return out


def pair_solve_profile(pc, prob, peak, reps=20):
    """Config 3: one COCG solve of the first Gauss-Legendre Schur-pair block
    (complex alpha M + beta K) to the preconditioner's inner tolerance, timed
    like inner_solve_profile (irk_mgc_cocg through the C ABI)."""
    import torch

    from paper_2403_08084_b200 import _lib
    from paper_2403_08084_b200 import sparsela as la

    plan = pc._schur_plan()
    if not plan["np"]:
        return None
    Md, Kd = [d.eliminated(pc.mask()) for d in pc._device_mats()]
    mgc = pc._schur_mg(plan, Md, Kd)
    if mgc is None:
        return None
    h = mgc[0]
    m = prob.m
    sett = pc.settings
    b = la.to_dev(np.random.default_rng(1).standard_normal(2 * m))
    x = la.dev_empty(2 * m)
    its = np.zeros(1, dtype=np.int32)
    rel = np.zeros(1)
    lib = _lib.load()

    def solve():
        st = lib.irk_mgc_cocg(_lib.ctx(), h.handle, _lib.ptr(b), 2, _lib.ptr(x), 2,
                              float(sett.rtol), float(sett.atol), int(sett.maxit),
                              _lib.hptr(its), _lib.hptr(rel))
        if st not in (0, _lib.IRK_ENOCONV):
            raise RuntimeError(_lib.last_error())
        return int(its[0])

    solve()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    n_it = sum(solve() for _ in range(reps))
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    per_it = t / max(n_it / reps, 1)
    if h.dst:
        kind = "sine-transform-preconditioned COCG (3D complex DST-I of the symmetrised stencil)"
        b_it = 160 * m + 160 * m
    else:
        kind = ("multigrid-COCG (structured 3D complex V-cycle)" if h.structured else
                "multigrid-COCG (generic complex V-cycle)")
        b_it = None
    out = dict(m=m, iterations_per_solve=n_it / reps, rtol=sett.rtol, method=kind,
               mg_levels=h.levels, us_per_solve=t * 1e6, us_per_iteration=per_it * 1e6)
    if b_it is not None:
        out["roofline"] = {
            "bound": "hbm", "algorithmic_bytes_per_iteration": int(b_it),
            "achieved": b_it / per_it / 1e9, "peak": peak, "unit": "GB/s",
            "frac": b_it / per_it / 1e9 / peak,
            "note": "per COCG iteration incl. one preconditioner application; the working "
                    f"set (complex vectors of {m * 16 / 1e6:.1f} MB) is largely L2-resident, "
                    "so HBM is an upper bound on the traffic, not the binding limit"}
    return out


def traffic_from_profiles():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except json.JSONDecodeError:
            return {}
    return {}


def workload_config(k):
    """The `config` object of both arms (identical, so the driver's
    same-config check holds): the BASELINE.json workload and its sizes."""
    from paper_2403_08084_b200.configs import DESCRIPTIONS, GRID, STEPS

    dim, N = GRID[k]
    m = (N + 1) ** dim
    edges = (2 * N * (N + 1) + N * N) if dim == 2 else (3 * N * (N + 1) ** 2 + 3 * N * N * (N + 1)
                                                         + N ** 3)
    op_bytes = (m + 2 * edges) * 20 + 3 * 8 * m * 4
    return {"workload": f"config {k}: {DESCRIPTIONS[k]}", "m": m, "nnz": m + 2 * edges,
            "trajectory_steps": STEPS[k],
            "timed": "steps 1..K of the trajectory from u0 (warm-up steps run first, then "
                     "the state is reset to u0)",
            "l2": ("inputs larger than L2 (operators + stage vectors "
                   f"~{op_bytes / 1e6:.0f} MB > 126 MB)") if op_bytes > L2_BYTES else
                  "working set smaller than L2: a 256 MB buffer is written between timed "
                  "steps (inside the timed region)"}


class L2Flush:
    def __init__(self, k):
        import torch

        cfg = workload_config(k)
        self.buf = None
        if not cfg["l2"].startswith("inputs larger"):
            self.buf = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")

    def __call__(self):
        if self.buf is not None:
            self.buf.fill_(1.0)


def time_trajectory(st, prob, steps, warmup, k, clk=None, sample_at=()):
    """W warm-up steps, reset to u0, then `steps` device-timed steps
    (CUDA events on the launching stream).  Returns (seconds, reports,
    launches)."""
    import torch

    from paper_2403_08084_b200 import _lib

    snap = (st.u.copy(), st.step_index, st._t_base)
    for _ in range(warmup):
        st.step_device(prob)
    torch.cuda.synchronize()
    st.u, st.step_index, st._t_base = snap[0].copy(), snap[1], snap[2]
    flush = L2Flush(k)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    w0 = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/
    e0.record(stream)
    for i in range(steps):
        flush()
        _, rep = st.step_device(prob)
        reps.append(rep)
        if clk is not None and i in sample_at:
            clk.sample()
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    if clk is not None:
        clk.mark(w0, time.perf_counter())
    return e0.elapsed_time(e1) / 1e3, reps, _lib.launch_count() - launches0, snap


def step_stats(reps):
    krylov = [r.krylov_iters for r in reps]
    inner = [sum((sum(v) if isinstance(v, list) else (v or 0)) for v in r.inner_iters)
             for r in reps]
    return {"krylov_iters_per_step": float(np.mean(krylov)) if krylov else None,
            "inner_iters_per_step": float(np.mean(inner)) if inner else None,
            "newton_iters_per_step": float(np.mean([r.newton_iters for r in reps])) if reps else None}


# ------------------------------------------------------- CPU port (oracle)


def spawn_cpu_jobs(ks, budget, avoid_cpu):
    """CPU baselines as subprocesses, one core each (pinned, in parallel when
    the affinity mask has a core per job), started after the GPU arm's
    measurements."""
    import subprocess

    try:
        cpus = sorted(os.sched_getaffinity(0))
    except AttributeError:
        cpus = list(range(os.cpu_count() or 1))
    free = [c for c in cpus if c != avoid_cpu]
    jobs = {}
    parallel = len(free) >= len(ks) + 1
    for i, k in enumerate(ks):
        cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-job", str(k),
               "--cpu-budget", str(budget)]
        if parallel:
            cmd = ["taskset", "-c", str(free[i % len(free)])] + cmd
        env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1",
                   MKL_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
        jobs[k] = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                   text=True, env=env) if parallel else cmd
    return jobs, parallel


def collect_cpu_jobs(jobs, parallel, timeout=900):
    import subprocess

    out = {}
    for k, j in jobs.items():
        try:
            if parallel:
                so, se = j.communicate(timeout=timeout)
            else:
                env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1",
                           CUDA_VISIBLE_DEVICES="")
                r = subprocess.run(j, capture_output=True, text=True, timeout=timeout, env=env)
                so, se = r.stdout, r.stderr
            line = [x for x in so.splitlines() if x.startswith("{")]
            out[k] = json.loads(line[-1]) if line else {"error": se[-400:]}
        except Exception as exc:  # a baseline must never sink the GPU line
            if parallel:
                j.kill()
            out[k] = {"error": f"{type(exc).__name__}: {exc}"[:400]}
    return out


def _cpu_env():
    sys.path.insert(0, str(ROOT / "oracle"))
    import irk_oracle as orc

    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count()
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return orc, {"cpu_model": model, "affinity_cores": cores}


_BLOCK = {1: "lu", 2: "lu", 3: "pcg", 4: "pcg", 5: "pcg"}
_BLOCK_TXT = {"lu": "exact SuperLU blocks (scipy splu: the reference's factorize_block, "
                    "sparsela.py:171-191)",
              "pcg": "Jacobi-PCG/COCG inner blocks (SuperLU infeasible at this size: 3D "
                     "fill-in, or per-Newton factorisations)"}


def cpu_port(k):
    """The CPU port of the reference path (oracle/irk_oracle.py Stepper:
    MGS FGMRES, the reference's preconditioners) with its setup done and
    timed separately, as cli.run_precond_bench does (cli.py:224-242)."""
    orc, env = _cpu_env()
    cfg = orc.config(k, None, block=_BLOCK[k])
    st = orc.Stepper(cfg["problem"], cfg["tab"], cfg["dt"], **cfg["settings"])
    t0 = time.perf_counter()
    st.setup()
    return orc, st, cfg, time.perf_counter() - t0, env


def cpu_job(k, budget):
    """Real steps of the CPU port from step 1 of config k on one core until
    `budget` seconds (at least one step).  Config 4 (DIRK on 4.2M DOFs: one
    exact factorisation ~10 min, or 3 x ~1500 Jacobi-PCG iterations per step)
    times one real stage solve and counts a step as its three stage solves."""
    orc, st, cfg, t_setup, env = cpu_port(k)
    if k == 4:
        p, tab, dt = cfg["problem"], cfg["tab"], cfg["dt"]
        A = np.asarray(tab.A)
        blk = st._dirk_blocks[A[0, 0]]
        rhs = -(p.K @ p.u0)
        rhs[p.dofs] = 0.0
        t0 = time.perf_counter()
        _, its = orc.jacobi_pcg(blk.C, rhs, 1e-12)
        t = time.perf_counter() - t0
        return {"value": 1.0 / (3 * t), "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"config 4: the first stage solve of step 1 (n = {len(rhs)}, Jacobi-PCG "
                          f"to rtol 1e-12: {its} iterations, {t:.1f} s) on 1 core; a step = its 3 "
                          f"stage solves (same operator and tolerance); setup {t_setup:.1f} s "
                          "excluded", **env}
    t0 = time.perf_counter()
    n = 0
    while n < cfg["steps"]:
        st.step()
        n += 1
        if time.perf_counter() - t0 >= budget:
            break
    t = time.perf_counter() - t0
    its = [r[1] for r in st.reports]
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"config {k}: real steps 1..{n} of the trajectory ({t:.1f} s; FGMRES its "
                      f"{its}) on 1 core, {_BLOCK_TXT[_BLOCK[k]]}, MGS FGMRES as the reference; "
                      f"setup {t_setup:.1f} s excluded (cli.run_precond_bench)", **env}


def run_reference(args, world, rank):
    """--impl reference: the CPU implementation of the path (the oracle
    port; the reference itself is Python and cannot travel to the box) on
    the host, rank 0 only: setup, W real warm-up steps, reset to u0, then K
    real timed steps -- steps 1..K of the trajectory, as the GPU arm."""
    if rank != 0:
        return
    k = args.config
    orc, st, cfg, t_setup, env = cpu_port(k)
    if k == 4:
        r = cpu_job(4, 0)
        value, sec, sample = r["value"], 1.0 / r["value"], r["sample"]
    else:
        for _ in range(args.warmup):
            st.step()
        st.reset()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            st.step()
            times.append(time.perf_counter() - t0)
        sec = float(np.mean(times))
        value = 1.0 / sec
        sample = (f"config {k}: real steps 1..{args.steps} of the trajectory after {args.warmup} "
                  f"warm-up steps and a reset to u0, {_BLOCK_TXT[_BLOCK[k]]}, MGS FGMRES as "
                  f"the reference (FGMRES its {[r[1] for r in st.reports]}); setup "
                  f"{t_setup:.1f} s excluded (cli.run_precond_bench); 1 core (the block "
                  "solves and the Gauss-Seidel sweep are sequential)")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded u0 per BASELINE.json config; assembled P1 operators)",
           "impl": "reference", "config": workload_config(k),
           "parallelism": "cpu, 1 core (rank 0)",
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                            "sample": sample, **env},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ----------------------------------------------------------------- ours


def run_ours(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_08084_b200 import _lib, configs

    _lib.load()
    k = args.config
    solo = rank == 0 and world == 1
    # experiments only: IRK_BENCH_BLOCK='{"mg_nu": 3}' overrides block-solver settings
    wl = configs.build(k, **json.loads(os.environ.get("IRK_BENCH_BLOCK", "{}")))
    st, prob = wl.stepper, wl.problem
    clk = ClockSampler(local).__enter__()
    clk.sample()  # the first NVML query costs ~2 ms: keep it out of the timed region
    barrier(world)
    sample_at = {args.steps // 3, (2 * args.steps) // 3, args.steps - 1}
    t_dev, reps, launches, snap = time_trajectory(st, prob, args.steps, args.warmup, k, clk,
                                                  sample_at)
    t_max, value = replica_throughput(t_dev, args.steps, world)

    # end to end through the public API with host buffers: every step sets
    # the state from a pinned host array (H2D), steps, and reads u_next back
    # (D2H into the pinned numpy array step() returns, the next input); the
    # same steps 1..K from u0
    flush = L2Flush(k)
    # the end-to-end path has its own first-use costs (pinned staging blocks
    # of the host allocator: a fresh cudaHostAlloc of 8-34 MB costs
    # milliseconds): W untimed steps through the same calls, then the reset
    u_host = torch.from_numpy(snap[0].copy()).pin_memory().numpy()
    for _ in range(args.warmup):
        st.u = u_host
        u_host, _ = st.step(prob)
    st.u, st.step_index, st._t_base = snap[0].copy(), snap[1], snap[2]
    u_host = torch.from_numpy(snap[0].copy()).pin_memory().numpy()
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        flush()
        st.u = u_host
        u_host, _ = st.step(prob)
    torch.cuda.synchronize()
    _, e2e_value = replica_throughput(time.perf_counter() - w0, args.steps, world)
    e2e = {"value": e2e_value, "unit": UNIT,
           "h2d_bytes_per_step": prob.m * 8, "d2h_bytes_per_step": prob.m * 8}

    peak, peak_kind = peaks()
    t_sa, b_sa, meta_sa = stage_apply_roofline(wl)
    inner_prof = inner_solve_profile(wl, peak)
    traffic = traffic_from_profiles()
    stats = step_stats(reps)
    roof = {"bound": "hbm", "achieved": b_sa / t_sa / 1e9, "peak": peak, "unit": "GB/s",
            "frac": b_sa / t_sa / 1e9 / peak,
            "traffic": traffic.get("k_stage_apply" if k == 2 else f"k_stage_apply_config{k}"),
            "us_per_launch": t_sa * 1e6, "algorithmic_bytes": b_sa, **meta_sa,
            "kernel": "K2 masked stage-operator apply (k_stage_apply_bulk: cp.async.bulk tiles on an "
                      "mbarrier ring; 2D stencils with staged value slabs, the 3D stencil with the "
                      "values straight to registers)",
            "timing": "40 applies replayed from one captured CUDA graph, CUDA events"}
    inner_solver = None
    if inner_prof is not None:
        solves = [len(r.inner_iters) for r in reps]
        per_it = inner_prof["us_per_iteration"] * 1e-6
        inner_solver = dict(inner_prof, solves_per_step=float(np.mean(solves)) if solves else None)
        if stats["inner_iters_per_step"]:
            inner_solver["step_share_est"] = min(
                1.0, stats["inner_iters_per_step"] * per_it * args.steps / t_dev)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded u0 per BASELINE.json config; assembled P1 operators)",
        "config": workload_config(k), "parallelism": f"replicas{world}",
        "e2e": e2e, "gpu_launches": launches,
        "roofline": roof, "inner_solver": inner_solver, "peak_source": peak_kind,
        **stats, "clocks": clk.summary(),
    }
    if solo and not args.no_workloads:
        out["workloads"] = other_workloads(k, args)
    if solo and not args.no_cpu_baseline:
        # the CPU baselines run after every GPU measurement (run alongside,
        # their memory traffic slowed the host side of the e2e steps ~10 %)
        ks = [k] + ([j for j in (1, 2, 3, 4, 5) if j != k] if not args.no_workloads else [])
        try:
            me = os.sched_getaffinity(0)
            me = min(me) if len(me) == 1 else -1
        except AttributeError:
            me = -1
        res = collect_cpu_jobs(*spawn_cpu_jobs(ks, args.cpu_budget, me))
        out["cpu_baseline"] = res.get(k)
        for j, r in res.items():
            if j != k and "workloads" in out and str(j) in out["workloads"]:
                out["workloads"][str(j)]["cpu_baseline"] = r
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def other_workloads(k0, args):
    """Every other BASELINE.json workload on this GPU: its whole trajectory
    (config steps) after 3 warm-up steps and a reset to u0, device-timed;
    config 2 also as written (inner blocks by Jacobi-PCG to 1e-6)."""
    import gc

    from paper_2403_08084_b200 import configs

    peak, _ = peaks()
    res = {}
    plan = [(j, {}) for j in (1, 2, 3, 4, 5) if j != k0]
    plan.append((2, {"method": "pcg"}))
    for j, block in plan:
        wl = configs.build(j, **block)
        t, reps, launches, _ = time_trajectory(wl.stepper, wl.problem, wl.steps, 3, j)
        key = str(j) if not block else f"{j}-spec-literal"
        r = {"workload": wl.description, "value": wl.steps / t, "unit": UNIT,
             "steps": wl.steps, "ms_per_step": 1e3 * t / wl.steps, "gpu_launches": launches,
             "config": workload_config(j), **step_stats(reps)}
        if block:
            r["workload"] = (f"config {j} as written: inner diagonal blocks by Jacobi-PCG to "
                             "rtol 1e-6 (BlockSolveSettings(method='pcg'))")
        else:
            t_sa, b_sa, meta = stage_apply_roofline(wl)
            r["roofline"] = {"bound": "hbm", "achieved": b_sa / t_sa / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": b_sa / t_sa / 1e9 / peak,
                             "us_per_launch": t_sa * 1e6, "algorithmic_bytes": b_sa, **meta}
            ip = inner_solve_profile(wl, peak)
            if ip is not None:
                r["inner_solver"] = ip
        res[key] = r
        del wl
        gc.collect()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-workloads", action="store_true",
                    help="headline workload only (no per-config lines, no extra CPU jobs)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--cpu-job", type=int, default=0, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_job:
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        print(json.dumps(cpu_job(args.cpu_job, args.cpu_budget)))
        return
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
