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

# FGMRES iterations per time step of the CPU port (Jacobi-PCG 1e-6 inner
# blocks) at full size, used to scale the bounded CPU sample to steps/s.
# Config 2 values measured with oracle/irk_oracle.py (block="pcg"); see
# profiles/cpu_port_iterations.json.
CPU_ITS_PER_STEP = {1: 15.7, 2: 11.0, 3: 4.0, 4: 3.0, 5: 20.0}


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
    op = st._stage_operator(prob, _SPLIT[st.formulation])
    dev_op = (ConstrainedStageOperator(op, prob.dirichlet.dofs)._dev_op()
              if prob.dirichlet is not None else op._dev_op())
    s, m = op.s, op.m
    nnz = prob.mass.nnz
    Y = la.to_dev(np.random.default_rng(0).standard_normal(s * m))
    Out = la.dev_empty(s * m)
    for _ in range(3):
        dev_op.dev_apply(Y, Out)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        dev_op.dev_apply(Y, Out)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    algo = nnz * 20 + (m + 1) * 4 + 2 * s * m * 8
    return t, algo, dict(s=s, m=m, nnz=nnz)


def pcg_iteration_roofline(wl, iters=200):
    """One Jacobi-PCG iteration (SpMV+direction kernel and update kernel) on
    the first preconditioner block M + dt*a_11*K (pre-combined, Dirichlet
    rows identity), timed over a fixed iteration count."""
    import torch

    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    st, prob = wl.stepper, wl.problem
    if st.formulation.name == "DIRK":
        fac = st._dirk_factor(st.tableau.A[0, 0], prob)
    else:
        pc = st._preconditioner(_SPLIT[st.formulation], prob)
        if pc is None or pc.kind.name == "SCHUR":
            return None
        fac = pc.block_factors[0]
    m, nnz = prob.m, prob.mass.nnz
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    fixed = la.BlockSolveSettings(rtol=0.0, atol=0.0, maxit=iters, raise_on_maxit=False)
    fac.dev_solve(b, x, settings=fixed)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    its = fac.dev_solve(b, x, settings=fixed)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / max(its, 1)
    # algorithmic bytes per iteration: B values + columns (12 B/nnz) + row
    # offsets, SpMV kernel vectors z, p_old in / p_new, q out (32 B/row),
    # update kernel p, q, dinv, x, r in / x, r, z out (64 B/row)
    algo = nnz * 12 + (m + 1) * 4 + 96 * m
    return t, algo, dict(m=m, nnz=nnz, iterations=its)


def traffic_from_profiles():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except json.JSONDecodeError:
            return {}
    return {}


def run_ours(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2403_08084_b200 import _lib, configs

    _lib.load()
    wl = configs.build(args.config)
    st, prob = wl.stepper, wl.problem
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        st.step_device(prob)
    torch.cuda.synchronize()
    barrier(world)
    # the e2e arm below replays exactly these timed steps (same states, same
    # solver work): snapshot the stepper state
    snap = (st.u_device.clone(), st.step_index, st._t_base)
    reps = []
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    if os.environ.get("IRK_BENCH_NOGC"):
        import gc

        gc.disable()
    if True:
        torch.cuda.synchronize()
        w_t0 = time.perf_counter()
        e0.record(stream)
        marks = []
        sample_at = {args.steps // 3, (2 * args.steps) // 3, args.steps - 1}
        for i in range(args.steps):
            _, rep = st.step_device(prob)
            reps.append(rep)
            if i in sample_at:
                ts0 = time.perf_counter()
                clk.sample()
                if os.environ.get("IRK_BENCH_TRACE"):
                    print(f"sample after step {i}: {1e3 * (time.perf_counter() - ts0):.2f} ms",
                          file=sys.stderr)
            if os.environ.get("IRK_BENCH_TRACE"):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                marks.append((ev, time.perf_counter()))
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark(w_t0, time.perf_counter())
    clk.__exit__(None, None, None)
    launches = _lib.launch_count() - launches0
    if marks:
        prev_e, prev_w = e0, None
        for k, (ev, wt) in enumerate(marks):
            print(f"step {k}: {prev_e.elapsed_time(ev):.2f} ms device, krylov "
                  f"{reps[k].krylov_iters}", file=sys.stderr)
            prev_e = ev
    t_dev = e0.elapsed_time(e1) / 1e3
    t_max, value = replica_throughput(t_dev, args.steps, world)

    # end to end through the public API with host buffers: pinned H2D of the
    # state, the step, the D2H read of u_next (numpy result of step()).
    st.u, st.step_index, st._t_base = snap[0], snap[1], snap[2]
    u_pin = torch.from_numpy(st.u.copy()).pin_memory()
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        st.u = u_pin
        u_host, _ = st.step(prob)
        u_pin.copy_(torch.from_numpy(u_host))
    torch.cuda.synchronize()
    _, e2e_value = replica_throughput(time.perf_counter() - w0, args.steps, world)
    e2e = {"value": e2e_value, "unit": UNIT,
           "h2d_bytes_per_step": prob.m * 8, "d2h_bytes_per_step": prob.m * 8}

    peak, peak_kind = peaks()
    t_sa, b_sa, meta_sa = stage_apply_roofline(wl)
    pcg = pcg_iteration_roofline(wl)
    traffic = traffic_from_profiles()
    krylov = [r.krylov_iters for r in reps]
    inner = [sum(sum(v) if isinstance(v, list) else v for v in r.inner_iters) for r in reps]
    stage_apply = {"bound": "hbm", "achieved": b_sa / t_sa / 1e9, "peak": peak, "unit": "GB/s",
                   "frac": b_sa / t_sa / 1e9 / peak, "traffic": traffic.get("k_stage_apply"),
                   "us_per_launch": t_sa * 1e6, "algorithmic_bytes": b_sa, **meta_sa}
    # roofline: the fused stage-operator apply (K2), the kernel the metric
    # names; HBM-bound with inputs larger than L2
    roof = dict(stage_apply, kernel="k_stage_apply_win (K2, masked stage operator)")
    inner_solver = None
    if pcg is not None:
        # the step's dominant cost: the inner Jacobi-PCG iteration.  Its
        # working set (~5 vectors of m doubles + the header-compressed
        # operator) stays L2-resident for the whole solve, so algorithmic
        # bytes / time can exceed the HBM peak; DRAM traffic per iteration is
        # near zero (profiles/r01) and the bound is L2/latency, not HBM.
        t_pc, b_pc, meta_pc = pcg
        inner_solver = {
            "kernel": "Jacobi-PCG iteration (k_cg_spmv_st + k_cg_update)",
            "us_per_iteration": t_pc * 1e6, "algorithmic_bytes": b_pc,
            "algorithmic_GBs": b_pc / t_pc / 1e9, "hbm_peak": peak,
            "bound": "l2-resident (algorithmic bytes/time above the HBM peak)",
            "step_share_est": (sum(inner) * t_pc / t_dev) if inner else None,
            "traffic": traffic.get("pcg_iteration"), **meta_pc}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded u0 per BASELINE.json config; assembled P1 operators)",
        "config": {"workload": f"config {args.config}: {wl.description}", "m": prob.m,
                   "nnz": prob.mass.nnz, "replicas": world, "parallelism": f"replicas{world}",
                   "l2": "inputs larger than L2 (operators + vectors > 126 MB)"},
        "e2e": e2e, "gpu_launches": launches,
        "roofline": roof, "inner_solver": inner_solver,
        "peak_source": peak_kind,
        "krylov_iters_per_step": float(np.mean(krylov)) if krylov else None,
        "inner_iters_per_step": float(np.mean(inner)) if inner else None,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_sample(args.config, budget=args.cpu_budget)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ------------------------------------------------------- CPU port (oracle)


def cpu_sample(k, budget=20.0):
    """Time the CPU port of the reference path (oracle/irk_oracle.py, the
    same algorithm with Jacobi-PCG inner blocks) on the full workload: setup
    excluded as in cli.run_precond_bench (cli.py:224-242), then the first
    step's FGMRES iterations until `budget` seconds; steps/s =
    1 / (seconds per FGMRES iteration x FGMRES iterations per step)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, str(ROOT / "oracle"))
    import irk_oracle as orc

    cfg = orc.config(k, None, block="pcg")
    p, tab, dt = cfg["problem"], cfg["tab"], cfg["dt"]
    stg = orc.Stepper(p, tab, dt, **cfg["settings"])
    s, m = tab.s, p.M.shape[0]
    t_setup0 = time.perf_counter()
    if cfg["settings"]["pc"] is not None:
        pc = orc.StagePC(cfg["settings"]["pc"], tab, p.M, [p.K], dt,
                         "ia" if cfg["settings"]["form"] == "ia" else "ai", p.dofs, "pcg",
                         cfg["settings"]["inner_rtol"])
    else:
        pc = None
    t_setup = time.perf_counter() - t_setup0
    A = np.asarray(tab.A)
    if k == 4:
        blk = orc.Block(p.M, p.K, 1.0, dt * A[0, 0], p.dofs, "pcg", 1e-12)
        rhs = -(p.K @ p.u0)
        rhs[p.dofs] = 0.0
        t0 = time.perf_counter()
        _, its = orc.jacobi_pcg(blk.C, rhs, 1e-12, maxit=400)
        t = time.perf_counter() - t0
        per_stage = t / its * 1558.0  # survey-measured CG iterations per stage solve
        sec_step = 3 * per_stage
        return {"value": 1.0 / sec_step, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"config 4: {its} Jacobi-PCG iterations of stage 1 (n=4.2M) on 1 core, "
                          f"{t / its * 1e3:.1f} ms/it, scaled by 3 stages x 1558 its/stage"}
    C1, C2 = (np.eye(s), A)
    op = lambda v: orc.kron_apply(C1, C2, p.M, [p.K], dt, v)  # noqa: E731
    idx = orc.stage_index(s, m, p.dofs)
    sop = orc.constrained(op, idx) if len(p.dofs) else op
    v = np.random.default_rng(0).standard_normal(s * m)
    n_it, t0 = 0, time.perf_counter()
    while True:
        z = pc.apply(v) if pc is not None else v
        w = sop(z)
        v = w / np.linalg.norm(w)
        n_it += 1
        if time.perf_counter() - t0 > budget:
            break
    t_it = (time.perf_counter() - t0) / n_it
    its = CPU_ITS_PER_STEP.get(k, 12.0)
    return {"value": 1.0 / (t_it * its), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"config {k} (m={m}): {n_it} FGMRES iterations (preconditioner apply + "
                      f"constrained stage apply) on 1 core, {t_it:.2f} s/it, scaled by {its} "
                      f"its/step; PC setup {t_setup:.1f} s excluded"}


def run_reference(args, world, rank):
    """--impl reference: the CPU port of the reference path on the host
    cores (rank 0 only), each step a bounded sample (one FGMRES iteration of
    the full workload, scaled to a time step)."""
    if rank != 0:
        return
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    samples = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(args.config, budget=budget)
        if i >= args.warmup:
            samples.append(1.0 / r["value"])
    sec = float(np.mean(samples))
    value = 1.0 / sec
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": f"config {args.config}", "parallelism": "cpu-1-core"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                            "sample": r["sample"]},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
