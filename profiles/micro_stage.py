"""Micro-benchmark of the fused stage-operator apply (K2) at config-2 size
(masked = the constrained operator FGMRES applies), CUDA events, inputs
larger than L2.  Prints us/apply and algorithmic GB/s vs the measured peak.

  python profiles/micro_stage.py [config]
"""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.bcs import ConstrainedStageOperator
    from paper_2403_08084_b200.stepper import _SPLIT

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    op = st._stage_operator(prob, _SPLIT[st.formulation])
    for masked in (True, False):
        dev = (ConstrainedStageOperator(op, prob.dirichlet.dofs)._dev_op()
               if masked and prob.dirichlet is not None else op._dev_op())
        s, m, nnz = op.s, op.m, prob.mass.nnz
        Y = la.to_dev(np.random.default_rng(0).standard_normal(s * m))
        Out = la.dev_empty(s * m)
        for _ in range(5):
            dev.dev_apply(Y, Out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        reps = 50
        e0.record()
        for _ in range(reps):
            dev.dev_apply(Y, Out)
        e1.record()
        torch.cuda.synchronize()
        t_eager = e0.elapsed_time(e1) / 1e3 / reps
        # device time: the applies replayed from one captured CUDA graph (the
        # eager loop can be bound by the host's ~35 us per Python call)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                dev.dev_apply(Y, Out)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        print(f"   (eager loop {t_eager * 1e6:.2f} us per apply)")
        algo = nnz * 20 + (m + 1) * 4 + 2 * s * m * 8
        peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
        print(f"config {k} stage apply masked={masked}: {t * 1e6:.2f} us, "
              f"{algo / t / 1e9:.0f} GB/s algorithmic = {algo / t / 1e9 / peak:.3f} of peak")


if __name__ == "__main__":
    main()
