"""Micro-benchmark of the inner Jacobi-PCG iteration on the first
preconditioner block of a config (fixed iteration count, CUDA events).

  python profiles/micro_pcg.py [config] [iters]
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    k = int(args[0]) if len(args) > 0 else 2
    iters = int(args[1]) if len(args) > 1 else 200
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    if st.formulation.name == "DIRK":
        fac = st._dirk_factor(st.tableau.A[0, 0], prob)
    else:
        fac = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    fixed = la.BlockSolveSettings(rtol=0.0, atol=0.0, maxit=iters, raise_on_maxit=False)
    fac.dev_solve(b, x, settings=fixed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0.record()
        its = fac.dev_solve(b, x, settings=fixed)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / max(its, 1))
    if "--prof" in sys.argv:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fac.dev_solve(b, x, settings=fixed)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=6,
                                        max_name_column_width=60))
    conv = la.BlockSolveSettings(rtol=1e-6)
    its_conv = fac.dev_solve(b, x, settings=conv)
    print(f"config {k} m={m}: {best:.2f} us/PCG iteration ({its} its fixed); "
          f"{its_conv} its to rtol 1e-6")


if __name__ == "__main__":
    main()
