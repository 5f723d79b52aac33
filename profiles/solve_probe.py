"""Wall vs device time of consecutive inner block solves (config 2 block 0)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    fac = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(3 * m)
    conv = la.BlockSolveSettings(rtol=1e-6)
    for _ in range(3):
        fac.dev_solve(b, x, ld_x=3, settings=conv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    w0 = time.perf_counter()
    e0.record()
    its = 0
    for _ in range(n):
        its += fac.dev_solve(b, x, ld_x=3, settings=conv)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / n * 1e3
    print(f"config {k}: {wall:.3f} ms wall / {e0.elapsed_time(e1) / n:.3f} ms events per solve, "
          f"{its / n:.1f} its per solve")


if __name__ == "__main__":
    main()
