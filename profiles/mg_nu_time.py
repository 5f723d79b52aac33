"""Structured MG-PCG solve time vs smoothing degree on the config-2 stage
blocks (rtol 1e-6, random rhs): `python profiles/mg_nu_time.py`."""
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

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    b = la.to_dev(np.random.default_rng(1).standard_normal(prob.m))
    x = la.dev_empty(prob.m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(len(pc.block_factors)):
        f0 = pc.block_factors[i]
        for nu in (2, 3, 4):
            s = la.BlockSolveSettings(rtol=1e-6, mg_nu=nu)
            f = la.BlockFactorization(prob.mass, prob.stiffness, f0.alpha, f0.beta, f0.dofs, s)
            for _ in range(3):
                its = f.dev_solve(b, x, settings=s)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                f.dev_solve(b, x, settings=s)
            e1.record()
            torch.cuda.synchronize()
            print(f"block {i} levels {f._mg.levels} structured {f._mg.structured}: nu {nu}: "
                  f"{its} its, {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/solve", flush=True)


if __name__ == "__main__":
    main()
