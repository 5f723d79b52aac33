"""One persistent Jacobi-PCG solve (config-2 first block, fixed iterations)
for an ncu capture of k_pcg_persist."""

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

    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    wl = configs.build(2)
    st, prob = wl.stepper, wl.problem
    fac = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
    b = la.to_dev(np.random.default_rng(1).standard_normal(prob.m))
    x = la.dev_empty(prob.m)
    its = fac.dev_solve(b, x, settings=la.BlockSolveSettings(rtol=0.0, maxit=iters))
    torch.cuda.synchronize()
    print("ok its", its)


if __name__ == "__main__":
    main()
