"""Inner MG-PCG iterations to rtol 1e-6 on the three config-2 stage blocks
for smoothing degrees nu (generic V-cycle path when nu != 2):
`python profiles/mg_nu_probe.py`."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    wl = configs.build(2)
    st, prob = wl.stepper, wl.problem
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    b = la.to_dev(np.random.default_rng(1).standard_normal(prob.m))
    x = la.dev_empty(prob.m)
    for i in range(3):
        f0 = pc.block_factors[i]
        for nu in (1, 2, 3, 4):
            for cs in (4, 8):
                s = la.BlockSolveSettings(rtol=1e-6, mg_nu=nu, mg_coarse_steps=cs)
                f = la.BlockFactorization(prob.mass, prob.stiffness, f0.alpha, f0.beta, f0.dofs, s)
                its = f.dev_solve(b, x, settings=s)
                print(f"block {i} beta {f0.beta:.3e} levels {f._mg.levels}: nu {nu} coarse {cs}: {its} its",
                      flush=True)


if __name__ == "__main__":
    main()
