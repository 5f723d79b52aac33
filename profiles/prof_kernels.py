"""Short driver for ncu captures of the hot kernels at config-2 size:
the fused stage-operator apply (masked), one Jacobi-PCG solve of 20
iterations on the first Gauss-Seidel block, and one CGS Arnoldi step.

  python profiles/prof_kernels.py            # plain run (must exit 0 first)
  ncu --set full -k regex:'k_stage_apply|k_cg_|k_multidot|k_orth' ... python profiles/prof_kernels.py
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import _lib, configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.bcs import ConstrainedStageOperator
    from paper_2403_08084_b200.stepper import _SPLIT

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    op = st._stage_operator(prob, _SPLIT[st.formulation])
    cop = ConstrainedStageOperator(op, prob.dirichlet.dofs)._dev_op()
    s, m = op.s, op.m
    Y = la.to_dev(np.random.default_rng(0).standard_normal(s * m))
    Out = la.dev_empty(s * m)
    for _ in range(3):
        cop.dev_apply(Y, Out)
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    fac = pc.block_factors[0]
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    its = fac.dev_solve(b, x, settings=la.BlockSolveSettings(rtol=0.0, maxit=20))
    n = s * m
    V = la.dev_empty(11 * n).view(11, n)
    V.normal_()
    h = la.dev_empty(128)
    _lib.call("irk_multidot", _lib.ctx(), n, 10, _lib.ptr(V), n, _lib.ptr(V[10]), _lib.ptr(h))
    _lib.call("irk_orth_update", _lib.ctx(), n, 10, _lib.ptr(V), n, _lib.ptr(h), _lib.ptr(V[10]), 0)
    torch.cuda.synchronize()
    print(f"ok: stage applies 3, pcg its {its}, launches {_lib.launch_count()}")


if __name__ == "__main__":
    main()
