"""Cost of one deferred multigrid-PCG block solve (config 2 block 0) as a
function of the iteration count: rtol = 0 and maxit = k force exactly k
iterations; T(k) = a + b k from CUDA events over back-to-back solves (no
host synchronisation between them, as inside a time step).
`python profiles/r02/solve_cost_probe.py`."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2403_08084_b200 import _lib, configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    wl = configs.build(2)
    st, prob = wl.stepper, wl.problem
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    fac = pc.block_factors[0]
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    reps = 30
    res = []
    for k in (1, 2, 3, 4, 5, 6, 8, 10, 12):
        sett = la.BlockSolveSettings(**{**fac.settings.__dict__, "rtol": 0.0, "maxit": k,
                                        "raise_on_maxit": False})
        with _lib.deferred_solves() as log:
            for _ in range(3):
                fac.dev_solve(b, x, settings=sett, defer=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fac.dev_solve(b, x, settings=sett, defer=True)
            e1.record()
            torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / reps
        res.append((k, t))
        print(f"maxit {k:3d}: {t:8.1f} us per solve", flush=True)
    ks = np.array([r[0] for r in res], float)
    ts = np.array([r[1] for r in res])
    b_, a_ = np.polyfit(ks, ts, 1)
    print(f"fit: T(k) = {a_:.1f} + {b_:.1f} k us")


if __name__ == "__main__":
    main()
