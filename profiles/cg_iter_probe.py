"""Per-iteration cost of the multigrid-PCG inner solve (config-2 block 0):
solve time vs iteration count over a sweep of tolerances (linear fit), and
the same for Jacobi-PCG (no V-cycle): `python profiles/cg_iter_probe.py`."""
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
    fac = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for method, rtols in (("auto", [1e-1, 1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12]),
                          ("pcg", [1e-1, 1e-2, 1e-3, 1e-4])):
        pts = []
        for rt in rtols:
            sett = la.BlockSolveSettings(method=method, rtol=rt, maxit=5000)
            for _ in range(2):
                its = fac.dev_solve(b, x, settings=sett)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                fac.dev_solve(b, x, settings=sett)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 10 * 1e3
            pts.append((its, t))
            print(f"{method} rtol {rt:g}: {its} its, {t:.1f} us", flush=True)
        a = np.array(pts, dtype=float)
        slope, icpt = np.polyfit(a[:, 0], a[:, 1], 1)
        print(f"{method}: {slope:.1f} us per iteration, {icpt:.1f} us fixed", flush=True)


if __name__ == "__main__":
    main()
