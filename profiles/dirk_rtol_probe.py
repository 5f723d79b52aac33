"""Config-4 (DIRK) final-state error vs the reference golden and steps/s for
stage-solve tolerances: `python profiles/dirk_rtol_probe.py`."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main():
    import torch

    import irk_oracle as oracle
    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200.sparsela import BlockSolveSettings

    g = np.load(ROOT / "tests" / "golden" / "full_config4.npz")
    for rt in [float(v) for v in sys.argv[1:]] or (1e-15, 1e-13, 1e-12):
        wl = configs.build(4)
        st, prob = wl.stepper, wl.problem
        st.dirk_solver = BlockSolveSettings(rtol=rt, atol=st.krylov.atol,
                                            maxit=max(20000, 10 * prob.m), raise_on_maxit=True)
        key = f"traj4_n{configs.GRID[4][1]}"
        P = oracle.sketch_rows(prob.m)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        worst = 0.0
        torch.cuda.synchronize()
        e0.record()
        for i in range(wl.steps):
            st.step_device(prob)
        e1.record()
        torch.cuda.synchronize()
        i = wl.steps - 1
        proj = P @ st.u
        ref = g[f"{key}_u{i}_proj"]
        worst = np.linalg.norm(proj - ref) / np.linalg.norm(ref)
        print(f"rtol {rt:g}: final-state rel L2 {worst:.3e}, "
              f"{wl.steps * 1000 / e0.elapsed_time(e1):.1f} steps/s (incl. setup)", flush=True)


if __name__ == "__main__":
    main()
