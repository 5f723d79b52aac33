"""Config-4 (DIRK) steps/s vs the multigrid smoothing degree of the stage
solve (rtol 1e-15): `python profiles/dirk_nu_probe.py`."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200.sparsela import BlockSolveSettings

    for nu in (2, 3, 4):
        wl = configs.build(4)
        st = wl.stepper
        st.dirk_solver = BlockSolveSettings(rtol=st.krylov.rtol * 1e-3, atol=st.krylov.atol,
                                            maxit=max(20000, 10 * wl.problem.m),
                                            raise_on_maxit=True, mg_nu=nu)
        for _ in range(3):
            st.step_device()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = [st.step_device()[1] for _ in range(5)]
        e1.record()
        torch.cuda.synchronize()
        inner = sum(sum(v) if isinstance(v, list) else v for r in reps for v in r.inner_iters) / 5
        print(f"nu {nu}: {5000 / e0.elapsed_time(e1):.2f} steps/s, inner its {inner:.1f}/step",
              flush=True)


if __name__ == "__main__":
    main()
