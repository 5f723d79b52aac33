"""Steps/s and outer Krylov iterations vs the inner block-solve tolerance
(the configs whose BASELINE text leaves it unspecified):
`python profiles/inner_rtol_sweep.py config [rtol ...]`."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    rtols = [float(v) for v in sys.argv[2:]] or [1e-6, 1e-4, 1e-3, 1e-2]
    for rt in rtols:
        wl = configs.build(k, inner_rtol=rt)
        st = wl.stepper
        for _ in range(3):
            st.step_device()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = [st.step_device()[1] for _ in range(5)]
        e1.record()
        torch.cuda.synchronize()
        print(f"config {k} inner rtol {rt:g}: {5000 / e0.elapsed_time(e1):.2f} steps/s, krylov "
              f"{sum(r.krylov_iters for r in reps) / 5:.1f}/step", flush=True)


if __name__ == "__main__":
    main()
