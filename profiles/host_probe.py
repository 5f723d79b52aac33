"""Host-side cost of a time step: cProfile of step_device (config 2)."""
import cProfile
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    wl = configs.build(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    st = wl.stepper
    for _ in range(3):
        st.step_device()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        st.step_device()
    torch.cuda.synchronize()
    pr.disable()
    ps = pstats.Stats(pr).sort_stats("tottime")
    ps.print_stats(18)


if __name__ == "__main__":
    main()
