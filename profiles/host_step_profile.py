"""Host-side cost of time steps (cProfile over step_device, GPU synchronised
at the end): `python profiles/host_step_profile.py [config] [steps]`."""
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = configs.build(k)
    st = wl.stepper
    for _ in range(3):
        st.step_device()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(steps):
        st.step_device()
    torch.cuda.synchronize()
    pr.disable()
    print(f"{(time.perf_counter() - t0) / steps * 1e3:.2f} ms/step wall (profiled)")
    s = io.StringIO()
    st_ = pstats.Stats(pr, stream=s); st_.sort_stats(sys.argv[3] if len(sys.argv) > 3 else "cumtime").print_stats(40)
    print(s.getvalue())


if __name__ == "__main__":
    main()
