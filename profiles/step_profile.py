"""Kernel-time breakdown of time steps (torch.profiler / CUPTI; no nsys in
the image).  Prints the top kernels by total device time over the profiled
steps.

  python profiles/step_profile.py [config] [steps]
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    wl = configs.build(k)
    st = wl.stepper
    for _ in range(2):
        st.step_device()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            st.step_device()
        torch.cuda.synchronize()
    tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70)
    print(tab)


if __name__ == "__main__":
    main()
