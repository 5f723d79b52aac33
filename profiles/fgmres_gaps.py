"""GPU idle time at the per-iteration host read of the FGMRES Hessenberg
column: IRK_FGMRES_GAPS=1 python profiles/fgmres_gaps.py [config] [steps].
Pairs (end of iteration j's GPU work, first enqueue of iteration j+1): the
elapsed time between them is the D2H copy + host latency the GPU waits."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("IRK_FGMRES_GAPS", "1")


def main():
    import numpy as np
    import torch

    from paper_2403_08084_b200 import configs
    from paper_2403_08084_b200 import sparsela as la

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = configs.build(k)
    st = wl.stepper
    for _ in range(3):
        st.step_device()
    torch.cuda.synchronize()
    la._GAPS.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st.step_device()
    e1.record()
    torch.cuda.synchronize()
    ev = la._GAPS
    gaps = []
    i = 0
    while i + 1 < len(ev):
        gaps.append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
        i += 2
    g = np.array(gaps)
    t = e0.elapsed_time(e1) / steps
    print(f"config {k}: {t:.2f} ms/step; {len(g) / steps:.1f} host reads/step, gap mean "
          f"{g.mean():.1f} us, median {np.median(g):.1f} us -> {g.sum() / steps / 1e3:.3f} ms/step")


if __name__ == "__main__":
    main()
