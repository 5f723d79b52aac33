"""Config 2, steps 1..20 from u0: per-step outer FGMRES iterations, inner CG
iterations and device time vs the inner block-solve tolerance / method.
`python profiles/r02/outer_its_probe.py [rtol ...]`."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    k = int(os.environ.get("CFG", "2"))
    rtols = [float(v) for v in sys.argv[1:]] or [1e-6, 1e-8, 1e-10]
    extra = json.loads(os.environ.get("BLOCK", "{}"))
    for rt in rtols:
        wl = configs.build(k, inner_rtol=rt, **extra)
        st = wl.stepper
        snap = (st.u.copy(), st.step_index, st._t_base)
        for _ in range(3):
            st.step_device()
        torch.cuda.synchronize()
        st.u, st.step_index, st._t_base = snap[0].copy(), snap[1], snap[2]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = [st.step_device()[1] for _ in range(wl.steps)]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / wl.steps
        kr = [r.krylov_iters for r in reps]
        inner = [sum(sum(v) if isinstance(v, list) else (v or 0) for v in r.inner_iters)
                 for r in reps]
        print(f"cfg {k} {extra} inner rtol {rt:g}: {1e3 / ms:.2f} steps/s; krylov {kr} "
              f"(mean {sum(kr) / len(kr):.2f}); inner/step {sum(inner) / len(inner):.1f}",
              flush=True)


if __name__ == "__main__":
    main()
