"""Time steps/s of a config for multigrid smoothing / coarsening variants
(`python profiles/mg_tune.py [config] [steps]`)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import configs

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    variants = [dict(method="pcg")] + [
        dict(mg_nu=nu, mg_coarse_ratio=r, mg_coarse_steps=c)
        for nu in (1, 2, 3) for r in (0.5, 4.0) for c in (4, 8)]
    if len(sys.argv) > 3:
        import json
        variants = json.loads(sys.argv[3])
    import gc

    for v in variants:
        gc.collect()
        torch.cuda.synchronize()
        wl = configs.build(k, **v)
        st = wl.stepper
        for _ in range(2):
            st.step_device()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = [st.step_device()[1] for _ in range(steps)]
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps
        per = []
        for _ in range(3):
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            st.step_device()
            f1.record()
            torch.cuda.synchronize()
            per.append(round(f0.elapsed_time(f1), 1))
        inner = sum(sum(sum(x) if isinstance(x, list) else x for x in r.inner_iters)
                    for r in reps) / steps
        kr = sum(r.krylov_iters for r in reps) / steps
        del wl, st
        print(f"{v}: {t:.2f} ms/step ({1e3 / t:.2f} steps/s), krylov {kr:.1f}, inner {inner:.1f}, next {per}")


if __name__ == "__main__":
    main()
