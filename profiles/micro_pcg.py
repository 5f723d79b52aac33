"""Micro-benchmark of one pre-combined block solve at config-2 size:
persistent cooperative PCG vs the two-kernel path (IRK_NO_PERSIST=1),
fixed iteration count, CUDA events.

  python profiles/micro_pcg.py [iters]
"""

import os
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

    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    wl = configs.build(2, n=n)
    st, prob = wl.stepper, wl.problem
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    fac = pc.block_factors[0]
    m = prob.m
    b = la.to_dev(np.random.default_rng(1).standard_normal(m))
    x = la.dev_empty(m)
    fixed = la.BlockSolveSettings(rtol=0.0, atol=0.0, maxit=iters)
    out = {}
    for mode in ("persist", "two-kernel"):
        if mode == "two-kernel":
            os.environ["IRK_NO_PERSIST"] = "1"
        else:
            os.environ.pop("IRK_NO_PERSIST", None)
            os.environ["IRK_PERSIST"] = "1"
        fac.dev_solve(b, x, settings=fixed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        its = fac.dev_solve(b, x, settings=fixed)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = e0.elapsed_time(e1) * 1e3 / its
        xs = x.clone()
        out[mode + "_x"] = xs
    d = (out["persist_x"] - out["two-kernel_x"]).norm().item() / out["two-kernel_x"].norm().item()
    print(f"m={m} its={iters}: persistent {out['persist']:.2f} us/it, two-kernel "
          f"{out['two-kernel']:.2f} us/it, rel diff {d:.2e}")


if __name__ == "__main__":
    main()
