"""Cost of one multigrid V-cycle of the config-2 stage block (block 0),
eager vs captured in a CUDA graph, for hierarchies truncated at different
depths (`python profiles/vcycle_probe.py [config] [ncu]`).  With `ncu` only
a few eager V-cycles run (for a per-kernel launch list)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import _lib, configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ncu = "ncu" in sys.argv[2:]
    wl = configs.build(k)
    st, prob = wl.stepper, wl.problem
    fac0 = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
    m = prob.m
    r = la.to_dev(np.random.default_rng(1).standard_normal(m))
    z = la.dev_empty(m)
    lib = _lib.load()
    ratios = [None] if ncu else ["generic", None, 2.0, 8.0, 32.0, 128.0]
    for ratio in ratios:
        if ratio in (None, "generic"):
            fac = fac0
            fac._mg.structured = ratio is None
        else:
            s = la.BlockSolveSettings(rtol=1e-6, mg_coarse_ratio=ratio)
            fac = la.BlockFactorization(prob.mass, prob.stiffness, fac0.alpha, fac0.beta,
                                        fac0.dofs, s)
        h = fac._mg.handle

        def vc():
            _lib.check(lib.irk_mg_vcycle(la.ctx(), h, la.ptr(r), la.ptr(z)), "vcycle")

        for _ in range(3):
            vc()
        torch.cuda.synchronize()
        if ncu:
            for _ in range(3):
                vc()
            torch.cuda.synchronize()
            return
        n = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            vc()
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / n * 1e3
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            vc()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    vc()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graphed = e0.elapsed_time(e1) / 50 * 1e3
        its = fac.dev_solve(r, la.dev_empty(m), settings=la.BlockSolveSettings(rtol=1e-6))
        torch.cuda.synchronize()
        e0.record()
        tot = 0
        for _ in range(10):
            tot += fac.dev_solve(r, z, settings=la.BlockSolveSettings(rtol=1e-6))
        e1.record()
        torch.cuda.synchronize()
        print(f"ratio {ratio}: levels {fac._mg.levels} structured {fac._mg.structured}: V-cycle {eager:.1f} us eager, "
              f"{graphed:.1f} us graphed; solve {e0.elapsed_time(e1) / 10 * 1e3:.1f} us, "
              f"{tot / 10:.1f} its", flush=True)


if __name__ == "__main__":
    main()
