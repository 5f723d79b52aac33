"""Cost of one sine-transform preconditioner application z = B_s^-1 r on the
config-2 (1024^2) and config-4 (2048^2) blocks, replayed from a captured CUDA
graph (warm L2, as inside a CG solve), plus its quality: ||r - B z|| / ||r||
(B_s differs from B only by the symmetrised diagonal coupling, ~1e-4).

  python profiles/r02/dst_probe.py [config ...]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2403_08084_b200 import _lib, configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200.stepper import _SPLIT

    lib = _lib.load()
    for k in [int(a) for a in sys.argv[1:]] or [2, 4]:
        wl = configs.build(k)
        st, prob = wl.stepper, wl.problem
        if st.formulation.name == "DIRK":
            fac = st._dirk_factor(st.tableau.A[0, 0], prob)
        else:
            fac = st._preconditioner(_SPLIT[st.formulation], prob).block_factors[0]
        assert fac._mg.dst, "no sine-transform preconditioner on this block"
        m = prob.m
        rh = np.random.default_rng(1).standard_normal(m)
        rh[fac.dofs] = 0.0
        r = la.to_dev(rh)
        z = la.dev_empty(m)
        h = fac._mg.handle

        def ap():
            _lib.check(lib.irk_mg_vcycle(la.ctx(), h, la.ptr(r), la.ptr(z)), "dst apply")

        for _ in range(3):
            ap()
        torch.cuda.synchronize()
        zz = la.to_host(z) if hasattr(la, "to_host") else z.cpu().numpy()
        res = rh - fac.matvec(zz)
        print(f"config {k}: ||r - B z|| / ||r|| = {np.linalg.norm(res) / np.linalg.norm(rh):.3e}")
        n = 50
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ap()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(n):
                    ap()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / n * 1e3
        print(f"config {k}: sine-transform application {t:.1f} us "
              f"({48 * m / t / 1e3:.0f} GB/s of its 48 B/point)")
        del wl, fac


if __name__ == "__main__":
    main()
