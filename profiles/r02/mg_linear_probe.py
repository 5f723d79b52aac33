"""Experiment: multigrid as a LINEAR fixed-count inner block solver
(stationary V-cycle iteration, optionally Chebyshev-accelerated with
Lanczos bounds of V*B) instead of MG-PCG to rtol 1e-6, on config 2:
(1) residual per iteration for a random right-hand side; (2) the outer
FGMRES iterations per time step when the GS preconditioner uses it.
Python-driven (slow): only the iteration counts matter here."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2403_08084_b200 import _lib, configs
    from paper_2403_08084_b200 import sparsela as la
    from paper_2403_08084_b200._lib import call, ctx, ptr
    from paper_2403_08084_b200.stepper import _SPLIT

    wl = configs.build(2)
    st, prob = wl.stepper, wl.problem
    pc = st._preconditioner(_SPLIT[st.formulation], prob)
    m = prob.m

    def V(fac, r):
        z = torch.empty_like(r)
        call("irk_mg_vcycle", ctx(), fac._mg.handle, ptr(r), ptr(z))
        return z

    def Bx(fac, x):
        y = torch.empty_like(x)
        fac._B.spmv(x, y)
        return y

    def lanczos(fac, k=30):
        # CG on B with the V-cycle preconditioner: tridiagonal from alpha/beta
        b = torch.randn(m, dtype=torch.float64, device="cuda")
        b = b - (Bx(fac, torch.zeros_like(b)))  # noop, keeps shapes
        x = torch.zeros_like(b); r = b.clone(); z = V(fac, r); p = z.clone()
        rz = float(r @ z); al, be = [], []
        for _ in range(k):
            q = Bx(fac, p); a = rz / float(p @ q)
            x += a * p; r -= a * q
            z = V(fac, r); rz2 = float(r @ z); bb = rz2 / rz; rz = rz2
            p = z + bb * p; al.append(a); be.append(bb)
        T = np.zeros((k, k))
        for i in range(k):
            T[i, i] = 1 / al[i] + (be[i - 1] / al[i - 1] if i else 0)
            if i + 1 < k:
                T[i, i + 1] = T[i + 1, i] = np.sqrt(be[i]) / al[i]
        ev = np.linalg.eigvalsh(T)
        return ev[0], ev[-1]

    bounds = []
    for i, fac in enumerate(pc.block_factors):
        lo, hi = lanczos(fac)
        bounds.append((lo, hi))
        print(f"block {i}: eig(V B) in [{lo:.4f}, {hi:.4f}]", flush=True)

    def solve(fac, bnd, b, k, mode):
        x = torch.zeros_like(b)
        r = b.clone()
        nb = float(torch.linalg.norm(b))
        hist = []
        if mode == "richardson":
            for _ in range(k):
                x += V(fac, r)
                r = b - Bx(fac, x)
                hist.append(float(torch.linalg.norm(r)) / nb)
            return x, hist
        lo, hi = bnd[0] * 0.95, bnd[1] * 1.02
        theta, delta = (hi + lo) / 2, (hi - lo) / 2
        sigma = theta / delta
        rho = 1 / sigma
        d = V(fac, r) / theta
        for i in range(k):
            x += d
            r = b - Bx(fac, x)
            hist.append(float(torch.linalg.norm(r)) / nb)
            rho_n = 1 / (2 * sigma - rho)
            d = rho_n * rho * d + (2 * rho_n / delta) * V(fac, r)
            rho = rho_n
        return x, hist

    b = torch.randn(m, dtype=torch.float64, device="cuda")
    for mode in ("richardson", "chebyshev"):
        _, h = solve(pc.block_factors[0], bounds[0], b, 10, mode)
        print(mode, " ".join(f"{v:.1e}" for v in h), flush=True)

    # outer FGMRES iterations with the linear solver in the preconditioner
    for mode, k in (("chebyshev", 4), ("chebyshev", 5), ("chebyshev", 6), ("richardson", 7)):
        for i, fac in enumerate(pc.block_factors):
            def dev_solve(rhs, x, ld_rhs=1, ld_x=1, nb=1, settings=None, defer=False,
                          checked=False, fac=fac, bnd=bounds[i]):
                y, _ = solve(fac, bnd, rhs.reshape(-1)[::ld_rhs][:m].clone(), k, mode)
                x.reshape(-1)[::ld_x][:m].copy_(y)
                return k
            fac.dev_solve = dev_solve
        snap = (st.u.copy(), st.step_index, st._t_base)
        its = []
        for _ in range(10):
            _, rep = st.step_device(prob)
            its.append(rep.krylov_iters)
        st.u, st.step_index, st._t_base = snap[0].copy(), snap[1], snap[2]
        print(f"{mode} k={k}: FGMRES its per step {its}", flush=True)


if __name__ == "__main__":
    main()
