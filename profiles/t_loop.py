import sys, numpy as np; sys.path.insert(0,'/root/repo')
from paper_2403_08084_b200 import configs, sparsela as la
from paper_2403_08084_b200.stepper import _SPLIT
n = int(sys.argv[1]); reps = int(sys.argv[2])
wl = configs.build(2, n=n)
st, prob = wl.stepper, wl.problem
pc = st._preconditioner(_SPLIT[st.formulation], prob)
m = prob.m
rng = np.random.default_rng(0)
xs = None
for r in range(reps):
    for i in range(3):
        fac = pc.block_factors[i]
        b = la.to_dev(rng.standard_normal(m)); x = la.dev_empty(m)
        fac.dev_solve(b, x, settings=la.BlockSolveSettings(rtol=1e-6))
print("ok", reps * 3, "solves")
