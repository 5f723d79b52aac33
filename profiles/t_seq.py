import sys; sys.path.insert(0,'/root/repo')
from paper_2403_08084_b200 import configs
seq = [int(a) for a in sys.argv[1:]] or [1024, 32]
for n in seq:
    wl = configs.build(2, n=n)
    u, rep = wl.stepper.step(wl.problem)
    print("n", n, "ok", rep.krylov_iters, flush=True)
