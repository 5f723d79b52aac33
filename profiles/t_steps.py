import sys; sys.path.insert(0,'/root/repo')
from paper_2403_08084_b200 import configs
n = int(sys.argv[1]); steps = int(sys.argv[2]); k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = configs.build(k, n=n)
for i in range(steps):
    u, rep = wl.stepper.step(wl.problem)
print("ok", steps, rep.krylov_iters)
