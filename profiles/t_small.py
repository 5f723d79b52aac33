import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import numpy as np
from paper_2403_08084_b200 import configs
wl=configs.build(2, n=32)
for i in range(2):
    u,rep=wl.stepper.step(wl.problem)
print("ok", rep.krylov_iters)
