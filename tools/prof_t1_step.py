import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1308_1472_b200 import fc
from workloads.configs import c1
w = c1(level=10, m=8)
for skip in (0, 1):
    f = fc.forest_for(w, 0, skip_quiescent=skip)
    f.set_q(np.ascontiguousarray(w.q0))
    for _ in range(2):
        f.step(w.dt0)
    f.close()
