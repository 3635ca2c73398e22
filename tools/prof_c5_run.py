import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1308_1472_b200 import fc
from workloads.configs import c5
w = c5()
f = fc.forest_for(w, 0)
f.set_q(np.ascontiguousarray(w.q0))
dt = w.dt0 * 0.5
for _ in range(5):
    f.step(dt)
f.run(dt, 3)
