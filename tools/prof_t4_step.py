"""Two T4 steps (C4 physics, L7/L8 band on the cubed sphere) in default mode, for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1308_1472_b200 import fc
from workloads.cubed_sphere import c4_workload

w = c4_workload(base_level=7, m=16, steps=2)
f = fc.forest_for(w, 0)
f.set_q(np.ascontiguousarray(w.q0))
for _ in range(2):
    f.step(w.dt0)
