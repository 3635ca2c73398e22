"""One T2 step (C2 physics, L8/L9) in full-update mode, for ncu of the scalar k_step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1308_1472_b200 import fc
from workloads.configs import c2

w = c2(base_level=8, m=16)
f = fc.forest_for(w, 0, skip_quiescent=0)
f.set_q(np.ascontiguousarray(w.q0))
for _ in range(3):
    f.step(w.dt0)
