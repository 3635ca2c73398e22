"""T3 steps (C3 physics, uniform L8, m = 32: 2 x 2 tiles of 16 per patch) in full-update mode, for
ncu of the systems k_step on a multi-tile patch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1308_1472_b200 import fc
from workloads.configs import c3

w = c3(level=8, m=32)
f = fc.forest_for(w, 0, skip_quiescent=0)
f.set_q(np.ascontiguousarray(w.q0))
for _ in range(2):
    f.step(w.dt0)
