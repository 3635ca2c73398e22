"""Where the C5 default step's time goes beyond its kernels: fc_step in a host loop (CFL to the
host every step, as bench.py) vs fc_run (graphs, fixed dt, no host round trip), and fc_stats'
device-time split.  Device time with CUDA events on the library stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1308_1472_b200 import fc
from workloads.configs import c5

w = c5()
stream = torch.cuda.current_stream()
f = fc.forest_for(w, 0)
f.set_stream(stream.cuda_stream)
f.set_q(np.ascontiguousarray(w.q0))
dt = w.dt0 * 0.5
for _ in range(5):
    f.step(dt)
K = 50
for mode in ("step_loop", "step_loop_timed", "run_graphs"):
    f.set_timing(1 if mode == "step_loop_timed" else 0)
    f.reset_stats()
    if mode == "run_graphs":
        f.run(dt, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if mode == "run_graphs":
        f.run(dt, K)
    else:
        for _ in range(K):
            f.step(dt)
    e1.record(stream)
    torch.cuda.synchronize()
    st = f.stats()
    print(mode, "ms/step", e0.elapsed_time(e1) / K, {k: st[k] for k in ("ms_step", "ms_copy", "ms_ghost", "steps")})
