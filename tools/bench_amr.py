"""AMR workloads on one GPU: global-dt vs sub-cycled stepping, with and without the reflux
(SURVEY §8(d) throughput variants T2; §8(f) #1-#2).  T2 = C2 physics (periodic advection, MC,
transverse) on the L{b}/L{b+1} forest of the C2 rule (refine a level-b patch iff its centre is
within 0.25 of (0.5, 0.5)).  For each mode: device time (CUDA events on the library's stream) to
advance the solution by one coarse dt = 2 fine dt, i.e. 2 x fc_step(dt_f) or 1 x
fc_step_subcycled(2 dt_f), averaged over K such intervals after W warm-ups.

    python tools/bench_amr.py [--base 8] [--m 16] [--steps 20] [--warmup 3] [--radius 0.25]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", type=int, default=8)
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--radius", type=float, default=0.25, help="refined disc radius of the C2 rule")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    from workloads.configs import c2
    w = c2(base_level=a.base, m=a.m, radius=a.radius)
    lv = w.forest.levels
    cells = w.num_patches * a.m * a.m
    fine_cells = int((lv == lv.max()).sum()) * a.m * a.m
    stream = torch.cuda.current_stream()
    dtf = w.dt0
    out = {"workload": f"T2: C2 physics, L{a.base}/L{a.base + 1}, m={a.m}, radius {a.radius}", "patches": w.num_patches, "cells": cells,
           "fine_cells": fine_cells}
    for mode in ("global", "subcycled"):
        for reflux in (0, 1):
            for skip in (1, 0):
                f = fc.forest_for(w, 0, skip_quiescent=skip)
                f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject,
                              skip, reflux)
                f.set_stream(stream.cuda_stream)
                f.set_q(np.ascontiguousarray(w.q0))

                def interval():
                    if mode == "global":
                        f.step(dtf)
                        f.step(dtf)
                    else:
                        f.step_subcycled(2 * dtf)
                for _ in range(a.warmup):
                    interval()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(a.steps):
                    interval()
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.steps
                upd = 2 * cells if mode == "global" else (cells - fine_cells) + 2 * fine_cells
                out[f"{mode}_reflux{reflux}_{'default' if skip else 'full'}"] = {
                    "ms_per_coarse_dt": ms, "level_cell_updates_per_coarse_dt": upd,
                    "cell_updates_per_s": upd / (ms / 1e3)}
                f.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
