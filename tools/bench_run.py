"""Per-step cost of the small fixed-dt configs (C1, C2, C4) with fc_step in a host loop (one host
round trip per step for the CFL) vs fc_run (the step captured as CUDA graphs, replayed back to back;
CFLs checked once at the end).  Device time with CUDA events around K steps after warm-up.

    python tools/bench_run.py [--steps 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    from workloads.configs import c1, c2
    from workloads.cubed_sphere import c4_workload
    stream = torch.cuda.current_stream()
    for w in (c1(), c2(), c4_workload()):
        out = {"config": w.name, "cells": w.cells, "steps": a.steps}
        for mode in ("step_loop", "run_graphs"):
            f = fc.forest_for(w, 0)
            f.set_stream(stream.cuda_stream)
            f.set_q(np.ascontiguousarray(w.q0))
            if mode == "step_loop":
                for _ in range(5):
                    f.step(w.dt0)
            else:
                f.run(w.dt0, a.steps)        # capture + warm-up
            f.set_q(np.ascontiguousarray(w.q0))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            if mode == "step_loop":
                for _ in range(a.steps):
                    f.step(w.dt0)
            else:
                f.run(w.dt0, a.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            ms = e0.elapsed_time(e1)
            out[mode] = {"us_per_step": 1000 * ms / a.steps, "wall_us_per_step": 1e6 * wall / a.steps,
                         "cell_updates_per_s": w.cells * a.steps / (ms / 1e3)}
            f.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
