"""Throughput of every BASELINE config (C1-C5 at full size) on one GPU, default (quiescent
shortcut on) and full-update modes: K steps of the config's own dt policy, CUDA events around the
step loop (each fc_step includes its CFL read-back).  Prints one JSON line per config and mode.

    python tools/bench_configs.py [--steps K]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=0, help="0 = the config's own step count")
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    from workloads.configs import make_config
    for name in a.configs.split(","):
        w = make_config(name)
        steps = a.steps or w.steps
        for skip in (1, 0):
            f = fc.forest_for(w, 0, skip_quiescent=skip)
            stream = torch.cuda.current_stream()
            f.set_stream(stream.cuda_stream)
            qd = torch.from_numpy(np.ascontiguousarray(w.q0)).cuda()
            f.set_q(qd)
            dt = w.dt0
            for _ in range(3):                       # warm-up
                rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            f.set_q(qd)
            dt = w.dt0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                rc, cfl = f.step(dt, raise_on_reject=False)
                if rc == fc.FC_ECFL:
                    dt = dt * w.cfl_target / cfl
                    rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            st = f.stats()
            print(json.dumps({"config": name, "mode": "default" if skip else "full_update", "steps": steps,
                              "cells": w.cells, "ms_per_step": ms / steps,
                              "cell_updates_per_s": w.cells * steps / (ms / 1e3),
                              "fused_path": st["uniform_fast_path"]}), flush=True)
            f.close()


if __name__ == "__main__":
    main()
