"""Throughput variants of SURVEY §8(d) on one GPU: T1 (C1 physics, uniform L10, m = 8), T2 (C2
physics, L8/L9), T3 (C3 physics, L8, m = 32), T4 (C4 physics, L7/L8 band) -- 20 steps of each
config's dt policy after 3 warm-ups, default (quiescent shortcut) and full-update modes, CUDA events
around the step loop.  Prints one JSON line per variant and mode with cell-updates/s and the
fraction of the HBM roofline rate (compulsory 16 meqn + 8 maux bytes per cell-update at the
measured copy bandwidth).

    python tools/bench_variants.py [--only T1,T2,T3,T4] [--steps 20]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make(name):
    from workloads.configs import c1, c2, c3
    from workloads.cubed_sphere import c4_workload
    if name == "T1":
        return c1(level=10, m=8)
    if name == "T2":
        return c2(base_level=8, m=16)
    if name == "T3":
        return c3(level=8, m=32)
    return c4_workload(base_level=7, m=16, steps=20)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="T1,T2,T3,T4")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    stream = torch.cuda.current_stream()
    for name in a.only.split(","):
        t0 = time.time()
        w = make(name)
        gen_s = time.time() - t0
        qd = torch.from_numpy(np.ascontiguousarray(w.q0)).cuda()
        for skip in (1, 0):
            f = fc.forest_for(w, 0, skip_quiescent=skip)
            f.set_stream(stream.cuda_stream)
            f.set_q(qd)
            dt = w.dt0
            for _ in range(3):
                rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            f.set_q(qd)
            dt = w.dt0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.steps):
                rc, cfl = f.step(dt, raise_on_reject=False)
                if rc == fc.FC_ECFL:
                    dt = dt * w.cfl_target / cfl
                    rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            rate = w.cells / (ms / 1e3)
            bpc = 16 * w.meqn + 8 * w.maux
            print(json.dumps({"variant": name, "workload": w.name, "mode": "default" if skip else "full_update",
                              "patches": w.num_patches, "cells": w.cells, "ms_per_step": ms,
                              "cell_updates_per_s": rate, "bytes_per_cell_update": bpc,
                              "hbm_roofline_frac": rate * bpc / (hbm * 1e9), "generate_s": gen_s}), flush=True)
            f.close()
        del qd


if __name__ == "__main__":
    main()
