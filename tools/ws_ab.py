"""A/B timing of the systems update kernels on one GPU: C5 (full size) and T3 (C3 physics L8,
m = 32), full-update mode, K steps after 3 warm-ups, CUDA events; the kernel is chosen by the
environment (FC_WS=0: phased k_step + ghost kernels; default: warp-sweep k_step_ws, fused gather).

    FC_WS=0 python tools/ws_ab.py [--steps 10] [--only C5,T3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--only", default="C5,T3")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    from workloads.configs import c3, c5
    stream = torch.cuda.current_stream()
    for name in a.only.split(","):
        w = c5() if name == "C5" else c3(level=8, m=32)
        qd = torch.from_numpy(np.ascontiguousarray(w.q0)).cuda()
        f = fc.forest_for(w, 0, skip_quiescent=0)
        f.set_stream(stream.cuda_stream)
        f.set_q(qd)
        dt = w.dt0
        for _ in range(3):
            rc, cfl = f.step(dt)
            dt = w.next_dt(dt, cfl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            rc, cfl = f.step(dt)
            dt = w.next_dt(dt, cfl)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        f.reset_stats()
        f.set_timing(True)
        for _ in range(3):
            rc, cfl = f.step(dt)
            dt = w.next_dt(dt, cfl)
        st = f.stats()
        f.close()
        print(json.dumps({"workload": name, "ws": os.environ.get("FC_WS", "1"), "ms_per_step": ms,
                          "G_cell_updates_per_s": w.cells / ms / 1e6,
                          "update_ms": st["ms_step"] / max(1, st["step_kernel_launches"]),
                          "ghost_ms": st["ms_ghost"] / max(1, st["steps"]), "cfl": cfl}), flush=True)
        del qd


if __name__ == "__main__":
    main()
