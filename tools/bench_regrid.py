"""Cost of one dynamic regrid (fc_regrid) on T2 (C2 physics, L8/L9, 104,212 patches): wall time of
the call (device tag + host planning + new handle creation + device transfer), split by a second
timing of fc_forest_create for the new mesh alone.

    python tools/bench_regrid.py [--base 8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", type=int, default=8)
    a = ap.parse_args()
    import numpy as np
    from paper_1308_1472_b200 import fc
    from workloads.configs import c2
    w = c2(base_level=a.base, m=16)
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    for _ in range(3):
        f.step(w.dt0)
    t0 = time.perf_counter()
    g = f.regrid(0.02, 0.002, a.base - 1, a.base + 1)
    t1 = time.perf_counter()
    lv, tr = g.leaves()
    t2 = time.perf_counter()
    h = fc.Forest(lv, tr, w.forest.conn, w.m, w.meqn, 0, 1.0, 0)
    t3 = time.perf_counter()
    print(json.dumps({"workload": f"T2 L{a.base}/L{a.base + 1}", "patches_before": w.num_patches,
                      "patches_after": int(len(lv)), "levels_after": np.bincount(lv).tolist(),
                      "regrid_s": t1 - t0, "forest_create_s": t3 - t2}))


if __name__ == "__main__":
    main()
