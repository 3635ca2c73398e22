"""C5 physics with the HLLE solver vs Roe + Harten-Hyman (full size, both update modes): device time
per step over K steps of the Clawpack dt policy from the IC (CUDA events on the library stream).
Second-order HLLE reaches a non-physical state on this problem (reading 25): reported as
such, with the step it happened at."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc
    from workloads.configs import EULER_HLLE, c5
    K = 20
    base = c5()
    stream = torch.cuda.current_stream()
    for name, w in (("roe_hh", base), ("hlle", dataclasses.replace(base, kind=EULER_HLLE, params=(base.params[0], 0.0)))):
        for skip in (1, 0):
            f = fc.forest_for(w, 0, skip_quiescent=skip)
            f.set_stream(stream.cuda_stream)
            f.set_q(np.ascontiguousarray(w.q0))
            dt = w.dt0
            for _ in range(3):
                rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            try:
                for k in range(K):
                    rc, cfl = f.step(dt, raise_on_reject=False)
                    dt = w.next_dt(dt, cfl)
            except fc.FcError as e:
                print(json.dumps({"solver": name, "mode": "default" if skip else "full_update",
                                  "error": str(e), "after_steps": 3 + k}))
                f.close()
                continue
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            print(json.dumps({"solver": name, "mode": "default" if skip else "full_update", "ms_per_step": ms,
                              "cell_updates_per_s": w.cells / (ms / 1e3)}))
            f.close()


if __name__ == "__main__":
    main()
