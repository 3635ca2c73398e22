"""Algorithmic fp64 flops per cell-update of each config, counted on the oracle's own patch update
(tools/count_flops.cpp) over a sample of patches from the config's initial state plus patches
advanced a few steps (so shocks, rarefactions and smooth regions are all represented).

    python tools/count_flops.py [C5 C3 C4 C1]     -> prints JSON {config: flops_per_cell_update}
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build():
    exe = os.path.join(ROOT, "tools", "count_flops")
    src = os.path.join(ROOT, "tools", "count_flops.cpp")
    deps = [src] + [os.path.join(ROOT, "oracle", f) for f in ("claw.c", "oracle.h", "oracle_internal.h")]
    if not os.path.exists(exe) or any(os.path.getmtime(d) > os.path.getmtime(exe) for d in deps):
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fpermissive", "-w", "-o", exe, src], check=True)
    return exe


def count(name, nsample=48, advance=3):
    import oracle
    from workloads.configs import make_config
    kw = {"C5": dict(level=5), "C3": dict(level=4), "C4": dict(base_level=3), "C1": {}}[name]
    w = make_config(name, **kw)
    q, _, dts = oracle.run(w, steps=advance)
    rng = np.random.default_rng(1308147)
    f = oracle.forest_for(w)
    ids = rng.choice(w.num_patches, size=min(nsample, w.num_patches), replace=False)
    exe = build()
    tot_f = tot_c = 0
    for state in (w.q0, q):
        with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as fq, \
                tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as fa:
            for p in ids:
                fq.write(f.padded_sample(state, int(p)).astype(np.float64).tobytes())
                if w.aux is not None:
                    fa.write(np.ascontiguousarray(w.aux[p]).tobytes())
        dx = np.ldexp(1.0, -int(w.forest.levels[ids[0]])) / w.m
        args = [exe, str(w.kind), repr(w.params[0]), repr(w.params[1]), str(w.limiter), str(w.m),
                str(w.meqn), repr(dts[-1]), repr(dx), fq.name] + ([fa.name] if w.aux is not None else [])
        out = subprocess.run(args, capture_output=True, text=True, check=True).stdout.split()
        tot_f += int(out[0])
        tot_c += int(out[1])
        os.unlink(fq.name)
        os.unlink(fa.name)
    return tot_f / tot_c


if __name__ == "__main__":
    names = sys.argv[1:] or ["C5", "C3", "C4", "C1"]
    print(json.dumps({n: count(n) for n in names}))
