"""Profiling driver: a few fc_step calls on a (scaled) config, for ncu / compute-sanitizer.

    python tools/prof_step.py --config C5 --level 6 --steps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--level", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--skip", type=int, default=1, help="skip_quiescent (0 = full update of every tile)")
    a = ap.parse_args()
    from workloads.configs import make_config
    from paper_1308_1472_b200 import fc
    kw = {}
    if a.level is not None:
        kw["base_level" if a.config in ("C2", "C4") else "level"] = a.level
    if a.m is not None:
        kw["m"] = a.m
    w = make_config(a.config, **kw)
    q, cfl, dts = fc.run(w, steps=a.steps, skip_quiescent=a.skip)
    print(f"{w.name}: {a.steps} steps, cells {w.cells}, cfl {cfl[-1]:.6f}")


if __name__ == "__main__":
    main()
