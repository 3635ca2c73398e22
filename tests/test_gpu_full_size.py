"""Full-size parity (BASELINE.json north_star: "on all five configs, every GPU result matches the
oracle within the stated tolerance ... after the stated number of steps"): C3 (200 steps), C4 (500)
and C5 (100) at BASELINE.json's full sizes, in the launch configuration bench.py times, against
the oracle's whole-forest run on all host cores (its OpenMP loop over patches is bitwise equal to
one thread, tests/test_oracle_openmp.py).  The GPU replays the oracle's dt list;
both GPU update modes (full update, exact quiescent shortcut) are checked.

Bars: per conserved component max|dq_k| <= 1e-12 max|q_k| over all interior
cells, total mass (sum q * area, Morton order) relative <= 1e-13, CFLs relative <= 1e-12.
Expected run time: C5 dominates (the oracle at ~16 M cell-updates/s on 16 cores: ~7 min).
"""
import os
import time

import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads.configs import c3, c5
from workloads.cubed_sphere import c4_workload

pytestmark = pytest.mark.gpu


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def check(w, qg, qo, cg, co):
    rel = []
    for k in range(w.meqn):
        scale = np.abs(qo[:, k]).max()
        if scale == 0.0:
            scale = np.abs(qo).max()
        err = np.abs(qg[:, k] - qo[:, k]).max()
        rel.append(err / scale)
        assert err <= 1e-12 * scale, (w.name, k, err, scale)
        area = np.ldexp(1.0, -2 * w.forest.levels.astype(np.int64))[:, None, None]
        if w.aux is not None:     # capacity form: the conserved mass is sum kappa q dA
            m = w.m
            area = area * w.aux[:, 0, 2:m + 2, 2:m + 2]
        mg, mo = (qg[:, k] * area).sum(), (qo[:, k] * area).sum()
        assert abs(mg - mo) <= 1e-13 * max(abs(mo), (np.abs(qo[:, k]) * area).sum()), (w.name, k, mg, mo)
    np.testing.assert_allclose(cg, co, rtol=1e-12, atol=0)
    return rel


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_config_after_its_steps(name):
    w = {"C3": lambda: c3(), "C4": lambda: c4_workload(), "C5": lambda: c5()}[name]()
    assert (name, w.steps) in (("C3", 200), ("C4", 500), ("C5", 100))
    t0 = time.time()
    qo, co, do = oracle.run(w, nthreads=host_cores())
    t_orc = time.time() - t0
    for skip in (0, 1):
        qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
        rel = check(w, qg, qo, cg, co)
        print(f"{w.name} {w.num_patches} patches x {w.steps} steps, skip={skip}: max rel err per "
              f"component {[f'{r:.2e}' for r in rel]}; oracle {t_orc:.0f} s on {host_cores()} cores")
