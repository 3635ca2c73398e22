"""GPU parity of the coarse/fine reflux (fc_problem.reflux): the CUDA path
(k_step face-flux records + k_reflux) against the oracle's orc_reflux on the same inputs, in both
update modes, and exact conservation of sum kappa q on the GPU itself.  Covers periodic AMR scalar
advection (C2 and a 4-tile m = 32 variant), AMR Euler on a periodic brick, the cubed-sphere band
(capacity form across rotated tree links) and a forest large enough for the quiescent filter."""
import dataclasses
import math

import numpy as np
import pytest

import oracle
import workloads.cubed_sphere as CS
from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import EULER_ROE, Workload, c2

pytestmark = pytest.mark.gpu
GAM = 1.4


def amr_euler(steps=15):
    r = np.random.default_rng(1308147 + 31)
    fr = F.forest_refined(F.brick(2, 1, periodic_x=True, periodic_y=True), 1,
                          lambda t, x, y, h: r.random(len(x)) < 0.5)
    m = 8
    X, Y = F.cell_centres(fr, m)
    X = X + fr.tree_ids[:, None, None]
    rho = 1.0 + 0.5 * np.exp(-20 * ((X - 1.0) ** 2 + (Y - 0.5) ** 2))
    u, v, p = 0.3 + 0 * X, -0.2 + 0 * X, 1.0 + 0.3 * np.sin(2 * np.pi * X)
    q0 = np.stack([rho, rho * u, rho * v, p / (GAM - 1) + 0.5 * rho * (u * u + v * v)], 1)
    return Workload("amr_euler", fr, m, 4, 0, EULER_ROE, (GAM, 1.0), q0, None, steps, 1e-3, "cfl", reflux=1)


def sphere_bump(steps=12):
    w = CS.c4_workload(base_level=3, m=8, steps=steps)
    X = w.info["centres"]
    c = np.array([math.cos(5 * math.pi / 6), math.sin(5 * math.pi / 6), 0.0])
    d = np.arccos(np.clip(X @ c, -1, 1))
    w.q0 = (0.1 + np.where(d < 0.5, 0.5 * (1 + np.cos(math.pi * d / 0.5)), 0.0))[:, None]
    return dataclasses.replace(w, reflux=1)


CASES = [dataclasses.replace(c2(steps=40), reflux=1),
         dataclasses.replace(c2(base_level=2, m=32, steps=30), reflux=1),
         dataclasses.replace(c2(base_level=5, m=8, steps=20), reflux=1),    # 1,300 patches: filter path
         amr_euler(),
         sphere_bump(),
         dataclasses.replace(CS.c4_workload(base_level=2, m=16, steps=30), reflux=1)]


def mass(w, q):
    h = np.ldexp(1.0, -w.forest.levels.astype(np.int64))[:, None, None] / w.m
    kap = w.aux[:, 0, 2:w.m + 2, 2:w.m + 2] if w.aux is not None else 1.0
    return np.array([(q[:, k] * kap * h * h).sum() for k in range(w.meqn)])


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name + "_reflux")
def test_reflux_parity_against_oracle(w, skip):
    qo, co, do = oracle.run(w)
    qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
    for k in range(w.meqn):
        scale = np.abs(qo[:, k]).max() or np.abs(qo).max()
        assert np.abs(qg[:, k] - qo[:, k]).max() <= 1e-12 * scale, (w.name, k)
    np.testing.assert_allclose(cg, co, rtol=1e-12, atol=0)
    m0, mo, mg = mass(w, w.q0), mass(w, qo), mass(w, qg)
    for k in range(w.meqn):
        assert abs(mg[k] - mo[k]) <= 1e-13 * max(abs(mo[k]), abs(m0[k])), (w.name, k)


@pytest.mark.parametrize("w", [CASES[0], CASES[3], CASES[4]], ids=lambda w: w.name)
def test_reflux_conserves_on_gpu(w):
    """sum kappa q after the run equals the initial total to roundoff on the GPU alone."""
    q, _, _ = fc.run(w)
    m0, m1 = mass(w, w.q0), mass(w, q)
    for k in range(w.meqn):
        assert abs(m1[k] - m0[k]) <= 1e-14 * w.steps * max(abs(m0[k]), 1e-300) + 1e-15, (w.name, k, m1[k] - m0[k])


def test_reflux_noop_on_uniform_forest():
    from workloads.configs import c5
    w = c5(level=3, m=16, steps=10)
    qa, ca, _ = fc.run(w)
    qb, cb, _ = fc.run(dataclasses.replace(w, reflux=1))
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)
