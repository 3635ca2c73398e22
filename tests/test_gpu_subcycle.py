"""GPU parity of sub-cycled stepping (fc_step_subcycled, PAPER.md:201-202,
277-290) against the oracle's orc_step_subcycled on the same inputs and the same coarse dt list,
with and without the reflux, in both update modes; exact conservation with the reflux on the GPU;
and the one-level case reducing to fc_step."""
import dataclasses
import math

import numpy as np
import pytest

import oracle
import workloads.cubed_sphere as CS
from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import EULER_ROE, Workload, c1, c2

pytestmark = pytest.mark.gpu
GAM = 1.4


def amr_euler(steps=8, m=8):
    r = np.random.default_rng(1308147 + 31)
    fr = F.forest_refined(F.brick(2, 1, periodic_x=True, periodic_y=True), 1,
                          lambda t, x, y, h: r.random(len(x)) < 0.5)
    X, Y = F.cell_centres(fr, m)
    X = X + fr.tree_ids[:, None, None]
    rho = 1.0 + 0.5 * np.exp(-20 * ((X - 1.0) ** 2 + (Y - 0.5) ** 2))
    u, v, p = 0.3 + 0 * X, -0.2 + 0 * X, 1.0 + 0.3 * np.sin(2 * np.pi * X)
    q0 = np.stack([rho, rho * u, rho * v, p / (GAM - 1) + 0.5 * rho * (u * u + v * v)], 1)
    return Workload("amr_euler" + ("" if m == 8 else f"_m{m}"), fr, m, 4, 0, EULER_ROE, (GAM, 1.0), q0, None, steps,
                    1e-3, "cfl")


def three_levels(steps=6):
    """C2 physics on a three-level forest (levels 2, 3, 4): refine at base 2 near the centre, then
    once more inside the refined region (2:1 balanced by construction: nested squares)."""
    f = F.forest_refined(F.periodic_unit_square(), 2, lambda t, x, y, h: (abs(x - 0.5) < 0.3) & (abs(y - 0.5) < 0.3))
    # second refinement: split level-3 leaves whose centre is within 0.15 of the centre
    lv, tr, ix, iy = [], [], [], []
    for p in range(f.num_patches):
        l, x, y = int(f.levels[p]), int(f.ix[p]), int(f.iy[p])
        h = 0.5 ** l
        if l == 3 and abs((x + 0.5) * h - 0.5) < 0.15 and abs((y + 0.5) * h - 0.5) < 0.15:
            for k in range(4):
                lv.append(4); tr.append(0); ix.append(2 * x + (k & 1)); iy.append(2 * y + (k >> 1))
        else:
            lv.append(l); tr.append(0); ix.append(x); iy.append(y)
    fr = F.Forest(levels=np.array(lv, np.int8), tree_ids=np.array(tr, np.int32), ix=np.array(ix), iy=np.array(iy),
                  conn=f.conn)
    m = 8
    X, Y = F.cell_centres(fr, m)
    q0 = np.exp(-100.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))[:, None]
    dt = 0.9 * (0.5 ** 4 / m) / 1.0
    from workloads.configs import ADV_CONST
    return Workload("three_levels", fr, m, 1, 0, ADV_CONST, (1.0, 0.5), q0, None, steps, dt, "fixed")


def sphere(steps=6):
    return CS.c4_workload(base_level=2, m=8, steps=steps)


CASES = [c2(steps=15), c2(base_level=2, m=32, steps=8), amr_euler(), sphere(), three_levels(),
         amr_euler(steps=6, m=16)]   # (m = 16: the warp-sweep kernel with computed ghosts per level)


def mass(w, q):
    h = np.ldexp(1.0, -w.forest.levels.astype(np.int64))[:, None, None] / w.m
    kap = w.aux[:, 0, 2:w.m + 2, 2:w.m + 2] if w.aux is not None else 1.0
    return np.array([(q[:, k] * kap * h * h).sum() for k in range(w.meqn)])


@pytest.mark.parametrize("reflux", [0, 1], ids=["plain", "reflux"])
@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name)
def test_subcycled_parity_against_oracle(w, skip, reflux):
    w = dataclasses.replace(w, reflux=reflux)
    qo, co, do = oracle.run_subcycled(w)
    qg, cg, _ = fc.run_subcycled(w, dt_list=do, skip_quiescent=skip)
    for k in range(w.meqn):
        scale = np.abs(qo[:, k]).max() or np.abs(qo).max()
        assert np.abs(qg[:, k] - qo[:, k]).max() <= 1e-12 * scale, (w.name, k)
    np.testing.assert_allclose(cg, co, rtol=1e-12, atol=0)
    mo, mg, m0 = mass(w, qo), mass(w, qg), mass(w, w.q0)
    for k in range(w.meqn):
        assert abs(mg[k] - mo[k]) <= 1e-13 * max(abs(mo[k]), abs(m0[k])), (w.name, k)


@pytest.mark.parametrize("w", [CASES[0], CASES[2], CASES[4]], ids=lambda w: w.name)
def test_subcycled_reflux_conserves_on_gpu(w):
    w = dataclasses.replace(w, reflux=1)
    q, _, _ = fc.run_subcycled(w)
    m0, m1 = mass(w, w.q0), mass(w, q)
    for k in range(w.meqn):
        assert abs(m1[k] - m0[k]) <= 1e-14 * w.steps * 4 * max(abs(m0[k]), 1e-300) + 1e-15, (w.name, k)


def test_one_level_subcycling_is_fc_step():
    w = c1(steps=6)
    qa, ca, _ = fc.run(w)
    qb, cb, _ = fc.run_subcycled(w)
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


@pytest.mark.parametrize("w", [CASES[1], CASES[3], CASES[4]], ids=lambda w: w.name)
def test_per_level_fills_bitwise_equal_whole_forest_fills(w, monkeypatch):
    """The restricted per-level ghost fills and snapshots (the default on one rank) produce the
    same state bitwise as whole-forest passes (FC_SUB_FULL_FILL=1, read when a handle first
    sub-cycles): the records kept for the cells level l reads are the full fill's, in order."""
    w = dataclasses.replace(w, reflux=1)
    qa, ca, _ = fc.run_subcycled(w)
    monkeypatch.setenv("FC_SUB_FULL_FILL", "1")
    qb, cb, _ = fc.run_subcycled(w)
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)
