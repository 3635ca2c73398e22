"""Pins for the oracle's sub-cycled stepping (oracle/subcycle.c; PAPER.md:201-202 [§3], 277-290
[§4]).

Independent references: (1) on a single-level forest sub-cycling is the global-dt step, bitwise;
(2) affine data under constant-velocity advection is translated exactly by the method (a pin of
the update, tests/test_oracle_step.py), by the averaging and the minmod interpolation, and is
linear in time -- so a sub-cycled AMR step, whose fine ghosts at the second sub-step come from the
*time-interpolated* coarse data, must still translate it exactly away from the outflow boundary (a
wrong interpolation weight or a stale coarse time shows up as an O(b u dt) error); (3) with the
reflux, sum q area is conserved exactly on the periodic AMR square, with the coarse flux x dt_c
balanced against the fine fluxes x dt_f of both sub-steps; (4) constant states stay exact;
(5) the sub-cycled solution approaches the global-dt one (both converge to the PDE solution).
"""
import dataclasses

import numpy as np

import oracle
from workloads import forests as F
from workloads.configs import ADV_CONST, Workload, c1, c2, c5


def area(w):
    return np.ldexp(1.0, -2 * w.forest.levels.astype(np.int64))[:, None, None] / (w.m * w.m)


def test_single_level_subcycling_is_the_global_step():
    for w in (c1(steps=5), c5(level=2, m=8, steps=5)):
        q1, c1_, _ = oracle.run(w)
        q2, c2_, _ = oracle.run_subcycled(w)
        np.testing.assert_array_equal(q1, q2)
        np.testing.assert_array_equal(c1_, c2_)


def test_affine_data_translated_exactly_across_subcycled_levels(rng):
    """Two-tree outflow brick, level 2 with a level-3 block in the middle (interior coarse/fine
    faces); affine q = a + b x + c y, constant (u, v); one sub-cycled step (1 coarse + 2 fine
    updates): every cell farther than 6 coarse cells from the outer boundary equals
    a + b (x - u dt) + c (y - v dt)."""
    fr = F.forest_refined(F.brick(2, 1, bc=F.OUTFLOW), 2,
                          lambda t, x, y, h: (np.abs(x + t - 1.0) < 0.3) & (np.abs(y - 0.5) < 0.3))
    assert len(set(fr.levels.tolist())) == 2
    m = 8
    X, Y = F.cell_centres(fr, m)
    X = X + fr.tree_ids[:, None, None]
    h = np.ldexp(1.0, -fr.levels.astype(np.int64))[:, None, None] / m
    for _ in range(4):
        u, v = rng.uniform(-1, 1, 2)
        a, b, c = rng.normal(size=3)
        q0 = (a + b * X + c * Y)[:, None]
        dtc = 0.8 * (0.25 / m) / max(abs(u), abs(v))      # coarse (level 2) Courant 0.8
        w = Workload("affine", fr, m, 1, 0, ADV_CONST, (u, v), q0, None, 1, dtc, "fixed")
        q, cfl, _ = oracle.run_subcycled(w, dt_list=[dtc])
        exact = a + b * (X - u * dtc) + c * (Y - v * dtc)
        far = (X > 6 * 0.25 / m) & (X < 2 - 6 * 0.25 / m) & (Y > 6 * 0.25 / m) & (Y < 1 - 6 * 0.25 / m)
        err = np.abs(q[:, 0] - exact)[far].max()
        assert err <= 1e-13 * max(1.0, np.abs(exact).max()), err
        assert 0.75 < cfl < 0.85


def test_subcycled_reflux_conserves_mass_exactly():
    w = dataclasses.replace(c2(steps=15), reflux=1)
    A = area(w)
    m0 = (w.q0[:, 0] * A).sum()
    q, cfl, dts = oracle.run_subcycled(w)
    assert abs((q[:, 0] * A).sum() - m0) <= 1e-14 * 15 * m0
    qn, _, _ = oracle.run_subcycled(dataclasses.replace(w, reflux=0))
    assert abs((qn[:, 0] * A).sum() - m0) > 1e-9 * m0
    assert np.allclose(dts, 2 * c2().dt0)          # the coarse level steps at twice the global dt


def test_subcycled_constant_state_exact():
    w = c2(steps=5)
    w = dataclasses.replace(w, q0=np.full_like(w.q0, 0.37), reflux=1)
    q, _, _ = oracle.run_subcycled(w)
    assert (q == 0.37).all()


def test_subcycled_close_to_global_dt():
    """Same final time: 20 global steps of dt vs 10 sub-cycled steps of 2 dt on C2; the two
    second-order solutions differ by far less than the solution scale."""
    w = c2(steps=20)
    qg, _, _ = oracle.run(w)
    qs, _, _ = oracle.run_subcycled(w, steps=10)
    assert np.abs(qg - qs).max() < 0.02 * np.abs(qg).max()
