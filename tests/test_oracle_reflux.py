"""Pins for the oracle's coarse/fine flux correction (oracle/forest.c orc_reflux, claw.c face
fluxes, PAPER.md:279-282 [§4] "conservative ... correction").

What fixes the reflux independently of its own code: discrete conservation.  Without it the
global-dt step loses sum kappa q across coarse/fine faces (the defect is
1/4 u dt dy s_x per face cell); with it the coarse cells' applied fluxes are replaced by the fine
ones, so the total must be invariant to roundoff -- on a periodic AMR square (scalar advection and
Euler, all four components), and on the cubed sphere across rotated / reversed tree links
(capacity form) for a bump that cannot reach the three-tree corners.  A dropped term, a wrong sign,
a mis-paired fine edge or a wrong orientation across a tree face breaks that.  On meshes without
coarse/fine faces the correction must be an exact no-op, and constant states must stay exact
(on the sphere: to the rounding of the stream-function edge velocities).
"""
import dataclasses
import math

import numpy as np
import pytest

import oracle
import workloads.cubed_sphere as CS
from workloads import forests as F
from workloads.configs import ADV_CONST, EULER_ROE, Workload, c1, c2, c5

GAM = 1.4


def area(w):
    return np.ldexp(1.0, -2 * w.forest.levels.astype(np.int64))[:, None, None] / (w.m * w.m)


def sphere_area(w):
    h = np.ldexp(1.0, -w.forest.levels.astype(np.int64))[:, None, None] / w.m
    return w.aux[:, 0, 2:w.m + 2, 2:w.m + 2] * h * h


def with_reflux(w, on=1, **kw):
    return dataclasses.replace(w, reflux=on, **kw)


def test_c2_mass_exact_with_reflux_and_not_without():
    w = c2(steps=30)
    A = area(w)
    m0 = (w.q0[:, 0] * A).sum()
    q1, _, _ = oracle.run(with_reflux(w))
    q0, _, _ = oracle.run(w)
    assert abs((q1[:, 0] * A).sum() - m0) <= 1e-14 * 30 * m0
    assert abs((q0[:, 0] * A).sum() - m0) > 1e-8 * m0      # the defect the reflux removes


def test_periodic_amr_euler_conserves_all_components(rng):
    """Euler on a periodic 2-tree brick refined at random (2:1 balanced by construction of the
    generator): every conserved component's total is invariant with the reflux."""
    r = np.random.default_rng(1308147 + 31)
    fr = F.forest_refined(F.brick(2, 1, periodic_x=True, periodic_y=True), 1,
                          lambda t, x, y, h: r.random(len(x)) < 0.5)
    m = 8
    X, Y = F.cell_centres(fr, m)
    X = X + fr.tree_ids[:, None, None]
    rho = 1.0 + 0.5 * np.exp(-20 * ((X - 1.0) ** 2 + (Y - 0.5) ** 2))
    u, v, p = 0.3 + 0 * X, -0.2 + 0 * X, 1.0 + 0.3 * np.sin(2 * np.pi * X)
    q0 = np.stack([rho, rho * u, rho * v, p / (GAM - 1) + 0.5 * rho * (u * u + v * v)], 1)
    w = Workload("amr_euler", fr, m, 4, 0, EULER_ROE, (GAM, 1.0), q0, None, 15, 1e-3, "cfl", reflux=1)
    assert len(set(fr.levels.tolist())) == 2
    A = area(w)
    q, _, _ = oracle.run(w)
    for k in range(4):
        tot0 = (q0[:, k] * A).sum()
        scale = (np.abs(q0[:, k]) * A).sum()
        assert abs((q[:, k] * A).sum() - tot0) <= 1e-14 * 15 * scale, k


def test_sphere_mass_exact_across_tree_faces():
    """C4 physics (capacity form, edge velocities) on the L3/L4 band mesh: a bump centred on the
    bells' latitude crosses coarse/fine faces, many of them on cube edges with rotated frames, but
    cannot reach the cube vertices in 12 steps: sum kappa q is exact with the reflux only."""
    w = CS.c4_workload(base_level=3, m=8, steps=12)
    X = w.info["centres"]
    c = np.array([math.cos(5 * math.pi / 6), math.sin(5 * math.pi / 6), 0.0])
    d = np.arccos(np.clip(X @ c, -1, 1))
    w.q0 = (0.1 + np.where(d < 0.5, 0.5 * (1 + np.cos(math.pi * d / 0.5)), 0.0))[:, None]
    A = sphere_area(w)
    m0 = (w.q0[:, 0] * A).sum()
    q1, _, _ = oracle.run(with_reflux(w))
    q0, _, _ = oracle.run(w)
    assert abs((q1[:, 0] * A).sum() - m0) <= 1e-14 * 12 * m0
    assert abs((q0[:, 0] * A).sum() - m0) > 1e-10 * m0
    # the c/f faces of this mesh do cross tree boundaries (AVG4 ghosts sourced from another tree)
    tab = oracle.forest_for(w).ghost_table()
    src_tree = w.forest.tree_ids[tab[:, :, 1]]
    own_tree = w.forest.tree_ids[:, None]
    assert ((tab[:, :, 0] == oracle.OP_AVG4) & (src_tree != own_tree)).any()


@pytest.mark.parametrize("w", [c1(), c5(level=2, m=8, steps=10)], ids=lambda w: w.name)
def test_reflux_is_a_noop_without_coarse_fine_faces(w):
    qa, ca, _ = oracle.run(w)
    qb, cb, _ = oracle.run(with_reflux(w))
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


def test_constant_state_exact_with_reflux():
    w = c2(steps=10)
    w = dataclasses.replace(w, q0=np.full_like(w.q0, 0.37))
    q, _, _ = oracle.run(with_reflux(w))
    assert (q == 0.37).all()
    # capacity form: the advective update keeps constants bitwise, the reflux adds
    # q (u_C - (u_f1 + u_f2) / 2), which the stream-function edge velocities make zero only up to
    # the rounding of their psi differences
    s = CS.c4_workload(base_level=2, m=8, steps=5)
    s.q0[:] = 0.37
    q, _, _ = oracle.run(with_reflux(s))
    np.testing.assert_allclose(q, 0.37, rtol=1e-14, atol=0)


def test_face_flux_records_match_the_physical_flux_for_uniform_flow():
    """For a uniform state every fluctuation and correction vanishes, so each recorded face flux
    is the outward physical flux: +-u q on x faces, +-v q on y faces (ADV_CONST), and the Euler
    flux vector for Euler."""
    m = 8
    qp = np.full((1, m + 4, m + 4), 0.7)
    fl = np.zeros((4, m, 1))
    pr = oracle.problem(ADV_CONST, (1.0, -0.5))
    L = oracle.lib()
    qn = np.zeros_like(qp)
    L.orc_step_patch_faces(oracle.C.byref(pr), m, 1, oracle._p(qp), None, 0.01, 0.1, 0.1, oracle._p(qn),
                           oracle._p(fl))
    np.testing.assert_array_equal(fl[0, :, 0], -1.0 * 0.7 * np.ones(m))
    np.testing.assert_array_equal(fl[1, :, 0], 1.0 * 0.7 * np.ones(m))
    np.testing.assert_array_equal(fl[2, :, 0], 0.5 * 0.7 * np.ones(m))
    np.testing.assert_array_equal(fl[3, :, 0], -0.5 * 0.7 * np.ones(m))
    rho, u, v, p = 1.3, 0.4, -0.2, 2.0
    E = p / (GAM - 1) + 0.5 * rho * (u * u + v * v)
    st = np.array([rho, rho * u, rho * v, E])
    qp = np.ascontiguousarray(np.broadcast_to(st[:, None, None], (4, m + 4, m + 4)))
    fl = np.zeros((4, m, 4))
    pr = oracle.problem(EULER_ROE, (GAM, 1.0))
    qn = np.zeros_like(qp)
    L.orc_step_patch_faces(oracle.C.byref(pr), m, 4, oracle._p(qp), None, 0.001, 0.1, 0.1, oracle._p(qn),
                           oracle._p(fl))
    fx = np.array([rho * u, rho * u * u + p, rho * u * v, (E + p) * u])
    fy = np.array([rho * v, rho * u * v, rho * v * v + p, (E + p) * v])
    np.testing.assert_allclose(fl[1], np.broadcast_to(fx, (m, 4)), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(fl[0], -np.broadcast_to(fx, (m, 4)), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(fl[3], np.broadcast_to(fy, (m, 4)), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(fl[2], -np.broadcast_to(fy, (m, 4)), rtol=1e-15, atol=1e-15)
