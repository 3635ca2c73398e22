"""GPU parity of the octree path (include/fc3.h, csrc/step3.cu) against the oracle (forest3.c):
the ghost rings, the states and the CFLs are bitwise equal (the same operations in the same order,
compiled without contraction), on uniform and two-level forests, periodic / outflow / mixed
bricks, MC / minmod / first order; a step above cfl_reject is not committed."""
import numpy as np
import pytest

from oracle import octree as O
from paper_1308_1472_b200 import fc, fc3
from workloads.octree import cell_centres, forest3

pytestmark = pytest.mark.gpu

CASES = [
    ("uniform_periodic", forest3((2, 1, 1), 1), 4),
    ("uniform_outflow", forest3((1, 2, 2), 1, periodic=(False, False, False)), 6),
    ("amr_periodic", forest3((2, 2, 1), 1, refine=lambda t, x, y, z, h: t == 0 and x < 0.5 and (y + z) < 0.9), 4),
    ("amr_mixed", forest3((2, 1, 2), 1, refine=lambda t, x, y, z, h: (t + x + y + z) < 1.2,
                          periodic=(True, False, True)), 8),
    ("amr_deep", forest3((1, 1, 1), 2, refine=lambda t, x, y, z, h: x + y < 0.6, periodic=(False, True, False)), 4),
    # m = 16 / 8 (the compiled-m kernels): regular patches (computed gather) and, in the second,
    # outflow patches (table gather) in one forest
    ("uniform_periodic_m16", forest3((1, 1, 1), 1), 16),
    ("uniform_mixed_m8", forest3((2, 1, 1), 2, periodic=(False, True, True)), 8),
]


def bump(f, m):
    c = cell_centres(f, m)
    return np.exp(-8.0 * ((c[:, 0] - 0.6) ** 2 + (c[:, 1] - 0.5) ** 2 + (c[:, 2] - 0.45) ** 2))


@pytest.mark.parametrize("name,f,m", CASES, ids=[c[0] for c in CASES])
def test_ghost_rings_bitwise(name, f, m, rng):
    q = rng.standard_normal((f.num_patches, m, m, m))
    g = fc3.Forest3(f, m)
    g.set_problem((0.5, 0.5, 0.5))
    g.set_q(q)
    g.ghost_fill()
    o = O.OracleForest3(f, m)
    np.testing.assert_array_equal(g.get_q_padded(), o.ghost_fill(o.pad(q)))
    g.close()


@pytest.mark.parametrize("lim,m2", [(fc.FC_LIM_MC, 2), (fc.FC_LIM_MINMOD, 2), (fc.FC_LIM_NONE, 1)],
                         ids=["mc", "minmod", "first_order"])
@pytest.mark.parametrize("name,f,m", CASES, ids=[c[0] for c in CASES])
def test_steps_bitwise(name, f, m, lim, m2):
    q0 = bump(f, m)
    vel = (0.8, -0.45, 0.3)
    lmax = int(f.levels.max())
    dt = 0.9 / (m * 2 ** lmax) / 0.8
    qg, cg = fc3.run3(f, m, q0, vel, dt, 12, limiter=lim, method2=m2)
    qo, co = O.run3(f, m, q0, vel, dt, 12, limiter=lim, method2=m2)
    np.testing.assert_array_equal(qg, qo)
    np.testing.assert_array_equal(cg, co)


def test_courant_one_shift_and_reject():
    m = 4
    f = forest3((2, 2, 1), 1)
    rng = np.random.default_rng(1308147 + 90)
    q0 = rng.integers(0, 256, (f.num_patches, m, m, m)).astype(float)
    dx = 1.0 / (2 * m)
    qg, cg = fc3.run3(f, m, q0, (1.0, 1.0, 1.0), dx, 3)
    qo, co = O.run3(f, m, q0, (1.0, 1.0, 1.0), dx, 3)
    np.testing.assert_array_equal(qg, qo)
    assert (cg == 1.0).all()
    g = fc3.Forest3(f, m)
    g.set_problem((1.0, 1.0, 1.0))
    g.set_q(q0)
    rc, c = g.step(1.5 * dx, raise_on_reject=False)
    assert rc == fc.FC_ECFL and c == 1.5
    np.testing.assert_array_equal(g.get_q(), q0)
    g.close()


@pytest.mark.parametrize("lim", [fc.FC_LIM_MC, fc.FC_LIM_MINMOD], ids=["mc", "minmod"])
@pytest.mark.parametrize("name,f,m", [c for c in CASES if c[2] in (8, 16)], ids=[c[0] for c in CASES if c[2] in (8, 16)])
def test_steps_bitwise_wide_range(name, f, m, lim):
    """Limiter ratios across the whole double range (quotients that overflow, underflow to
    subnormals, zero numerators and zero waves, exactly equal neighbours): the compiled-m pencils'
    grouped division (nvcc's fast path, the operator where its range check fails) gives the
    oracle's IEEE quotient bit for bit."""
    rng = np.random.default_rng(1308147 + 91)
    n = f.num_patches * m ** 3
    q0 = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-160, 160, n)
    q0[rng.random(n) < 0.15] = 0.0
    rep = rng.random(n) < 0.15
    q0[1:][rep[1:]] = q0[:-1][rep[1:]]
    q0 = q0.reshape(f.num_patches, m, m, m)
    vel = (0.8, -0.45, 0.3)
    dt = 0.9 / (m * 2 ** int(f.levels.max())) / 0.8
    qg, cg = fc3.run3(f, m, q0, vel, dt, 3, limiter=lim, method2=2)
    qo, co = O.run3(f, m, q0, vel, dt, 3, limiter=lim, method2=2)
    np.testing.assert_array_equal(qg.view(np.int64), qo.view(np.int64))
    np.testing.assert_array_equal(cg, co)


def test_regular_rings_equal_the_table_gather(monkeypatch):
    """Patches whose ring is all aligned same-level copies compute their sources from their 27
    neighbours (csrc/step3.cu, `nb27` / `ring_reg`); FC3_REGULAR=0 (read when the forest is
    created) keeps the per-patch table for every patch: the same copies, so the same bits."""
    name, f, m = CASES[-1]
    q0 = bump(f, m)
    vel = (0.8, -0.45, 0.3)
    dt = 0.9 / (m * 2 ** int(f.levels.max())) / 0.8
    qa, ca = fc3.run3(f, m, q0, vel, dt, 6)
    monkeypatch.setenv("FC3_REGULAR", "0")
    qb, cb = fc3.run3(f, m, q0, vel, dt, 6)
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)
