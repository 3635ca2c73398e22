"""GPU parity of the dynamic regrid (fc_regrid)
against the oracle's orc_regrid: the new leaf list bit-exact, the transferred state bitwise (the
interpolation and the averaging are exact-order on both sides), on single- and multi-tree forests
(periodic square, outflow brick, cubed sphere); and a dynamic-AMR run -- cycles of steps and
regrids -- equal to the oracle's within the step tolerance."""
import dataclasses

import numpy as np
import pytest

import oracle
import workloads.cubed_sphere as CS
from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import c1, c2, c5

pytestmark = pytest.mark.gpu


def oracle_regrid(w, q, rt, ct, minl, maxl):
    of = oracle.forest_for(w)
    qp = of.ghost_fill(of.pad(q))
    return of.regrid(qp, rt, ct, minl, maxl)


def gpu_regrid(w, q, rt, ct, minl, maxl):
    f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0, 0)
    f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject)
    if w.aux is not None:
        f.set_aux(np.ascontiguousarray(w.aux))
    f.set_q(np.ascontiguousarray(q))
    g = f.regrid(rt, ct, minl, maxl)
    lv, tr = g.leaves()
    return lv, tr, g.get_q(), g


def spiky(w, rng):
    q = w.q0.copy()
    q[rng.integers(0, w.num_patches, 3), :, 2, 5] += 1.0
    return q


CASES = [(c2(steps=1), (0.4, 0.01, 2, 5)), (c2(steps=1), (0.05, 0.02, 1, 6)),
         (c1(level=3, m=8), (0.3, 0.05, 2, 4)), (c5(level=3, m=8, steps=1), (0.5, 0.05, 2, 4)),
         (CS.c4_workload(base_level=2, m=8, steps=1), (0.2, 0.02, 1, 3))]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].name}_{c[1][0]}_{c[1][1]}")
def test_regrid_matches_oracle_bitwise(case, rng):
    w, prm = case
    for q in (w.q0, spiky(w, rng)):
        lo, to, qo, so = oracle_regrid(w, q, *prm)
        lg, tg, qg, g = gpu_regrid(w, q, *prm)
        np.testing.assert_array_equal(lg, lo)
        np.testing.assert_array_equal(tg, to)
        np.testing.assert_array_equal(qg, qo)
        g.close()


def test_dynamic_amr_run_matches_oracle():
    """C2 physics with the reflux, 4 cycles of (10 steps, regrid): the bump moves and the mesh
    follows it; the GPU (fc_step + fc_regrid on the new handles) and the oracle end on the same
    mesh and state, and sum q area is conserved through steps and regrids.  Levels 2..4 keep the
    fixed dt (0.9 dx_4) within CFL 1."""
    w = dataclasses.replace(c2(steps=10), reflux=1)
    prm = (0.1, 0.02, 2, 4)
    # oracle
    wo, qo = w, w.q0
    meshes_o = []
    for cycle in range(4):
        wo = dataclasses.replace(wo, q0=qo)
        qo, co, do = oracle.run(wo)
        lv, tr, qo, _ = oracle_regrid(wo, qo, *prm)
        fr = F.Forest(lv, tr, np.zeros(len(lv), np.int64), np.zeros(len(lv), np.int64), w.forest.conn)
        wo = dataclasses.replace(wo, forest=fr)
        meshes_o.append(len(lv))
    # GPU, replaying the oracle's dt list per cycle (fixed dt policy: identical)
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    meshes_g = []
    for cycle in range(4):
        for _ in range(w.steps):
            f.step(w.dt0)
        g = f.regrid(*prm)
        f.close()
        f = g
        meshes_g.append(f.count)
    assert meshes_g == meshes_o and len(set(meshes_o)) > 1         # the mesh changed along the way
    lv, tr = f.leaves()
    np.testing.assert_array_equal(lv, wo.forest.levels)
    qg = f.get_q()
    scale = np.abs(qo).max()
    assert np.abs(qg - qo).max() <= 1e-12 * scale
    A = np.ldexp(1.0, -2 * lv.astype(np.int64))[:, None, None]
    A0 = np.ldexp(1.0, -2 * w.forest.levels.astype(np.int64))[:, None, None]
    m0 = (w.q0[:, 0] * A0).sum()
    assert abs((qg[:, 0] * A).sum() - m0) <= 1e-13 * m0
