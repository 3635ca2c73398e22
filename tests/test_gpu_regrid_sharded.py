"""Multi-rank dynamic regrid ("Morton repartition + NCCL migration"; fc_regrid on
NCCL handles, the fc_regrid_* stages with the manual transport): R rank handles in one process on
one GPU, halo and migration buffers moved with device copies.  The new mesh, its partition and the
migrated + transferred state equal the one-rank regrid bitwise, and a dynamic run (cycles of steps
and regrids on the shards) equals the one-rank run bitwise."""
import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads.configs import c1, c2

from test_gpu_sharded import d2d

pytestmark = pytest.mark.gpu


def make_shards(levels, trees, conn, w, R):
    hs = []
    for r in range(R):
        f = fc.Forest(levels, trees, conn, w.m, w.meqn, w.maux, 1.0, 0, r, R, None)
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject, 1)
        hs.append(f)
    wire(hs)
    return hs


def wire(hs):
    R = len(hs)
    for rnd in (1, 2):
        for r in range(R):
            for s in range(R):
                if s != r:
                    hs[s].halo_set_requests(rnd, r, hs[r].halo_requests(s, rnd))
    for f in hs:
        f.halo_finalize()


def move(bufs, R):
    for r in range(R):
        _, recv, _, roff = bufs[r]
        for s in range(R):
            if s == r:
                continue
            send, _, soff, _ = bufs[s]
            n = roff[s + 1] - roff[s]
            assert n == soff[r + 1] - soff[r]
            d2d(recv + 8 * roff[s], send + 8 * soff[r], 8 * n)


def halo(hs, rnd):
    for f in hs:
        f.halo_pack(rnd)
    move([f.halo_buffers(rnd) for f in hs], len(hs))
    for f in hs:
        f.halo_unpack(rnd)


def step(hs, dt):
    halo(hs, 1)
    for f in hs:
        f.step_local(dt, 1)
    halo(hs, 2)
    c = max(f.step_local(dt, 2) for f in hs)
    for f in hs:
        assert f.commit(c) == fc.FC_OK
    return c


def regrid(hs, prm, weights=0):
    R = len(hs)
    halo(hs, 1)
    for f in hs:
        f.regrid_fill(1)
    halo(hs, 2)
    for f in hs:
        f.regrid_fill(2)
    tags = np.concatenate([f.regrid_tags() for f in hs])
    gs = [f.regrid_begin(tags, *prm, level_weights=weights) for f in hs]
    move([hs[r].regrid_buffers(gs[r]) for r in range(R)], R)
    for g in gs:
        g.regrid_finish()
    wire(gs)
    for f in hs:
        f.close()
    return gs


CASES = [(c2(steps=1), (0.4, 0.01, 2, 5)), (c2(steps=1), (0.05, 0.02, 1, 6)), (c1(level=3, m=8), (0.3, 0.05, 2, 4))]


@pytest.mark.parametrize("R", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].name}_{c[1][0]}")
def test_sharded_regrid_equals_one_rank_bitwise(case, R):
    w, prm = case
    one = fc.forest_for(w, 0)
    one.set_q(np.ascontiguousarray(w.q0))
    g1 = one.regrid(*prm)
    lv1, tr1 = g1.leaves()
    q1 = g1.get_q()
    hs = make_shards(w.forest.levels, w.forest.tree_ids, w.forest.conn, w, R)
    for f in hs:
        f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    gs = regrid(hs, prm)
    lv, tr = gs[0].leaves()
    np.testing.assert_array_equal(lv, lv1)
    np.testing.assert_array_equal(tr, tr1)
    assert [g.first for g in gs] == [r * len(lv) // R for r in range(R)]
    np.testing.assert_array_equal(np.concatenate([g.get_q() for g in gs if g.count]), q1)
    for g in gs:
        g.close()
    g1.close()
    one.close()


@pytest.mark.parametrize("R", [2, 3])
def test_sharded_dynamic_amr_run_equals_one_rank(R):
    """C2 physics, 3 cycles of (6 steps, regrid): the mesh changes, the partition follows it, and
    every rank's state after the last cycle is the one-rank run's, bitwise."""
    w = c2(steps=6)
    prm = (0.1, 0.02, 2, 4)
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    hs = make_shards(w.forest.levels, w.forest.tree_ids, w.forest.conn, w, R)
    for h in hs:
        h.set_q(np.ascontiguousarray(w.q0[h.first:h.first + h.count]))
    sizes = []
    for cycle in range(3):
        for _ in range(w.steps):
            c1_ = f.step(w.dt0)[1]
            c = step(hs, w.dt0)
            assert c == c1_
        g = f.regrid(*prm)
        f.close()
        f = g
        hs = regrid(hs, prm)
        sizes.append(f.count)
    assert len(set(sizes)) > 1 or sizes[0] != w.num_patches
    np.testing.assert_array_equal(np.concatenate([h.get_q() for h in hs if h.count]), f.get_q())
    for h in hs:
        h.close()
    f.close()


def test_sharded_regrid_level_weights():
    """level_weights = 1: the new Morton cuts balance sum 2^(level - coarsest) (a sub-cycled step's
    work) instead of the count; every rank's weight is within one patch of the ideal share, and the
    state is the one-rank regrid's, bitwise."""
    w, prm = c2(steps=1), (0.4, 0.01, 2, 5)
    R = 3
    one = fc.forest_for(w, 0)
    one.set_q(np.ascontiguousarray(w.q0))
    g1 = one.regrid(*prm)
    lv, _ = g1.leaves()
    hs = make_shards(w.forest.levels, w.forest.tree_ids, w.forest.conn, w, R)
    for f in hs:
        f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    gs = regrid(hs, prm, weights=1)
    wt = np.ldexp(1.0, lv.astype(np.int64) - int(lv.min()))
    shares = [wt[g.first:g.first + g.count].sum() for g in gs]
    assert abs(sum(shares) - wt.sum()) == 0 and max(shares) - min(shares) <= 2 * wt.max()
    assert [g.first for g in gs] != [r * len(lv) // R for r in range(R)]    # not the count cut
    np.testing.assert_array_equal(np.concatenate([g.get_q() for g in gs if g.count]), g1.get_q())
