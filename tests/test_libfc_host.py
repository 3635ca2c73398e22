"""CPU tests of libfc.so without a GPU: it loads, exports every symbol include/fc.h declares, and
its host planner (per-direction neighbour lookup + composed tree transforms) produces ghost
tables bit-identical to the oracle's brute-force point-location tables; invalid forests are
rejected with the same error classes; the sharded halo plan is consistent across ranks."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import c1, c2, c3, c5

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fc.h")).read()
    declared = sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fc_\w+)\s*\(", hdr, re.M)))
    assert declared == sorted(fc.EXPORTS)
    L = fc.lib()
    for name in declared:
        assert hasattr(L, name), name


def host_table(levels, tree_ids, conn, m, meqn=1, rank=0, nranks=1):
    f = fc.Forest(levels, tree_ids, conn, m, meqn, device=-1, rank=rank, nranks=nranks)
    return f, f.ghost_table()


def oracle_table(levels, tree_ids, conn, m):
    return oracle.OracleForest(levels, tree_ids, conn, m).ghost_table()


from workloads.cubed_sphere import c4_workload


@pytest.mark.parametrize("w", [c1(), c1(level=3, m=4), c2(), c3(level=2, m=8), c3(level=1, m=32),
                               c5(level=2, m=8), c5(level=1, m=16), c4_workload(),
                               c4_workload(base_level=2, m=8, uniform=True)], ids=lambda w: w.name)
def test_table_bit_exact_configs(w):
    _, t = host_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    o = oracle_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    np.testing.assert_array_equal(t, o)


def _random_forest(rng, conn, base, m):
    def refine(t, x, y, h):
        return rng.random(len(x)) < 0.35
    return F.forest_refined(conn, base, refine)


CONNS = {
    "periodic": F.periodic_unit_square(),
    "walls": F.walled_unit_square(F.WALL),
    "outflow": F.walled_unit_square(F.OUTFLOW),
    "brick3x2": F.brick(3, 2, bc=F.WALL),
    "brick2x2_periodic": F.brick(2, 2, periodic_x=True, periodic_y=True),
    "reversed": F.brick(2, 1, bc=F.OUTFLOW, reversed_x_links=(0,)),
}


@pytest.mark.parametrize("name", sorted(CONNS))
def test_table_bit_exact_random_two_level_forests(rng, name):
    conn = CONNS[name]
    for trial in range(4):
        m = [4, 8, 6, 16][trial]
        fr = _random_forest(rng, conn, 2, m)
        _, t = host_table(fr.levels, fr.tree_ids, conn, m)
        o = oracle_table(fr.levels, fr.tree_ids, conn, m)
        np.testing.assert_array_equal(t, o)


def test_rejects_invalid_forests_like_the_oracle():
    conn = F.periodic_unit_square()
    cases = [([2, 1, 1, 1, 2, 2, 2], [0] * 7, conn, fc.FC_ETILING),      # misaligned leaf
             ([1] * 3, [0] * 3, conn, fc.FC_ETILING),                     # incomplete tree
             ([0, 0], [1, 0], F.brick(2, 1), fc.FC_ETILING)]              # decreasing tree ids
    bad = F.brick(2, 1)
    bad.tree_to_face[1] = 3
    cases.append(([0, 0], [0, 1], bad, fc.FC_ECONN))
    # a level-0 neighbour of a level-2 leaf: one tree refined twice at a corner, the other not
    fr = F.forest_refined(F.brick(2, 1), 0, lambda t, x, y, h: np.array([t == 0]))
    lv = list(fr.levels)
    tr = list(fr.tree_ids)
    lv = [1, 2, 2, 2, 2] + lv[2:]      # tree 0's SE child (touching tree 1, level 0) at level 2
    tr = [0, 0, 0, 0, 0] + tr[2:]
    cases.append((lv, tr, F.brick(2, 1), fc.FC_EBALANCE))
    for levels, trees, cn, code in cases:
        with pytest.raises(fc.FcError) as ei:
            fc.Forest(np.array(levels), np.array(trees), cn, 8, 1, device=-1)
        assert ei.value.code == code, (levels, code, ei.value)
        with pytest.raises(ValueError):
            oracle.OracleForest(np.array(levels, np.int8), np.array(trees, np.int32), cn, 8).ghost_table()


def test_bad_descriptor_fields():
    w = c1()
    for kw in ({"m": 7}, {"m": 2}):
        with pytest.raises(fc.FcError) as ei:
            fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, kw["m"], 1, device=-1)
        assert ei.value.code == fc.FC_EINVAL


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_sharded_tables_and_halo_plan(nranks):
    """Every rank's table is the oracle's table restricted to its Morton range, and the remote
    cells a rank needs are exactly the sources in its table owned by other ranks."""
    for w in (c1(), c2(), c5(level=2, m=8)):
        o = oracle_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
        P = w.num_patches
        for r in range(nranks):
            f, t = host_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, rank=r, nranks=nranks)
            p0, p1 = (r * P) // nranks, ((r + 1) * P) // nranks
            assert (f.first, f.count) == (p0, p1 - p0)
            np.testing.assert_array_equal(t, o[p0:p1])
            srcs = set()
            for rec in t.reshape(-1, 8):
                op, q = rec[0], rec[1]
                if op in (1, 2, 3) and not (p0 <= q < p1):
                    srcs.add(q)
            counts = f.halo_counts()
            assert counts[r] == 0
            owners = {s * nranks // P for s in srcs}
            for s in range(nranks):
                lo, hi = (s * P) // nranks, ((s + 1) * P) // nranks
                has = any(lo <= q < hi for q in srcs)
                assert (counts[s] > 0) == has, (w.name, r, s)
            del owners


def test_more_ranks_than_patches():
    """Ranks past the patch count own empty Morton ranges (the Fig. 3 "idle processors" case)."""
    w = c1(level=1, m=8)          # 4 patches
    o = oracle_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    seen = 0
    for r in range(8):
        f, t = host_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, rank=r, nranks=8)
        assert f.count == ((r + 1) * 4) // 8 - (r * 4) // 8
        np.testing.assert_array_equal(t, o[f.first:f.first + f.count])
        seen += f.count
    assert seen == 4


def test_single_patch_forest_tables():
    """A one-leaf periodic tree: every ghost cell copies from the patch itself (wrap-around)."""
    w = c1(level=0, m=8)
    _, t = host_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    assert (t[..., 0] == 1).all() and (t[..., 1] == 0).all()
    np.testing.assert_array_equal(t, oracle_table(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m))


# ---- coarse/fine reflux planning -----------------------------------------------
def test_reflux_plan_single_rank_and_cross_rank_requests():
    """fc_set_problem(reflux = 1) plans the coarse/fine flux pairing on the host: on one rank for C2
    and the cubed sphere; with Morton shards that cut coarse/fine pairs each rank requests the fine
    faces it needs from their owners (fc_reflux_requests): every requested fine patch is owned by
    the peer asked, every face index is 0..3, no key repeats, and some pair of C2's three shards
    does need one; conforming forests request nothing."""
    from workloads.cubed_sphere import c4_workload
    for w in (c2(), c4_workload(base_level=2, m=8, steps=1)):
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, device=-1)
        f.set_problem(w.kind, w.params[0], w.params[1], reflux=1)
        assert len(f.reflux_requests(0)) == 0
    w = c2()
    R = 3
    hs = [fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, 1, device=-1, rank=r, nranks=R)
          for r in range(R)]
    total = 0
    for f in hs:
        f.set_problem(w.kind, w.params[0], w.params[1], reflux=1)
    for r, f in enumerate(hs):
        for s in range(R):
            keys = f.reflux_requests(s)
            if s == r:
                assert len(keys) == 0
                continue
            total += len(keys)
            assert len(set(keys.tolist())) == len(keys)
            q, face = keys // 4, keys % 4
            assert ((q >= hs[s].first) & (q < hs[s].first + hs[s].count)).all() and ((face >= 0) & (face < 4)).all()
    assert total > 0
    w = c5(level=2, m=8)
    for r in range(3):
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, 4, device=-1, rank=r, nranks=3)
        f.set_problem(w.kind, w.params[0], w.params[1], reflux=1)
        assert all(len(f.reflux_requests(s)) == 0 for s in range(3))


def test_custom_partition_ranges_and_validation():
    """fc_forest_desc.partition sets each rank's Morton range (empty ranks allowed); cut points
    that decrease or do not cover 0..P are rejected with FC_EINVAL."""
    w = c2()
    P = w.num_patches
    part = [0, 13, 13, 70, P]
    for r in range(4):
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, 1, device=-1, rank=r, nranks=4,
                      partition=part)
        assert (f.first, f.count) == (part[r], part[r + 1] - part[r])
    for bad in ([0, 20, 10, 70, P], [0, 13, 13, 70, P - 1], [1, 13, 13, 70, P]):
        with pytest.raises(fc.FcError) as e:
            fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, 1, device=-1, rank=0, nranks=4,
                      partition=bad)
        assert e.value.code == fc.FC_EINVAL


# ---- COMPACT table (FC_TABLE_COMPACT): the planner's per-direction lookup vs the oracle's read-back
# from its brute-force per-cell records (oracle/compact.py) -----------------------------------------
def compact_pair(levels, tree_ids, conn, m):
    from oracle.compact import compact_table
    f = fc.Forest(levels, tree_ids, conn, m, 1, device=-1)
    return f.ghost_table(fc.FC_TABLE_COMPACT), compact_table(oracle.OracleForest(levels, tree_ids, conn, m))


@pytest.mark.parametrize("w", [c1(), c2(), c3(level=2, m=8), c5(level=2, m=8), c4_workload(base_level=2, m=8),
                               c4_workload(base_level=2, m=8, uniform=True)], ids=lambda w: w.name)
def test_compact_table_bit_exact_configs(w):
    t, o = compact_pair(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    np.testing.assert_array_equal(t, o)
    kinds = set(np.unique(t[:, :, 0]).tolist())
    if w.name.startswith("C2") or "C4_L2_m8" == w.name:
        assert {1, 2} <= kinds                       # coarser and finer neighbours occur
    if w.name.startswith("C4"):
        assert 4 in kinds and len(set(t[:, :, 3].ravel().tolist()) - {-1}) > 1   # corners, rotations


@pytest.mark.parametrize("name", sorted(CONNS))
def test_compact_table_bit_exact_random_two_level_forests(rng, name):
    conn = CONNS[name]
    for trial in range(3):
        m = [4, 8, 6][trial]
        fr = _random_forest(rng, conn, 2, m)
        t, o = compact_pair(fr.levels, fr.tree_ids, conn, m)
        np.testing.assert_array_equal(t, o)


def test_compact_table_worked_example():
    """Hand-checked rows: C2's mesh (reading 11) -- a level-3 patch left of the refined plus shape
    sees two finer leaves on its +x face; a level-4 patch on the rim sees a coarser leaf, half given
    by its own position; everything is axis-aligned (xform 0) on the single periodic tree."""
    w = c2()
    t, _ = compact_pair(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)
    assert (t[:, :, 3][t[:, :, 0] <= 2] == 0).all()
    lv = w.forest.levels
    fine_face = np.nonzero((t[:, :4, 0] == 2).any(axis=1))[0]
    assert len(fine_face) and (lv[fine_face] == 3).all()
    p = int(fine_face[0])
    d = int(np.nonzero(t[p, :4, 0] == 2)[0][0])
    a, b = t[p, d, 1], t[p, d, 2]
    assert lv[a] == lv[b] == 4 and a != b
    coarse = np.nonzero((t[:, :4, 0] == 1).any(axis=1))[0]
    assert (lv[coarse] == 4).all() and set(t[coarse][:, :4, 4][t[coarse][:, :4, 0] == 1].tolist()) == {0, 1}


def test_library_exports_every_declared_octree_symbol():
    from paper_1308_1472_b200 import fc3
    hdr = open(os.path.join(ROOT, "include", "fc3.h")).read()
    declared = sorted(set(re.findall(r"^\s*int\s+(fc3_\w+)\s*\(", hdr, re.M)))
    assert declared == sorted(fc3.EXPORTS3)
    L = fc.lib()
    for name in declared:
        assert hasattr(L, name), name


def test_octree_tables_bit_exact_with_the_oracle():
    """The planner's hash lookups (plan3.cpp) vs the oracle's Morton binary searches (forest3.c):
    identical canonical records on uniform / AMR, periodic / outflow / mixed bricks."""
    from oracle.octree import OracleForest3
    from paper_1308_1472_b200 import fc3
    from workloads.octree import forest3
    cases = [forest3((2, 1, 1), 1), forest3((1, 2, 2), 1, periodic=(False, False, False)),
             forest3((2, 2, 1), 1, refine=lambda t, x, y, z, h: t == 0 and x < 0.5 and (y + z) < 0.9),
             forest3((2, 1, 2), 1, refine=lambda t, x, y, z, h: (t + x + y + z) < 1.2, periodic=(True, False, True)),
             forest3((1, 1, 1), 2, refine=lambda t, x, y, z, h: x + y < 0.6, periodic=(False, True, False))]
    for f in cases:
        for m in (4, 6):
            g = fc3.Forest3(f, m, device=-1)
            np.testing.assert_array_equal(g.ghost_table(), OracleForest3(f, m).ghost_table())
            g.close()
