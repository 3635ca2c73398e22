"""Pins for the oracle's forest decode and brute-force ghost tables (oracle/forest.c).

Every expected value here comes from the paper/SPEC text (tests/golden/spec_examples.json) or
from independent geometry written in this file (global-grid index arithmetic, a leaf raster),
never from the oracle itself or from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import forests as F
from workloads.configs import c1, c2, c3, c5

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def mk(levels, tree_ids, conn, m=4):
    return oracle.OracleForest(np.array(levels, np.int8), np.array(tree_ids, np.int32), conn, m)


# ---- decode -------------------------------------------------------------------------------------
def test_morton_spec_examples():
    ex = GOLD["morton"]
    # level 2, Lmax 2, (1,1) -> Morton index 3, i.e. the 4th leaf of a uniform level-2 tree
    f = mk([2] * 16, [0] * 16, F.periodic_unit_square())
    x, y, lmax = f.coords()
    e = ex[0]
    assert lmax == e["lmax"] and (x[e["index"]], y[e["index"]]) == (e["x"], e["y"])
    # level-1 quadrant (2,0) in Lmax=2 units is the second level-1 child in z-order
    f = mk([2, 2, 2, 2, 1, 1, 1], [0] * 7, F.periodic_unit_square())
    x, y, lmax = f.coords()
    e = ex[1]
    assert lmax == 2
    level1 = [(int(a), int(b)) for a, b, l in zip(x, y, [2, 2, 2, 2, 1, 1, 1]) if l == 1]
    # children of the root in z-order are (0,0) [refined here], (2,0), (0,2), (2,2)
    assert [(0, 0)] + level1 == [(0, 0), (2, 0), (0, 2), (2, 2)]
    assert level1.index((e["x"], e["y"])) + 2 == e["position_among_level1_children"]


def test_patch_count_law():
    """a uniform level-l tree has 2^(2l) patches; any other count fails."""
    for l in GOLD["patch_count_law"]["levels"]:
        n = 2 ** (2 * l)
        mk([l] * n, [0] * n, F.periodic_unit_square())
        if l > 0:
            with pytest.raises(ValueError):
                mk([l] * (n - 1), [0] * (n - 1), F.periodic_unit_square())
            with pytest.raises(ValueError):
                mk([l] * (n + 1), [0] * (n + 1), F.periodic_unit_square())


def test_resolution_bookkeeping():
    g = GOLD["resolution"]
    for l, cells in zip(g["levels"], g["cells_per_side"]):
        f = mk([l] * 4 ** l, [0] * 4 ** l, F.periodic_unit_square(), m=g["m"])
        x, y, lmax = f.coords()
        assert (x.max() + 1) * g["m"] == cells and (y.max() + 1) * g["m"] == cells


def test_decode_matches_independent_zorder_generator():
    """The generator enumerates z-order by recursive child expansion (no bit interleaving);
    the oracle decodes by de-interleaving a Morton cursor.  They must agree."""
    for w in (c1(), c2(), c3(level=3, m=8), c5(level=2, m=8)):
        f = oracle.forest_for(w)
        x, y, lmax = f.coords()
        s = 2 ** (lmax - w.forest.levels.astype(np.int64))
        np.testing.assert_array_equal(x, w.forest.ix * s)
        np.testing.assert_array_equal(y, w.forest.iy * s)


def test_tiling_errors():
    conn = F.periodic_unit_square()
    with pytest.raises(ValueError):     # misaligned: a level-1 leaf starting at Morton index 1
        mk([2, 1, 1, 1, 2, 2, 2], [0] * 7, conn)
    with pytest.raises(ValueError):     # decreasing tree ids
        mk([0, 0], [1, 0], F.brick(2, 1))
    with pytest.raises(ValueError):     # tree 1 missing
        mk([0], [0], F.brick(2, 1))
    bad = F.brick(2, 1)
    bad.tree_to_face[1] = 3             # asymmetric link
    with pytest.raises(ValueError):
        mk([0, 0], [0, 1], bad)


# ---- ghost tables ---------------------------------------------------------------------------------
def _ring_cells(m):
    out = []
    for j in range(-1, m + 3):
        for i in range(-1, m + 3):
            if 1 <= i <= m and 1 <= j <= m:
                continue
            out.append((i, j))
    return out


def test_table_uniform_periodic_matches_global_index():
    """Uniform periodic tree: every ring cell copies the global cell (gx mod N, gy mod N)."""
    for w in (c1(), c1(level=3, m=4)):
        f = oracle.forest_for(w)
        tab = f.ghost_table()
        m = w.m
        lvl = int(w.forest.levels[0])
        N = (2 ** lvl) * m
        owner = {(int(a), int(b)): p for p, (a, b) in enumerate(zip(w.forest.ix, w.forest.iy))}
        for p in range(w.num_patches):
            for r, (i, j) in enumerate(_ring_cells(m)):
                gx = (int(w.forest.ix[p]) * m + i - 1) % N
                gy = (int(w.forest.iy[p]) * m + j - 1) % N
                q = owner[(gx // m, gy // m)]
                assert tuple(tab[p, r, :4]) == (oracle.OP_COPY, q, gx % m + 1, gy % m + 1)


def test_table_walls_matches_mirror_rule():
    """Walled unit square: ghost cells outside the domain are BCX/BCY wall mirrors of the own
    patch (y-face BC is the final writer at domain corners), the rest copy the global cell."""
    w = c3(level=2, m=8)
    f = oracle.forest_for(w)
    tab = f.ghost_table()
    m, N = w.m, 4 * w.m
    owner = {(int(a), int(b)): p for p, (a, b) in enumerate(zip(w.forest.ix, w.forest.iy))}
    for p in range(w.num_patches):
        for r, (i, j) in enumerate(_ring_cells(m)):
            gx = int(w.forest.ix[p]) * m + i - 1
            gy = int(w.forest.iy[p]) * m + j - 1
            rec = tuple(tab[p, r, :5])
            if gy < 0 or gy >= N:
                mj = 1 - j if gy < 0 else 2 * m + 1 - j
                assert rec == (oracle.OP_BCY, p, i, mj, F.WALL)
            elif gx < 0 or gx >= N:
                mi = 1 - i if gx < 0 else 2 * m + 1 - i
                assert rec == (oracle.OP_BCX, p, mi, j, F.WALL)
            else:
                q = owner[(gx // m, gy // m)]
                assert rec[:4] == (oracle.OP_COPY, q, gx % m + 1, gy % m + 1)


def test_table_amr_matches_leaf_raster():
    """C2 (two levels, periodic): locate every ghost-cell centre in a raster of leaf ids painted
    from the generator's coordinates, and derive the op and source index geometrically."""
    w = c2()
    f = oracle.forest_for(w)
    tab = f.ghost_table()
    m = w.m
    L = 4                                   # finest level
    H = 2 * m * 2 ** L                      # raster resolution: half fine cells
    lv = w.forest.levels.astype(int)
    raster = np.full((H, H), -1, np.int64)
    for p in range(w.num_patches):
        s = 2 * m * 2 ** (L - lv[p])        # patch width in half-fine-cell units
        x0, y0 = int(w.forest.ix[p]) * s, int(w.forest.iy[p]) * s
        raster[y0:y0 + s, x0:x0 + s] = p
    assert (raster >= 0).all()
    counts = {}
    for p in range(w.num_patches):
        s = 2 * m * 2 ** (L - lv[p])
        cw = s // m                          # own cell width
        x0, y0 = int(w.forest.ix[p]) * s, int(w.forest.iy[p]) * s
        for r, (i, j) in enumerate(_ring_cells(m)):
            X = (x0 + (i - 1) * cw + cw // 2) % H
            Y = (y0 + (j - 1) * cw + cw // 2) % H
            q = raster[Y, X]
            sq = 2 * m * 2 ** (L - lv[q])
            qw = sq // m
            qx0, qy0 = int(w.forest.ix[q]) * sq, int(w.forest.iy[q]) * sq
            rec = tab[p, r]
            assert rec[1] == q
            if lv[q] == lv[p]:
                exp = (oracle.OP_COPY, (X - qx0) // qw + 1, (Y - qy0) // qw + 1)
                got = (rec[0], rec[2], rec[3])
            elif lv[q] == lv[p] + 1:      # the ghost covers a 2x2 block of q's cells
                exp = (oracle.OP_AVG4, (X - cw // 2 - qx0) // qw + 1, (Y - cw // 2 - qy0) // qw + 1)
                got = (rec[0], rec[2], rec[3])
            else:
                I, J = (X - qx0) // qw + 1, (Y - qy0) // qw + 1
                sx = 1 if (X - qx0) % qw > qw // 2 else -1
                sy = 1 if (Y - qy0) % qw > qw // 2 else -1
                exp = (oracle.OP_INTERP, I, J, sx, sy)
                got = (rec[0], rec[2], rec[3], rec[4], rec[5])
            assert got == exp, (p, i, j)
            counts[rec[0]] = counts.get(rec[0], 0) + 1
    assert counts[oracle.OP_AVG4] > 0 and counts[oracle.OP_INTERP] > 0


def test_table_reciprocity():
    """face-neighbour reciprocity, on uniform, AMR and multi-tree forests."""
    for w in (c1(), c2(), c5(level=2, m=8)):
        f = oracle.forest_for(w)
        tab = f.ghost_table()
        m = w.m
        rc = _ring_cells(m)
        face = [r for r, (i, j) in enumerate(rc) if (1 <= i <= m) != (1 <= j <= m)]
        for p in range(w.num_patches):
            srcs = set(int(tab[p, r, 1]) for r in face
                       if tab[p, r, 0] in (oracle.OP_COPY, oracle.OP_AVG4, oracle.OP_INTERP))
            for q in srcs:
                back = set(int(tab[q, r, 1]) for r in face
                           if tab[q, r, 0] in (oracle.OP_COPY, oracle.OP_AVG4, oracle.OP_INTERP))
                assert p in back, (p, q)
