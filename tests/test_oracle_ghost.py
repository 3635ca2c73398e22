"""Pins for the oracle's ghost fill (oracle/ghost.c).

Expected values come from SPEC's worked examples (tests/golden), from a monolithic padded global
array assembled here with numpy's own padding modes (periodic = wrap, outflow = edge,
wall = symmetric + negated normal momentum), from exact affine data, and from the algebraic
conservation identity of the interpolation (mean of 4 children = coarse value).
"""
import json
import os

import numpy as np

import oracle
from workloads import forests as F
from workloads.configs import c1, c2, c3, c5

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def ring_mask(m):
    k = np.zeros((m + 4, m + 4), bool)
    k[:, :] = True
    k[2:m + 2, 2:m + 2] = False
    return k


def assemble_global(w, q):
    """Uniform single-level forest of a brick of trees -> global array [meqn][Ny][Nx]
    (trees side by side along x as the brick builders lay them out)."""
    m = w.m
    lvl = int(w.forest.levels[0])
    nt = w.forest.conn.num_trees
    N = 2 ** lvl * m
    G = np.zeros((q.shape[1], N, nt * N))
    for p in range(w.num_patches):
        t = int(w.forest.tree_ids[p])
        x0 = t * N + int(w.forest.ix[p]) * m
        y0 = int(w.forest.iy[p]) * m
        G[:, y0:y0 + m, x0:x0 + m] = q[p]
    return G, N


def compare_rings_with_global(w, q, Gp):
    f = oracle.forest_for(w)
    qp = f.ghost_fill(f.pad(q))
    m = w.m
    N = 2 ** int(w.forest.levels[0]) * m
    rm = ring_mask(m)
    for p in range(w.num_patches):
        t = int(w.forest.tree_ids[p])
        x0 = t * N + int(w.forest.ix[p]) * m
        y0 = int(w.forest.iy[p]) * m
        ref = Gp[:, y0:y0 + m + 4, x0:x0 + m + 4]
        np.testing.assert_array_equal(qp[p][:, rm], ref[:, rm])


def test_ghost_equivalence_periodic(rng):
    """SPEC.md:209 / acceptance 10: rings equal the wrapped global array."""
    w = c1()
    q = rng.standard_normal(w.q0.shape)
    G, _ = assemble_global(w, q)
    Gp = np.pad(G, ((0, 0), (2, 2), (2, 2)), mode="wrap")
    compare_rings_with_global(w, q, Gp)


def test_ghost_equivalence_walls(rng):
    """Reflecting walls: mirror + negated normal momentum, x faces then y faces (Clawpack bc2)."""
    w = c3(level=2, m=8)
    q = rng.standard_normal(w.q0.shape)
    G, _ = assemble_global(w, q)
    Gx = np.pad(G, ((0, 0), (0, 0), (2, 2)), mode="symmetric")
    Gx[1, :, :2] *= -1.0
    Gx[1, :, -2:] *= -1.0
    Gp = np.pad(Gx, ((0, 0), (2, 2), (0, 0)), mode="symmetric")
    Gp[2, :2, :] *= -1.0
    Gp[2, -2:, :] *= -1.0
    compare_rings_with_global(w, q, Gp)


def test_ghost_equivalence_brick_outflow(rng):
    """4-tree brick with outflow (C5 layout): edge padding; tree faces crossed aligned."""
    w = c5(level=2, m=8)
    q = rng.standard_normal(w.q0.shape)
    G, _ = assemble_global(w, q)
    Gp = np.pad(G, ((0, 0), (2, 2), (2, 2)), mode="edge")
    compare_rings_with_global(w, q, Gp)


def test_ghost_reversed_tree_link(rng):
    """2-tree brick whose shared face is declared reversed: tree 1's frame is the physical one
    reflected in y.  Its rings, mapped back to the physical frame, equal the padded global array."""
    m, lvl = 8, 1
    N = 2 ** lvl * m
    G = rng.standard_normal((1, N, 2 * N))
    Gp = np.pad(G, ((0, 0), (2, 2), (2, 2)), mode="edge")
    for reversed_link in (False, True):
        conn = F.brick(2, 1, bc=F.OUTFLOW, reversed_x_links=(0,) if reversed_link else ())
        fr = F.forest_uniform(conn, lvl)
        q = np.zeros((fr.num_patches, 1, m, m))
        for p in range(fr.num_patches):
            t = int(fr.tree_ids[p])
            x0, y0 = int(fr.ix[p]) * m, int(fr.iy[p]) * m
            blk = G[:, :, t * N:(t + 1) * N]
            if t == 1 and reversed_link:
                blk = blk[:, ::-1, :]           # tree 1's own frame
            q[p] = blk[:, y0:y0 + m, x0:x0 + m]
        f = oracle.OracleForest(fr.levels, fr.tree_ids, conn, m)
        qp = f.ghost_fill(f.pad(q))
        rm = ring_mask(m)
        for p in range(fr.num_patches):
            t = int(fr.tree_ids[p])
            x0, y0 = int(fr.ix[p]) * m, int(fr.iy[p]) * m
            if t == 1 and reversed_link:
                # physical rows of tree 1 reflected: local padded row a <-> physical padded row
                ref = Gp[:, ::-1, :][:, y0:y0 + m + 4, N + x0:N + x0 + m + 4]
            else:
                ref = Gp[:, y0:y0 + m + 4, t * N + x0:t * N + x0 + m + 4]
            np.testing.assert_array_equal(qp[p][:, rm], ref[:, rm])


def _records_by_op(f, op):
    tab = f.ghost_table()
    m = f.m
    cells = [(i, j) for j in range(-1, m + 3) for i in range(-1, m + 3)
             if not (1 <= i <= m and 1 <= j <= m)]
    out = []
    for p in range(f.P):
        for r, (i, j) in enumerate(cells):
            if tab[p, r, 0] == op:
                out.append((p, i, j, tab[p, r]))
    return out


def test_spec_average_examples():
    """fine constant -> same constant; fine 2x2 block (1,2,3,4) -> 2.5."""
    w = c2()
    f = oracle.forest_for(w)
    p, i, j, rec = _records_by_op(f, oracle.OP_AVG4)[0]
    for ex in GOLD["average"]:
        q = np.zeros(w.q0.shape)
        src, a, b = rec[1], rec[2], rec[3]
        q[src, 0, b - 1, a - 1], q[src, 0, b - 1, a], q[src, 0, b, a - 1], q[src, 0, b, a] = ex["fine"]
        qp = f.ghost_fill(f.pad(q))
        assert qp[p, 0, j + 1, i + 1] == ex["coarse_ghost"]


def test_spec_interpolate_examples():
    """coarse row (c,c,c) -> c; (1,2,3) -> {1.75, 2.25}; (1,5,2) -> {5, 5}
    (the two fine ghosts on either side of the coarse centre along x, constant column in y)."""
    w = c2()
    f = oracle.forest_for(w)
    recs = _records_by_op(f, oracle.OP_INTERP)
    # a coarse cell whose x-stencil (I-1, I, I+1) is interior to its patch
    for p, i, j, rec in recs:
        if 2 <= rec[2] <= w.m - 1:
            break
    src, I, J = rec[1], rec[2], rec[3]
    pair = [(pp, ii, jj, rr) for pp, ii, jj, rr in recs
            if pp == p and rr[1] == src and rr[2] == I and rr[3] == J and rr[5] == rec[5]]
    assert sorted(int(r[4]) for *_, r in pair) == [-1, 1]
    for ex in GOLD["interpolate"]:
        row = ex["row"]
        q = np.full(w.q0.shape, row[1])      # constant in y: the y slope vanishes
        q[src, 0, J - 1, I - 2:I + 1] = row
        qp = f.ghost_fill(f.pad(q))
        got = sorted(qp[pp, 0, jj + 1, ii + 1] for pp, ii, jj, _ in pair)
        assert got == sorted(ex["ghosts"])


def test_interp_conservative_and_no_new_extrema(rng):
    """the 4 fine ghosts under one coarse cell average to it (to rounding), and
    every interpolated value lies within the coarse plus-stencil's range."""
    w = c2()
    f = oracle.forest_for(w)
    recs = _records_by_op(f, oracle.OP_INTERP)
    for trial in range(20):
        q = rng.standard_normal(w.q0.shape) * 10.0 ** rng.integers(-3, 4)
        qp = f.ghost_fill(f.pad(q))
        groups = {}
        for p, i, j, rec in recs:
            key = (p, int(rec[1]), int(rec[2]), int(rec[3]))
            groups.setdefault(key, []).append(qp[p, 0, j + 1, i + 1])
            C = qp[rec[1], 0]
            I, J = rec[2] + 1, rec[3] + 1
            st = [C[J, I], C[J, I - 1], C[J, I + 1], C[J - 1, I], C[J + 1, I]]
            g = qp[p, 0, j + 1, i + 1]
            assert min(st) <= g <= max(st)
        for (p, src, I, J), vals in groups.items():
            if len(vals) == 4:
                c = qp[src, 0, J + 1, I + 1]
                assert abs(np.mean(vals) - c) <= 4e-16 * max(abs(c), max(np.abs(vals)))


def test_affine_data_exact_away_from_boundaries():
    """averaging is exact for affine data; interpolation is exact where the limiter
    is inactive (monotone affine data): every copy/average/interpolate ghost equals the affine
    function at the ghost-cell centre."""
    conn = F.walled_unit_square(F.OUTFLOW)
    fr = F.forest_refined(conn, 2, lambda t, x, y, h: (abs(x - 0.5) < 0.25) & (abs(y - 0.5) < 0.25))
    m = 8
    X, Y = F.cell_centres(fr, m, ghost=2)
    fn = lambda x, y: 3.0 + 2.0 * x - 5.0 * y
    q = fn(X, Y)[:, None, 2:m + 2, 2:m + 2].copy()
    f = oracle.OracleForest(fr.levels, fr.tree_ids, conn, m)
    qp = f.ghost_fill(f.pad(q))
    tab = f.ghost_table()
    cells = [(i, j) for j in range(-1, m + 3) for i in range(-1, m + 3)
             if not (1 <= i <= m and 1 <= j <= m)]
    seen = set()
    for p in range(f.P):
        for r, (i, j) in enumerate(cells):
            op = tab[p, r, 0]
            if op in (oracle.OP_COPY, oracle.OP_AVG4, oracle.OP_INTERP):
                seen.add(int(op))
                exact = fn(X[p, j + 1, i + 1], Y[p, j + 1, i + 1])
                assert abs(qp[p, 0, j + 1, i + 1] - exact) <= 1e-14 * 8, (p, i, j, op)
    assert seen == {oracle.OP_COPY, oracle.OP_AVG4, oracle.OP_INTERP}


def test_constant_state_exact_all_configs():
    for w in (c1(), c2(), c3(level=2, m=8), c5(level=2, m=8)):
        f = oracle.forest_for(w)
        q = np.full(w.q0.shape, 0.7)
        qp = f.ghost_fill(f.pad(q))
        if w.meqn >= 3:   # wall BCs negate momentum; zero momentum keeps the state constant
            q[:, 1:3] = 0.0
            qp = f.ghost_fill(f.pad(q))
            assert (qp[:, 0] == 0.7).all() and (qp[:, 1:3] == 0.0).all()
        else:
            assert (qp == 0.7).all()
