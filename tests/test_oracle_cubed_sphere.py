"""Pins for the cubed-sphere (C4) inputs and the oracle's multiblock ghost logic on them.

Independent references: the sphere's area (4 pi), the continuous velocity field omega n_hat x X
(sign and magnitude of the stream-function edge fluxes), the cube embedding of the trees
(a ghost cell across a tree face folds onto the neighbour face at the same distance from the
shared edge), the 8 cube vertices (three-tree corners), exact constant preservation, and
conservation of sum kappa q while the solution is constant near the cube corners.
"""
import math

import numpy as np
import pytest

import oracle
from workloads import cubed_sphere as CS


@pytest.fixture(scope="module")
def uni():
    return CS.c4_workload(base_level=2, m=8, uniform=True, steps=5)


def cell_area(w):
    h = np.ldexp(1.0, -w.forest.levels.astype(np.int64))[:, None, None] / w.m
    return w.aux[:, 0, 2:w.m + 2, 2:w.m + 2] * h * h


def test_c4_mesh_counts():
    """Reading 12: the band rule at base level 4 refines 684 parents -> 3588 patches."""
    w = CS.c4_workload()
    assert w.num_patches == 3588 and w.info["refined_parents"] == 684
    assert (w.forest.levels == 4).sum() == 852 and (w.forest.levels == 5).sum() == 2736
    assert abs(CS.band_latitude() - (-0.6591)) < 1e-4


def test_capacity_sums_to_sphere_area(uni):
    assert abs(cell_area(uni).sum() - 4 * math.pi) < 1e-12


def test_connectivity_symmetric_and_cube_like():
    c = CS.cube_connectivity()
    for t in range(6):
        for f in range(4):
            nt, code = c.tree_to_tree[4 * t + f], c.tree_to_face[4 * t + f]
            assert nt != t
            assert c.tree_to_tree[4 * nt + (code & 3)] == t
            assert c.tree_to_face[4 * nt + (code & 3)] == f + 4 * (code >> 2)
    # every tree touches 4 distinct others (not its antipode)
    for t in range(6):
        assert len(set(c.tree_to_tree[4 * t:4 * t + 4].tolist())) == 4


def test_edge_velocities_match_solid_body_rotation():
    """u~ d_eta = flux through the left edge ~ (omega n_hat x X) . nu |edge| at the midpoint."""
    m = 16
    for t in range(6):
        aux, _ = CS.patch_geometry(CS.cube_connectivity(), t, 0.25, 0.25, 0.5, m)
        d = 0.5 / m
        for (i, j) in ((5, 7), (10, 3), (2, 12)):
            xa, ya = 0.25 + (i - 1) * d, 0.25 + (j - 1) * d
            a, b = CS.sphere_point(t, xa, ya), CS.sphere_point(t, xa, ya + d)
            mid = (a + b) / np.linalg.norm(a + b)
            tang = (b - a) / np.linalg.norm(b - a)
            nu = np.cross(tang, mid)                 # +xi side normal (right-handed frames)
            vel = CS.OMEGA * np.cross(CS.AXIS, mid)
            seg = math.acos(float(np.clip(a @ b, -1, 1)))
            approx = float(vel @ nu) * seg
            exact = aux[1, j + 1, i + 1] * d
            assert abs(exact - approx) <= 1e-4 * max(1.0, abs(approx)), (t, i, j, exact, approx)


def test_discrete_divergence_free(uni):
    m = uni.m
    a = uni.aux
    div = (a[:, 1, 2:m + 2, 3:m + 3] - a[:, 1, 2:m + 2, 2:m + 2]) + \
          (a[:, 2, 3:m + 3, 2:m + 2] - a[:, 2, 2:m + 2, 2:m + 2])
    assert np.abs(div).max() < 1e-12 * np.abs(a[:, 1:]).max()


def test_ghost_sources_fold_onto_neighbour_face(uni):
    """Across a tree face, a same-level ghost at outward distance d from the shared edge takes its
    value from the neighbour-face cell at distance d from that edge, at the same edge position
    (checked in the cube embedding only)."""
    f = oracle.forest_for(uni)
    tab = f.ghost_table()
    x, y, lmax = f.coords()
    m = uni.m
    cells = [(i, j) for j in range(-1, m + 3) for i in range(-1, m + 3) if not (1 <= i <= m and 1 <= j <= m)]
    checked = 0
    for p in range(uni.num_patches):
        t = int(uni.forest.tree_ids[p])
        L = int(uni.forest.levels[p])
        h = 0.5 ** L
        for r, (i, j) in enumerate(cells):
            rec = tab[p, r]
            if rec[0] != oracle.OP_COPY or uni.forest.tree_ids[rec[1]] == t:
                continue
            xi = x[p] / 2 ** lmax + (i - 0.5) * h / m
            eta = y[p] / 2 ** lmax + (j - 0.5) * h / m
            outx, outy = xi < 0 or xi > 1, eta < 0 or eta > 1
            if outx and outy:
                continue
            n = CS.FRAMES[t][0]
            if outx:
                xe = 0.0 if xi < 0 else 1.0
                dist = abs(xi - xe) * 2.0
                edge = CS.cube_point(t, xe, eta)
            else:
                ye = 0.0 if eta < 0 else 1.0
                dist = abs(eta - ye) * 2.0
                edge = CS.cube_point(t, xi, ye)
            expect = edge - dist * n
            q = rec[1]
            tq = int(uni.forest.tree_ids[q])
            hq = 0.5 ** int(uni.forest.levels[q])
            xs = x[q] / 2 ** lmax + (rec[2] - 0.5) * hq / m
            ys = y[q] / 2 ** lmax + (rec[3] - 0.5) * hq / m
            got = CS.cube_point(tq, xs, ys)
            np.testing.assert_allclose(got, expect, atol=1e-12)
            checked += 1
    assert checked > 500


def test_corner3_cells_sit_at_cube_vertices(uni):
    f = oracle.forest_for(uni)
    tab = f.ghost_table()
    x, y, lmax = f.coords()
    m = uni.m
    cells = [(i, j) for j in range(-1, m + 3) for i in range(-1, m + 3) if not (1 <= i <= m and 1 <= j <= m)]
    n3 = 0
    for p in range(uni.num_patches):
        t = int(uni.forest.tree_ids[p])
        h = 0.5 ** int(uni.forest.levels[p])
        for r, (i, j) in enumerate(cells):
            if tab[p, r, 0] != oracle.OP_CORNER3:
                continue
            n3 += 1
            cx = x[p] / 2 ** lmax + (0.0 if i < 1 else h)
            cy = y[p] / 2 ** lmax + (0.0 if j < 1 else h)
            v = CS.cube_point(t, cx, cy)
            assert np.allclose(np.abs(v), 1.0)
    assert n3 == 8 * 3 * 4   # 8 vertices x 3 patch corners x 4 cells


def test_constant_state_exact_on_sphere():
    w = CS.c4_workload(base_level=2, m=8, steps=5)
    w.q0[:] = 0.37
    q, _, _ = oracle.run(w)
    assert (q == 0.37).all()


def test_conservation_away_from_cube_corners(uni):
    """A bump at a face centre, run for steps in which it cannot reach the three-tree corners:
    sum kappa q is conserved to roundoff (the CORNER3 averages are the only non-conservative
    ghosts on a uniform sphere)."""
    w = CS.c4_workload(base_level=3, m=8, uniform=True, steps=6)
    X = w.info["centres"]
    d = np.arccos(np.clip(X @ np.array([1.0, 0.0, 0.0]), -1, 1))
    w.q0 = (0.1 + np.where(d < 0.3, 0.5 * (1 + np.cos(math.pi * d / 0.3)), 0.0))[:, None]
    A = cell_area(w)
    m0 = (w.q0[:, 0] * A).sum()
    q, cfl, _ = oracle.run(w)
    assert abs((q[:, 0] * A).sum() - m0) <= 1e-14 * 6 * m0
