"""Pins for the octree oracle (oracle/forest3.c; reading 26), independent of its code:
  * decode: the generator's recursive z-order geometry, the 8^l leaf law, tiling errors;
  * ghost fill on uniform forests: bitwise the monolithic padded grid (numpy np.pad with 'wrap'
    on periodic axes, 'edge' on outflow axes: Clawpack's zero-order extrapolation, x then y then z);
  * coarse/fine ghosts: constants stay constant, affine data are reproduced exactly, the mean of
    the 8 interpolated children is the coarse value, no new extrema;
  * the split step: constant states bitwise; data varying along one axis only equals the
    independent 1D wave-propagation code of tests/test_oracle_1d_reduction.py; Courant number 1
    shifts integer data exactly by (1, 1, 1) (first and second order); conservation on periodic
    forests; affine data translated exactly across coarse/fine faces away from outflow faces.
"""
import importlib.util
import os

import numpy as np
import pytest

from oracle.octree import OP_AVG8, OP_BCX, OP_BCZ, OP_COPY, OP_INTERP, OracleForest3, run3
from workloads.octree import cell_centres, forest3, leaf_geometry

HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location("red1d", os.path.join(HERE, "test_oracle_1d_reduction.py"))
red1d = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(red1d)


def assemble(f, m, q):
    """uniform forest interiors [P][m][m][m] -> global grid [Z][Y][X] (brick units)"""
    lv = int(f.levels[0])
    assert (f.levels == lv).all()
    N = (2 ** lv) * m
    Tx, Ty, Tz = f.dims
    G = np.zeros((Tz * N, Ty * N, Tx * N))
    for p, (t, x0, y0, z0, h) in enumerate(leaf_geometry(f)):
        tx, ty, tz = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        X, Y, Z = round((tx + x0) * N), round((ty + y0) * N), round((tz + z0) * N)
        G[Z:Z + m, Y:Y + m, X:X + m] = q[p]
    return G


def scatter(f, m, G):
    lv = int(f.levels[0])
    N = (2 ** lv) * m
    Tx, Ty, Tz = f.dims
    q = np.zeros((f.num_patches, m, m, m))
    for p, (t, x0, y0, z0, h) in enumerate(leaf_geometry(f)):
        tx, ty, tz = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        X, Y, Z = round((tx + x0) * N), round((ty + y0) * N), round((tz + z0) * N)
        q[p] = G[Z:Z + m, Y:Y + m, X:X + m]
    return q


# ---- decode ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("dims,base", [((1, 1, 1), 2), ((2, 1, 3), 1)])
def test_decode_matches_recursive_geometry_and_the_8_to_the_l_law(dims, base):
    f = forest3(dims, base, refine=lambda t, x, y, z, h: (x + y + z) < 0.9)
    o = OracleForest3(f, 4)
    x, y, z, lmax = o.coords()
    for p, (t, x0, y0, z0, h) in enumerate(leaf_geometry(f)):
        assert (x[p], y[p], z[p]) == (round(x0 * 2 ** lmax), round(y0 * 2 ** lmax), round(z0 * 2 ** lmax))
    u = forest3(dims, base)
    assert u.num_patches == int(np.prod(dims)) * 8 ** base


def test_decode_rejects_bad_tilings():
    f = forest3((1, 1, 1), 1)
    with pytest.raises(ValueError):                      # incomplete tree
        OracleForest3(type(f)(f.levels[:7], f.tree_ids[:7], f.t2t, f.fbc, f.dims), 4)
    lv = np.array([2] * 8 + [1] * 7, np.int8)             # level-2 block first: fine, then the rest
    OracleForest3(type(f)(lv, np.zeros(15, np.int32), f.t2t, f.fbc, f.dims), 4)
    lv2 = np.array([2] + [1] * 7 + [2] * 7, np.int8)      # a level-1 leaf not aligned to its size
    with pytest.raises(ValueError):
        OracleForest3(type(f)(lv2, np.zeros(15, np.int32), f.t2t, f.fbc, f.dims), 4)


# ---- ghost fill: uniform forests against the monolithic padded grid --------------------------------
@pytest.mark.parametrize("dims,periodic,m", [((2, 1, 1), (True, True, True), 4),
                                             ((1, 2, 2), (False, False, False), 6),
                                             ((2, 2, 1), (True, False, True), 4)])
def test_uniform_fill_equals_monolithic_padding(rng, dims, periodic, m):
    f = forest3(dims, 1, periodic=periodic)
    o = OracleForest3(f, m)
    G = rng.standard_normal(tuple(reversed([d * 2 * m for d in dims])))
    q = scatter(f, m, G)
    padded = o.ghost_fill(o.pad(q))
    P = G
    for axis, per in zip((2, 1, 0), periodic):          # x, y, z (outflow: edge = Clawpack bc3 order)
        width = [(0, 0)] * 3
        width[axis] = (2, 2)
        P = np.pad(P, width, mode="wrap" if per else "edge")
    N = 2 * m
    for p, (t, x0, y0, z0, h) in enumerate(leaf_geometry(f)):
        Tx, Ty = dims[0], dims[1]
        tx, ty, tz = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        X, Y, Z = round((tx + x0) * N), round((ty + y0) * N), round((tz + z0) * N)
        np.testing.assert_array_equal(padded[p], P[Z:Z + m + 4, Y:Y + m + 4, X:X + m + 4])


def amr_forest(dims=(2, 1, 1), periodic=(True, True, True)):
    return forest3(dims, 1, refine=lambda t, x, y, z, h: t == 0 and x < 0.5 and (y + z) < 0.9,
                   periodic=periodic)


def test_coarse_fine_ghosts_constant_and_affine():
    m = 4
    f = amr_forest(periodic=(False, False, False))
    o = OracleForest3(f, m)
    rec = o.ghost_table()
    ops = set(np.unique(rec[:, :, 0]).tolist())
    assert {OP_COPY, OP_AVG8, OP_INTERP} <= ops
    pc = o.ghost_fill(o.pad(np.full((f.num_patches, m, m, m), 2.5)))
    assert (pc == 2.5).all()
    # affine data: every COPY / AVG8 / INTERP ghost equals the affine function at the ghost centre
    a = np.array([0.3, -1.2, 0.7, 2.1])
    cen = cell_centres(f, m)
    q = a[0] + a[1] * cen[:, 0] + a[2] * cen[:, 1] + a[3] * cen[:, 2]
    pad = o.ghost_fill(o.pad(q))
    n = m + 4
    ring = [(i, j, k) for k in range(-1, m + 3) for j in range(-1, m + 3) for i in range(-1, m + 3)
            if not (1 <= i <= m and 1 <= j <= m and 1 <= k <= m)]
    geo = leaf_geometry(f)
    Tx, Ty = f.dims[0], f.dims[1]
    checked = 0
    n_interp = [0]
    for p in range(f.num_patches):
        t, x0, y0, z0, h = geo[p]
        tx, ty, tz = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        for r, (i, j, k) in enumerate(ring):
            if rec[p, r, 0] not in (OP_COPY, OP_AVG8, OP_INTERP):
                continue
            if rec[p, r, 0] == OP_INTERP:   # slopes next to an outflow face are clipped: skip those
                ts, xs, ys, zs, hs = geo[rec[p, r, 1]]
                cs = [(ts % Tx) + xs, ((ts // Tx) % Ty) + ys, (ts // (Tx * Ty)) + zs]
                cc = [cs[d] + hs * (rec[p, r, 2 + d] - 0.5) / m for d in range(3)]
                if any(cc[d] < 1.5 * hs / m or cc[d] > f.dims[d] - 1.5 * hs / m for d in range(3)):
                    continue
            X = tx + x0 + h * (i - 0.5) / m
            Y = ty + y0 + h * (j - 0.5) / m
            Z = tz + z0 + h * (k - 0.5) / m
            want = a[0] + a[1] * X + a[2] * Y + a[3] * Z
            assert abs(pad[p, k + 1, j + 1, i + 1] - want) <= 1e-13 * 4, (p, (i, j, k), rec[p, r])
            checked += 1
            n_interp[0] += rec[p, r, 0] == OP_INTERP
    assert checked > 1000 and n_interp[0] > 50


def test_interpolated_children_average_to_the_coarse_cell_and_add_no_extrema(rng):
    m = 4
    f = amr_forest()
    o = OracleForest3(f, m)
    rec = o.ghost_table()
    q = rng.standard_normal((f.num_patches, m, m, m))
    pad = o.ghost_fill(o.pad(q))
    ring = [(i, j, k) for k in range(-1, m + 3) for j in range(-1, m + 3) for i in range(-1, m + 3)
            if not (1 <= i <= m and 1 <= j <= m and 1 <= k <= m)]
    groups = {}
    for p in range(f.num_patches):
        for r, (i, j, k) in enumerate(ring):
            if rec[p, r, 0] == OP_INTERP:
                key = (p, *rec[p, r, 1:5])
                groups.setdefault(key, []).append(pad[p, k + 1, j + 1, i + 1])
    full = 0
    for (p, src, I, J, K), vals in groups.items():
        c = pad[src]
        qc = c[K + 1, J + 1, I + 1]
        nb = [c[K + 1, J + 1, I], c[K + 1, J + 1, I + 2], c[K + 1, J, I + 1], c[K + 1, J + 2, I + 1],
              c[K, J + 1, I + 1], c[K + 2, J + 1, I + 1], qc]
        assert min(vals) >= min(nb) - 1e-15 and max(vals) <= max(nb) + 1e-15
        if len(vals) == 8:
            full += 1
            assert abs(np.mean(vals) - qc) <= 4e-16 * max(1.0, abs(qc)) * 8
    assert full > 20


# ---- the split step ------------------------------------------------------------------------------------
def test_constant_state_is_a_fixed_point():
    m = 4
    f = amr_forest()
    q0 = np.full((f.num_patches, m, m, m), 0.75)
    q, c = run3(f, m, q0, (0.9, -0.4, 0.3), 0.02, 3)
    np.testing.assert_array_equal(q, q0)
    assert np.allclose(c, 0.02 * (4 * m) * 0.9, rtol=1e-15, atol=0)   # finest level 2: dx = 1 / (4 m)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_one_axis_data_reduce_to_the_1d_code(rng, axis):
    """Data varying along one axis only: the other two sweeps see no jump; the result is LeVeque's
    1D wave propagation (the independent numpy code) along every pencil, whatever the other
    velocity components."""
    m = 4
    dims = (2, 1, 1) if axis == 0 else ((1, 2, 1) if axis == 1 else (1, 1, 2))
    f = forest3(dims, 1)
    N = 2 * m * 2
    prof = rng.uniform(0.0, 1.0, N)
    shape = [1, 1, 1]
    shape[2 - axis] = N
    Gs = [N if d == 2 else 2 * m for d in dims]
    G = np.broadcast_to(prof.reshape(shape), tuple(reversed(Gs))).copy()
    vel = [0.4, -0.7, 0.55]
    vel[axis] = -0.8
    dx = 1.0 / (2 * m)
    dt = 0.9 * dx / 0.8
    q, c = run3(f, m, scatter(f, m, G), vel, dt, 1)
    ring = np.concatenate([prof[-2:], prof, prof[:2]])[None, :]
    q1, _ = red1d.wave_prop_1d("adv", ring, dt, dx, u=vel[axis])
    got = assemble(f, m, q)
    got = np.moveaxis(got, 2 - axis, -1).reshape(-1, N)
    for row in got:
        assert np.abs(row - q1[0]).max() <= 1e-14 * np.abs(prof).max()
    assert abs(c[0] - dt / dx * 0.8) <= 1e-15


@pytest.mark.parametrize("method2", [1, 2])
def test_courant_one_shifts_by_one_cell_in_each_direction(rng, method2):
    m = 4
    f = forest3((2, 2, 1), 1)
    G = rng.integers(0, 256, (2 * m, 4 * m, 4 * m)).astype(float)
    dx = 1.0 / (2 * m)
    q, c = run3(f, m, scatter(f, m, G), (1.0, 1.0, 1.0), dx, 1, method2=method2)
    np.testing.assert_array_equal(assemble(f, m, q), np.roll(G, (1, 1, 1), axis=(0, 1, 2)))
    assert c[0] == 1.0


def test_conservation_on_a_periodic_uniform_forest(rng):
    m = 6
    f = forest3((1, 2, 1), 1)
    q0 = rng.uniform(0.0, 1.0, (f.num_patches, m, m, m))
    q, _ = run3(f, m, q0, (0.5, -0.3, 0.8), 0.8 / (2 * m) / 0.8, 8)
    assert abs(q.sum() - q0.sum()) <= 1e-14 * q0.sum() * 8


def test_affine_data_translate_exactly_across_coarse_fine_faces():
    """Lax-Wendroff-limited sweeps are exact on affine data and the c/f ghosts reproduce affine
    data, so one step shifts q(x) = a + b.x to q(x - u dt) exactly, away from the outflow faces."""
    m = 4
    f = amr_forest(dims=(2, 2, 2), periodic=(False, False, False))
    a = np.array([0.3, -0.9, 0.6, 1.4])
    cen = cell_centres(f, m)
    q0 = a[0] + a[1] * cen[:, 0] + a[2] * cen[:, 1] + a[3] * cen[:, 2]
    vel = np.array([0.7, -0.5, 0.4])
    dt = 0.4 / (4 * m)
    q, _ = run3(f, m, q0, vel, dt, 1)
    want = q0 - dt * (a[1] * vel[0] + a[2] * vel[1] + a[3] * vel[2])
    inner = np.ones(cen.shape[0:1] + cen.shape[2:], bool)
    for d in range(3):
        inner &= (cen[:, d] > 3.5 / (2 * m)) & (cen[:, d] < f.dims[d] - 3.5 / (2 * m))
    assert inner.sum() > 500
    assert np.abs(q[inner] - want[inner]).max() <= 1e-13
