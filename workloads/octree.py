"""Forests of octrees (3D) for the octree path (reading 26): aligned bricks of
Tx x Ty x Tz trees, each face periodic (a link to the opposite face) or outflow.  Input generation
only (leaf lists in Morton order, connectivity, initial states); no method arithmetic.

Morton order within a tree: x in bits 3k, y in 3k+1, z in 3k+2; children of an octant in z-order
(child c = (c & 1, (c >> 1) & 1, c >> 2)).  Trees in x-fastest order over the brick.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

OUTFLOW = 1


@dataclass
class Forest3:
    levels: np.ndarray          # int8 [P]
    tree_ids: np.ndarray        # int32 [P]
    t2t: np.ndarray             # int32 [6T]: tree across face f (-x, +x, -y, +y, -z, +z)
    fbc: np.ndarray             # int8 [6T]: 1 physical (outflow), 0 linked
    dims: tuple                 # (Tx, Ty, Tz)

    @property
    def num_patches(self):
        return len(self.levels)

    @property
    def num_trees(self):
        return int(np.prod(self.dims))


def brick_connectivity(dims, periodic=(True, True, True)):
    Tx, Ty, Tz = dims
    T = Tx * Ty * Tz
    t2t = np.zeros(6 * T, np.int32)
    fbc = np.zeros(6 * T, np.int8)
    for t in range(T):
        x, y, z = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        c = [x, y, z]
        for a, n in enumerate(dims):
            for side in (0, 1):
                f = 2 * a + side
                cc = list(c)
                cc[a] += 1 if side else -1
                if 0 <= cc[a] < n or periodic[a]:
                    cc[a] %= n
                    t2t[6 * t + f] = cc[0] + Tx * (cc[1] + Ty * cc[2])
                else:
                    t2t[6 * t + f] = t
                    fbc[6 * t + f] = OUTFLOW
    return t2t, fbc


def forest3(dims=(1, 1, 1), base: int = 1, refine=None, periodic=(True, True, True)) -> Forest3:
    """Leaves of level `base` in every tree, the ones with refine(t, x0, y0, z0, h) true (origin and
    size in tree units) split once more (two levels: 2:1 balanced by construction)."""
    lv, tr = [], []

    def rec(t, l, x0, y0, z0, h):
        split = l < base or (l == base and refine is not None and refine(t, x0, y0, z0, h))
        if not split:
            lv.append(l)
            tr.append(t)
            return
        hh = h / 2
        for c in range(8):
            rec(t, l + 1, x0 + (c & 1) * hh, y0 + ((c >> 1) & 1) * hh, z0 + (c >> 2) * hh, hh)

    T = int(np.prod(dims))
    for t in range(T):
        rec(t, 0, 0.0, 0.0, 0.0, 1.0)
    t2t, fbc = brick_connectivity(dims, periodic)
    return Forest3(np.array(lv, np.int8), np.array(tr, np.int32), t2t, fbc, tuple(dims))


def leaf_geometry(f: Forest3):
    """per leaf (tree, x0, y0, z0, h) in tree units: x0 etc. of the leaf's lower corner."""
    lmax = int(f.levels.max())
    geo = [None] * f.num_patches
    for t in range(f.num_trees):
        c = 0
        for p in np.nonzero(f.tree_ids == t)[0]:
            l = int(f.levels[p])
            size = 1 << (3 * (lmax - l))
            x = y = z = 0
            for b in range(lmax):
                x |= ((c >> (3 * b)) & 1) << b
                y |= ((c >> (3 * b + 1)) & 1) << b
                z |= ((c >> (3 * b + 2)) & 1) << b
            h = 2.0 ** -l
            geo[p] = (t, x / 2 ** lmax, y / 2 ** lmax, z / 2 ** lmax, h)
            c += size
    return geo


def cell_centres(f: Forest3, m: int):
    """global coordinates (brick units: tree edge 1) of every interior cell centre: [P][3][m][m][m]
    (index [p][:, k, j, i])."""
    geo = leaf_geometry(f)
    Tx, Ty, _ = f.dims
    out = np.zeros((f.num_patches, 3, m, m, m))
    ii = (np.arange(m) + 0.5) / m
    for p, (t, x0, y0, z0, h) in enumerate(geo):
        tx, ty, tz = t % Tx, (t // Tx) % Ty, t // (Tx * Ty)
        X = tx + x0 + h * ii
        Y = ty + y0 + h * ii
        Z = tz + z0 + h * ii
        out[p, 0] = X[None, None, :]
        out[p, 1] = Y[None, :, None]
        out[p, 2] = Z[:, None, None]
    return out
