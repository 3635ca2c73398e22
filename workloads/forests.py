"""Forest-of-quadtrees inputs: leaf lists in Morton (z-) order and tree connectivities.

Conventions (PAPER.md:131-146 [§2], PAPER.md:240-245 [§4]):
  * faces of a tree: 0 = -x, 1 = +x, 2 = -y, 3 = +y;
  * tree_to_tree[4t+f] = neighbour tree across face f of tree t,
    tree_to_face[4t+f] = nf + 4*reversed (nf = the neighbour's face, reversed = the two faces'
    tangential coordinates increase in opposite directions along the shared edge);
    a face linked to itself (same tree, same face) is a physical boundary;
  * face_bc[4t+f] = 0 (OUTFLOW) or 1 (WALL), only meaningful on physical faces;
  * leaves are listed tree by tree (trees ascending), z-order inside a tree with the
    child order SW, SE, NW, NE (x provides the even Morton bits).

The leaf lists are produced by recursive z-order enumeration; their Morton *decoding* is part
of the method (table build) and lives in the oracle / libfc, not here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

OUTFLOW = 0
WALL = 1


@dataclass
class Connectivity:
    tree_to_tree: np.ndarray  # int32 [4T]
    tree_to_face: np.ndarray  # int8  [4T]
    face_bc: np.ndarray       # int8  [4T]

    @property
    def num_trees(self) -> int:
        return len(self.tree_to_tree) // 4


@dataclass
class Forest:
    levels: np.ndarray      # int8  [P]
    tree_ids: np.ndarray    # int32 [P]
    ix: np.ndarray          # int64 [P] x origin in units of the leaf's own size (generator-side only)
    iy: np.ndarray          # int64 [P]
    conn: Connectivity
    meta: dict = field(default_factory=dict)

    @property
    def num_patches(self) -> int:
        return len(self.levels)

    def origin(self):
        """Leaf origin (x0, y0) and edge length h in tree coordinates (tree = unit square)."""
        h = np.ldexp(1.0, -self.levels.astype(np.int64))
        return self.ix * h, self.iy * h, h


def _conn(t2t, t2f, bc) -> Connectivity:
    return Connectivity(np.asarray(t2t, np.int32), np.asarray(t2f, np.int8), np.asarray(bc, np.int8))


def periodic_unit_square() -> Connectivity:
    """One tree whose -x face is linked to its own +x face and -y to +y (aligned)."""
    return _conn([0, 0, 0, 0], [1, 0, 3, 2], [OUTFLOW] * 4)


def walled_unit_square(bc: int = WALL) -> Connectivity:
    """One tree, all four faces physical with the given boundary kind."""
    return _conn([0, 0, 0, 0], [0, 1, 2, 3], [bc] * 4)


def brick(nx: int, ny: int, periodic_x: bool = False, periodic_y: bool = False,
          bc: int = OUTFLOW, reversed_x_links=()) -> Connectivity:
    """nx*ny trees on a lattice, tree t = tx + nx*ty covering [tx, tx+1] x [ty, ty+1].

    ``reversed_x_links`` lists tree ids t whose +x face link to t+1 is declared reversed
    (used only by the tiny 2-tree tests that reflect the second tree's frame)."""
    T = nx * ny
    t2t = np.zeros(4 * T, np.int32)
    t2f = np.zeros(4 * T, np.int8)
    fbc = np.full(4 * T, bc, np.int8)
    for ty in range(ny):
        for tx in range(nx):
            t = tx + nx * ty
            # -x
            if tx > 0 or periodic_x:
                t2t[4 * t + 0] = (tx - 1) % nx + nx * ty
                t2f[4 * t + 0] = 1
            else:
                t2t[4 * t + 0], t2f[4 * t + 0] = t, 0
            # +x
            if tx < nx - 1 or periodic_x:
                t2t[4 * t + 1] = (tx + 1) % nx + nx * ty
                t2f[4 * t + 1] = 0
            else:
                t2t[4 * t + 1], t2f[4 * t + 1] = t, 1
            # -y
            if ty > 0 or periodic_y:
                t2t[4 * t + 2] = tx + nx * ((ty - 1) % ny)
                t2f[4 * t + 2] = 3
            else:
                t2t[4 * t + 2], t2f[4 * t + 2] = t, 2
            # +y
            if ty < ny - 1 or periodic_y:
                t2t[4 * t + 3] = tx + nx * ((ty + 1) % ny)
                t2f[4 * t + 3] = 2
            else:
                t2t[4 * t + 3], t2f[4 * t + 3] = t, 3
    for t in reversed_x_links:
        t2f[4 * t + 1] |= 4
        t2f[4 * (t + 1) + 0] |= 4
    return _conn(t2t, t2f, fbc)


def zorder_coords(level: int):
    """(ix, iy) of the 4**level quadrants of one tree at `level`, in z-order (SW, SE, NW, NE
    recursively), built by repeated child expansion rather than bit interleaving."""
    ix = np.zeros(1, np.int64)
    iy = np.zeros(1, np.int64)
    cx = np.array([0, 1, 0, 1], np.int64)
    cy = np.array([0, 0, 1, 1], np.int64)
    for _ in range(level):
        ix = (2 * ix[:, None] + cx[None, :]).reshape(-1)
        iy = (2 * iy[:, None] + cy[None, :]).reshape(-1)
    return ix, iy


def forest_uniform(conn: Connectivity, level: int) -> Forest:
    T = conn.num_trees
    ix, iy = zorder_coords(level)
    n = len(ix)
    return Forest(levels=np.full(T * n, level, np.int8),
                  tree_ids=np.repeat(np.arange(T, dtype=np.int32), n),
                  ix=np.tile(ix, T), iy=np.tile(iy, T), conn=conn)


def forest_refined(conn: Connectivity, base_level: int, refine) -> Forest:
    """Every tree uniformly at `base_level`; a base quadrant (tree, ix, iy) for which
    ``refine(tree, x_centre, y_centre, h)`` is true is replaced by its 4 children (z-order).
    The predicate receives tree-coordinate centres (vectorised over one tree)."""
    bx, by = zorder_coords(base_level)
    h = 0.5 ** base_level
    lv, tr, ox, oy = [], [], [], []
    cx = np.array([0, 1, 0, 1], np.int64)
    cy = np.array([0, 0, 1, 1], np.int64)
    for t in range(conn.num_trees):
        flag = np.asarray(refine(t, (bx + 0.5) * h, (by + 0.5) * h, h), bool)
        # expand in z-order: each base leaf contributes 1 or 4 entries
        cnt = np.where(flag, 4, 1)
        idx = np.repeat(np.arange(len(bx)), cnt)
        # position inside the family (0..3) for refined ones
        start = np.cumsum(cnt) - cnt
        sub = np.arange(len(idx)) - np.repeat(start, cnt)
        f = flag[idx]
        lv.append(np.where(f, base_level + 1, base_level).astype(np.int8))
        tr.append(np.full(len(idx), t, np.int32))
        ox.append(np.where(f, 2 * bx[idx] + cx[sub % 4], bx[idx]))
        oy.append(np.where(f, 2 * by[idx] + cy[sub % 4], by[idx]))
    return Forest(levels=np.concatenate(lv), tree_ids=np.concatenate(tr),
                  ix=np.concatenate(ox), iy=np.concatenate(oy), conn=conn)


def cell_centres(forest: Forest, m: int, ghost: int = 0):
    """Tree-coordinate cell centres, arrays [P, m+2g, m+2g] ([patch][j][i], x fastest)."""
    x0, y0, h = forest.origin()
    dx = h / m
    k = np.arange(-ghost, m + ghost) + 0.5
    X = x0[:, None, None] + dx[:, None, None] * k[None, None, :]
    Y = y0[:, None, None] + dx[:, None, None] * k[None, :, None]
    X = np.broadcast_to(X, (len(x0), len(k), len(k)))
    Y = np.broadcast_to(Y, (len(x0), len(k), len(k)))
    return X, Y
