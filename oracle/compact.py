"""COMPACT ghost table (include/fc.h FC_TABLE_COMPACT) derived from the oracle's brute-force
per-cell ghost records (forest.c, orc_ghost_records: point location of every ghost-cell centre).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of the product planner: there the
table comes from one neighbour lookup per direction (PAPER.md:141-144 [§2]); here it is read back
from the geometry of the ring cells' sources --
  kind   the one ghost operation of the direction's ring cells (COPY: same level, INTERP: coarser,
         AVG4: finer, BCX / BCY: physical, CORNER3: cube corner);
  nbrs   the source patches of those cells (for a finer face, the source at the lowest tangential
         ring index first);
  xform  the image of one step along x and along y of the ring, as a displacement of the source
         positions (in quarter source cells: COPY centre 4 i - 2, AVG4 block centre 4 i, INTERP
         quadrant 4 i - 2 + sign);
  half   (coarser faces) the parity of the patch's own tangential position at its level.
"""
from __future__ import annotations

import numpy as np

from . import OP_AVG4, OP_BCX, OP_BCY, OP_COPY, OP_CORNER3, OP_INTERP

KIND = {OP_COPY: 0, OP_INTERP: 1, OP_AVG4: 2, OP_BCX: 3, OP_BCY: 3, OP_CORNER3: 4}


def ring_cells(m: int):
    """(i, j) of the ring cells in storage order (j = -1..m+2 outer, i inner, interior skipped)."""
    return [(i, j) for j in range(-1, m + 3) for i in range(-1, m + 3)
            if not (1 <= i <= m and 1 <= j <= m)]


def regions(m: int):
    """direction d -> the ring cells (i, j) of that face strip / corner block."""
    lo, hi, mid = (-1, 0), (m + 1, m + 2), range(1, m + 1)
    faces = [[(i, j) for j in mid for i in lo], [(i, j) for j in mid for i in hi],
             [(i, j) for j in lo for i in mid], [(i, j) for j in hi for i in mid]]
    corners = [[(i, j) for j in ys for i in xs] for ys, xs in ((lo, lo), (lo, hi), (hi, lo), (hi, hi))]
    return faces + corners


def _pos(rec):
    """source position of a COPY / AVG4 / INTERP record in quarter source cells"""
    op, si, sj, a, b = rec[0], rec[2], rec[3], rec[4], rec[5]
    if op == OP_COPY:
        return np.array([4 * si - 2, 4 * sj - 2])
    if op == OP_AVG4:
        return np.array([4 * si, 4 * sj])
    return np.array([4 * si - 2 + a, 4 * sj - 2 + b])


def _axis_code(v):
    """(axis, negative) of a displacement along one source axis"""
    assert (v[0] == 0) != (v[1] == 0), v
    return (0, v[0] < 0) if v[0] != 0 else (1, v[1] < 0)


def compact_table(of) -> np.ndarray:
    """[P][8][5] for an oracle.OracleForest."""
    m = of.m
    cells = ring_cells(m)
    index = {c: r for r, c in enumerate(cells)}
    regs = regions(m)
    x, y, lmax = of.coords()
    levels = np.asarray(of.levels)
    out = np.full((of.P, 8, 5), -1, np.int32)
    for p in range(of.P):
        rec = of.ghost_records(p)
        size = 1 << (lmax - int(levels[p]))
        for d, reg in enumerate(regs):
            rr = [rec[index[c]] for c in reg]
            ops = {int(r[0]) for r in rr}
            assert len(ops) == 1, (p, d, ops)
            op = ops.pop()
            e = out[p, d]
            e[0] = KIND[op]
            if e[0] >= 3:
                continue
            if op == OP_AVG4 and d < 4:     # finer face: sources along the face, lower first
                near = 0 if d in (0, 2) else 1
                strip = [c for c in reg if (c[0] if d < 2 else c[1]) == (0 if near == 0 else m + 1)]
                srcs = [int(rec[index[c]][1]) for c in strip]
                e[1], e[2] = srcs[0], srcs[-1]
                assert len(set(srcs)) == 2, (p, d, srcs)
            else:
                srcs = {int(r[1]) for r in rr}
                assert len(srcs) == 1, (p, d, srcs)
                e[1] = srcs.pop()
            (i0, j0) = reg[0]
            ex = _pos(rec[index[(i0 + 1, j0)]]) - _pos(rec[index[(i0, j0)]])
            ey = _pos(rec[index[(i0, j0 + 1)]]) - _pos(rec[index[(i0, j0)]])
            if op == OP_INTERP:   # a one-cell step of the fine ring is half a coarse cell: never 0
                pass
            ax, nx = _axis_code(ex)
            ay, ny = _axis_code(ey)
            assert ax != ay, (p, d, ex, ey)
            e[3] = 4 * ax + 2 * int(nx) + int(ny)
            if op == OP_INTERP and d < 4:
                tang = y[p] if d < 2 else x[p]
                e[4] = (tang // size) & 1
    return out
