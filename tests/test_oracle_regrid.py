"""Pins for the oracle's dynamic regrid (oracle/regrid.c; PAPER.md:148-155 [§2], 207-211 [§3];
SURVEY §8(f) #3).

Independent references: (1) conservation -- the limited interpolation has the parent as the mean
of its 4 children and the averaging is the mean, so sum q area is unchanged to rounding; (2) the
output forest tiles every tree (the oracle's own decoder accepts it) and is 2:1 balanced across
faces and corners, checked here by brute force over all pairs of touching leaves (periodic wrap
included); (3) a constant state stays exactly constant; (4) refining everything and coarsening it
back returns the original data to rounding; (5) every tagged patch is refined, untagged data is
never refined except to keep the balance, and a spike next to a coarser neighbour forces that
neighbour to refine (the balance ripple).
"""
import itertools

import numpy as np

import oracle
from workloads import forests as F
from workloads.configs import c1, c2


def regrid(w, q, rt, ct, minl, maxl):
    of = oracle.forest_for(w)
    qp = of.ghost_fill(of.pad(q))
    return of.regrid(qp, rt, ct, minl, maxl)


def area(levels, m):
    return np.ldexp(1.0, -2 * levels.astype(np.int64))[:, None, None] / (m * m)


def leaf_boxes(levels, trees, conn, m):
    of = oracle.OracleForest(levels, trees, conn, m)     # raises unless the leaves tile the trees
    x, y, lmax = of.coords()
    s = np.left_shift(1, lmax - levels.astype(np.int64))
    return x, y, s, 1 << lmax


def assert_balanced_periodic(levels, trees, conn, m):
    """single periodic tree: every two leaves whose closed squares touch (mod the period) differ
    by at most one level"""
    x, y, s, N = leaf_boxes(levels, trees, conn, m)

    def touch(a0, a1, b0, b1):
        return any(max(a0, b0 + k) <= min(a1, b1 + k) for k in (-N, 0, N))
    bad = 0
    for p, q in itertools.combinations(range(len(levels)), 2):
        if abs(int(levels[p]) - int(levels[q])) <= 1:
            continue
        if touch(x[p], x[p] + s[p], x[q], x[q] + s[q]) and touch(y[p], y[p] + s[p], y[q], y[q] + s[q]):
            bad += 1
    assert bad == 0


def test_regrid_conserves_mass_and_keeps_balance():
    w = c2(steps=1)
    nl, nt, q2, src = regrid(w, w.q0, 0.4, 0.01, 2, 5)
    assert (src[:, 0] == 2).any() and (src[:, 0] == 3).any()      # both refined and coarsened
    m0 = (w.q0[:, 0] * area(w.forest.levels, w.m)).sum()
    m1 = (q2[:, 0] * area(nl, w.m)).sum()
    assert abs(m1 - m0) <= 1e-14 * abs(m0)
    assert_balanced_periodic(nl, nt, w.forest.conn, w.m)
    oracle.OracleForest(nl, nt, w.forest.conn, w.m).ghost_table()   # ghost sources resolve (EBALANCE otherwise)


def test_constant_state_stays_constant_and_coarsens():
    w = c2(steps=1)
    q = np.full_like(w.q0, 0.37)
    nl, nt, q2, src = regrid(w, q, 0.05, 0.01, 2, 5)
    assert (q2 == 0.37).all()
    assert (src[:, 0] != 2).all()                                  # nothing refined (max - min = 0)
    assert len(nl) < len(w.forest.levels)                           # families coarsened


def test_refine_all_then_coarsen_all_round_trip(rng):
    w = c1(level=2, m=8)
    X, Y = F.cell_centres(w.forest, w.m)
    q = (np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y))[:, None]
    nl, nt, q2, src = regrid(w, q, -1.0, -1.0, 2, 3)
    assert (nl == 3).all() and len(nl) == 4 * len(w.forest.levels)
    w2 = c1(level=3, m=8)
    assert (w2.forest.levels == nl).all() and (w2.forest.tree_ids == nt).all()
    nl2, nt2, q3, _ = regrid(w2, q2, np.inf, np.inf, 2, 3)
    assert (nl2 == 2).all()
    np.testing.assert_allclose(q3, q, rtol=0, atol=1e-15 * np.abs(q).max())


def test_tagged_patches_refined_and_balance_ripple():
    """A spike in one level-4 patch of C2 that touches a level-3 patch: that patch is tagged and
    refined to level 5, which forces its level-3 neighbour to level 4 (2:1 balance); nothing else
    changes (thresholds above the smooth data's variation, no coarsening)."""
    w = c2(steps=1)
    lv = w.forest.levels
    of = oracle.forest_for(w)
    tab = of.ghost_table()
    # a level-4 patch with an INTERP ghost (a coarser neighbour)
    p = next(int(i) for i in range(len(lv)) if lv[i] == 4 and (tab[i, :, 0] == oracle.OP_INTERP).any())
    coarse_nbrs = set(int(tab[p, r, 1]) for r in range(tab.shape[1]) if tab[p, r, 0] == oracle.OP_INTERP)
    q = np.full_like(w.q0, 0.1)
    q[p, 0, 3, 3] = 1.0
    nl, nt, q2, src = regrid(w, q, 0.5, -1.0, 3, 6)
    refined = set(int(s[1]) for s in src if s[0] == 2)
    assert refined == {p} | coarse_nbrs and all(lv[r] == 3 for r in coarse_nbrs) and coarse_nbrs
    assert_balanced_periodic(nl, nt, w.forest.conn, w.m)
    m0 = (q[:, 0] * area(lv, w.m)).sum()
    assert abs((q2[:, 0] * area(nl, w.m)).sum() - m0) <= 1e-14 * m0
