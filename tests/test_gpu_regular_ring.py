"""Regular rings (plan_ring_regular in csrc/plan.cpp): a patch whose every ring cell is a copy of
the aligned cell of a same-level local neighbour has its fused-gather source addresses computed
from 9 neighbour block offsets (the scalar sweeps move the ring in 16-byte pairs) instead of
being read from the per-cell ring table.  The planner admits a patch only after checking every
computed address against the table, so the gathered windows -- and every state and CFL of a run
-- are bitwise those of the table path (FC_REGULAR_RING=0); the oracle parity of the default mode
(tests/test_gpu_parity.py, tests/test_gpu_full_size.py) covers both against the paper."""
import numpy as np
import pytest

from paper_1308_1472_b200 import fc
from workloads.configs import c1, c2, c3, c4, c5

from test_gpu_subcycle import amr_euler

pytestmark = pytest.mark.gpu


def run(w, monkeypatch, regular):
    monkeypatch.setenv("FC_REGULAR_RING", "1" if regular else "0")
    f = fc.forest_for(w, 0)
    st = f.stats()
    q, c, _ = fc.run(w, f=f)
    return q, c, st


def boundary_free(w):
    """patches of a uniform walled / outflow forest with no physical-boundary ring cell"""
    table = fc.forest_for(w, -1).ghost_table()   # host-only handle: (P, G, 8) records
    bc = np.isin(table[:, :, 0], (4, 5)).any(axis=1)   # BCX / BCY records (include/fc.h)
    return int((~bc).sum())


CASES = [
    ("C1_periodic_m8", c1(level=3, steps=8), "all"),
    ("C2_amr_m16", c2(steps=6), "some"),
    ("C3_walls_m32_tiles", c3(level=2, steps=4), "interior"),
    ("C4_cubed_sphere", c4(base_level=2, steps=4), "some"),
    ("C5_outflow_m16", c5(level=3, steps=4), "interior"),
    ("euler_amr", amr_euler(), "any"),   # (small: every patch next to a wall or a level change)
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_regular_ring_bitwise_equals_table_gather(case, monkeypatch):
    name, w, kind = case
    qa, ca, sa = run(w, monkeypatch, True)
    qb, cb, sb = run(w, monkeypatch, False)
    assert sb["regular_patches"] == 0
    P = w.forest.num_patches
    if kind == "all":
        assert sa["regular_patches"] == P
    elif kind == "interior":
        assert sa["regular_patches"] == boundary_free(w) > 0
    elif kind == "some":
        assert 0 < sa["regular_patches"] < P
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)
