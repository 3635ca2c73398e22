"""GPU parity of the Euler HLLE solver (FC_EULER_HLLE, solvers.cuh EulerHlle)
against the oracle's rp_hlle (pinned in tests/test_oracle_hlle.py): C5's shock-bubble physics on
small uniform forests and an AMR brick (fused AMR gather), both update modes, the dt policy
replayed; the quiescent shortcut bitwise equal to the full update; Sod's tube (1D) kept
y-independent on the GPU."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads.configs import EULER_HLLE, c5

from test_gpu_parity import assert_parity
from test_gpu_subcycle import amr_euler
from test_oracle_hlle import sod_workload

pytestmark = pytest.mark.gpu


def hlle(w):
    return dataclasses.replace(w, kind=EULER_HLLE, params=(w.params[0], 0.0), name=w.name + "_hlle")


RUNS = [hlle(c5(level=2, m=16, steps=20)), hlle(c5(level=3, m=8, steps=20)), hlle(amr_euler(steps=10)),
        sod_workload(2)[0]]


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", RUNS, ids=lambda w: w.name)
def test_hlle_parity_against_oracle(w, skip):
    qo, co, do = oracle.run(w)
    qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
    assert_parity(w, qg, qo, cg, co)


def test_hlle_quiescent_shortcut_is_exact():
    w = hlle(c5(level=3, m=16, steps=30))
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=1)
    q0, c0_, _ = fc.run(w, dt_list=do, skip_quiescent=0)
    np.testing.assert_array_equal(q1, q0)
    np.testing.assert_allclose(c1_, c0_, rtol=1e-14, atol=0)


def test_hlle_sod_stays_one_dimensional():
    w, _ = sod_workload(3)
    q, _, _ = fc.run(w)
    assert np.ptp(q[:, 0], axis=1).max() < 1e-12
