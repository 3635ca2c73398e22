"""fc_run: fixed-dt multi-step runs replayed as CUDA graphs (no host round trip per step) give
bitwise the same states and CFLs as the same number of fc_step calls, for the fixed-dt configs
(C1, C2, C4) in both update modes and with the reflux; a run whose CFL exceeds the bound is undone."""
import dataclasses

import numpy as np
import pytest

from paper_1308_1472_b200 import fc
from workloads.configs import c1, c2
from workloads.cubed_sphere import c4_workload

pytestmark = pytest.mark.gpu

CASES = [c1(steps=30), c2(steps=30), dataclasses.replace(c2(steps=30), reflux=1),
         c4_workload(base_level=2, m=16, steps=30), c1(level=5, m=16, steps=20)]


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name + ("_reflux" if w.reflux else ""))
def test_run_equals_step_loop_bitwise(w, skip):
    qa, ca, _ = fc.run(w, skip_quiescent=skip)
    f = fc.forest_for(w, 0, skip_quiescent=skip)
    f.set_q(np.ascontiguousarray(w.q0))
    half = w.steps // 2
    rc1, c1_ = f.run(w.dt0, half)
    rc2, c2_ = f.run(w.dt0, w.steps - half)        # a second run continues from the first
    qb = f.get_q()
    np.testing.assert_array_equal(qb, qa)
    np.testing.assert_array_equal(np.concatenate([c1_, c2_]), ca)
    assert f.stats()["steps"] == w.steps


def test_run_rejected_is_undone():
    w = c1(steps=10)
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    rc, c = f.run(3.0 * w.dt0, 5, raise_on_reject=False)
    assert rc == fc.FC_ECFL and c.max() > 1.0
    np.testing.assert_array_equal(f.get_q(), w.q0)
    rc, c = f.run(w.dt0, 10)
    qa, ca, _ = fc.run(w)
    np.testing.assert_array_equal(f.get_q(), qa)


def test_run_after_set_problem_uses_the_new_problem():
    """fc_set_problem between two fc_run calls with the same dt: the second run must replay the
    new problem's kernels (limiter, transverse variant, skip mode), not the first run's graphs."""
    w = c2(steps=10)
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    f.run(w.dt0, 5)                                    # graphs captured for MC, method3 = 2
    q_mid = f.get_q()
    f.set_problem(w.kind, *w.params, limiter=fc.FC_LIM_MINMOD, method3=1, skip_quiescent=0)
    f.run(w.dt0, 5)
    q_run = f.get_q()
    g = fc.forest_for(w, 0)                            # reference: fc_step loop from the same state
    g.set_problem(w.kind, *w.params, limiter=fc.FC_LIM_MINMOD, method3=1, skip_quiescent=0)
    g.set_q(q_mid)
    for _ in range(5):
        g.step(w.dt0)
    np.testing.assert_array_equal(q_run, g.get_q())
