"""the oracle's optional OpenMP loop over patches (orc_step) must be bitwise
identical to one thread -- each patch's update reads only q_old and writes only its own cells, and
the CFL max is order-independent.  Checked on small versions of C1-C5 and an AMR Euler forest."""
import numpy as np
import pytest

import oracle
from workloads.configs import c1, c2, c3, c5
from workloads.cubed_sphere import c4_workload

CASES = [c1(steps=5), c2(steps=5), c3(level=2, m=8, steps=5), c4_workload(base_level=1, m=8, steps=5),
         c5(level=2, m=8, steps=5)]


@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name)
def test_openmp_bitwise_equal_to_one_thread(w):
    q1, c1_, d1 = oracle.run(w, nthreads=1)
    q4, c4_, d4 = oracle.run(w, nthreads=4)
    np.testing.assert_array_equal(q1, q4)
    np.testing.assert_array_equal(c1_, c4_)
    np.testing.assert_array_equal(d1, d4)
