"""The fused two-hop ring gather on AMR forests (plan_ring_amr in csrc/plan.cpp,
k_cg_avg / k_cg_interp in csrc/kernels.cu): the step gathers every ring cell itself -- copies from
the source cells, averages and limited interpolations from a computed-ghost buffer -- instead of
the ghost kernels writing the rings.  The computed values use the ghost kernels' arithmetic, so
the run is bitwise the ghost-kernel run (FC_FUSED_RING=0), and the oracle parity of the default
mode (tests/test_gpu_parity.py) covers it against the paper's definitions."""
import dataclasses

import numpy as np
import pytest

from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import SWE_ROE, Workload, c2, c3, c3_ic

from test_gpu_subcycle import amr_euler, three_levels

pytestmark = pytest.mark.gpu


def walled_amr_swe(steps=6):
    """C3 physics (reflecting walls) on a two-level forest: AMR next to physical boundaries."""
    f = F.forest_refined(F.walled_unit_square(F.WALL), 2, lambda t, x, y, h: (x < 0.5) & (y < 0.5))
    m = 8
    q = c3_ic(f, m, 0, f.num_patches)
    dt = 0.9 * (0.5 ** 3 / m) / np.sqrt(2.0)
    return Workload("walled_amr_swe", f, m, 3, 0, SWE_ROE, (1.0, 0.0), q, None, steps, dt, "cfl")


CASES = [(c2(steps=12), 2), (three_levels(), 2), (amr_euler(), 2), (walled_amr_swe(), None),
         (dataclasses.replace(c2(steps=8), reflux=1), 2)]


def run(w, monkeypatch, fused):
    monkeypatch.setenv("FC_FUSED_RING", "1" if fused else "0")
    f = fc.forest_for(w, 0)
    path = f.stats()["uniform_fast_path"]
    q, c, _ = fc.run(w, f=f)
    return q, c, path


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name + ("_reflux" if c[0].reflux else ""))
def test_fused_amr_gather_bitwise_equals_ghost_kernels(case, monkeypatch):
    w, want = case
    qa, ca, pa = run(w, monkeypatch, True)
    qb, cb, pb = run(w, monkeypatch, False)
    assert pb == 0
    if want is not None:
        assert pa == want, pa
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


def test_fused_amr_gather_in_cuda_graph_runs(monkeypatch):
    """fc_run replays the computed-ghost kernels inside its graphs: bitwise fc_step in a loop."""
    w = three_levels(steps=10)
    monkeypatch.setenv("FC_FUSED_RING", "1")
    f = fc.forest_for(w, 0)
    f.set_q(np.ascontiguousarray(w.q0))
    f.run(w.dt0, w.steps)
    qa = f.get_q()
    f.close()
    g = fc.forest_for(w, 0)
    g.set_q(np.ascontiguousarray(w.q0))
    for _ in range(w.steps):
        g.step(w.dt0)
    np.testing.assert_array_equal(qa, g.get_q())
    g.close()


@pytest.mark.parametrize("w", [dataclasses.replace(c2(steps=6), reflux=1), three_levels(steps=4)],
                         ids=lambda w: w.name)
def test_fused_amr_gather_in_subcycled_steps(w, monkeypatch):
    """Sub-cycling on one rank uses the fused gather too (computed ghosts from each level's
    snapshot, no ring writes): bitwise the ghost-kernel sub-cycled run."""
    monkeypatch.setenv("FC_FUSED_RING", "1")
    qa, ca, _ = fc.run_subcycled(w)
    monkeypatch.setenv("FC_FUSED_RING", "0")
    qb, cb, _ = fc.run_subcycled(w)
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


@pytest.mark.parametrize("w", [c3(level=2, m=32, steps=10), c3(level=1, m=20, steps=10)],
                         ids=lambda w: w.name)
def test_fused_gather_on_multi_tile_patches(w, monkeypatch):
    """Uniform forests with m = tiles x T (m = 32: 2 x 2 tiles of 16; m = 20: 5 x 5 of 4), walls:
    each tile's window takes its interior part by row copies and its ring part from the sources
    (gather_ring_tiles, wall ghosts in shared memory) -- bitwise the ghost-kernel run of the same
    (phased) kernel.  (FC_WS=0: the warp-sweep kernel's own gather is checked below.)"""
    monkeypatch.setenv("FC_WS", "0")
    qa, ca, pa = run(w, monkeypatch, True)
    qb, cb, pb = run(w, monkeypatch, False)
    assert pa == 1 and pb == 0
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


@pytest.mark.parametrize("uniform", [False, True], ids=["band", "uniform"])
def test_fused_gather_capacity_form_on_the_cubed_sphere(uniform, monkeypatch):
    """The capacity form (C4 physics) on the cubed sphere takes the fused path: its CORNER3 ghosts
    at the 8 cube vertices are computed ghosts (the mean of two face ghosts' sources) -- bitwise the
    ghost-kernel run, AMR band and uniform sphere."""
    from workloads.cubed_sphere import c4_workload
    w = c4_workload(base_level=2, m=16, steps=12, uniform=uniform) if uniform else c4_workload(base_level=2, m=16, steps=12)
    qa, ca, pa = run(w, monkeypatch, True)
    qb, cb, pb = run(w, monkeypatch, False)
    assert pa == 2 and pb == 0
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


@pytest.mark.parametrize("w", [c3(level=2, m=32, steps=10), c3(level=3, m=16, steps=10)], ids=lambda w: w.name)
def test_warp_sweep_gather_matches_ghost_kernel_run(w, monkeypatch):
    """The warp-sweep systems kernel (step_ws.cu) gathers its windows itself (cp.async from the
    neighbours' interiors, wall ghosts in shared memory; m = 32: 2 x 2 tiles).  Against the phased
    kernel on ghost-kernel rings: the same method in another operation order, so agreement to
    rounding (1e-13 relative), and both within the oracle's tolerance (tests/test_gpu_parity.py)."""
    monkeypatch.delenv("FC_WS", raising=False)
    qa, ca, pa = run(w, monkeypatch, True)
    monkeypatch.setenv("FC_WS", "0")
    qb, cb, pb = run(w, monkeypatch, False)
    assert pa == 1 and pb == 0
    for k in range(w.meqn):
        scale = np.abs(qb[:, k]).max()
        assert np.abs(qa[:, k] - qb[:, k]).max() <= 1e-13 * scale, k
    np.testing.assert_allclose(ca, cb, rtol=1e-13, atol=0)
