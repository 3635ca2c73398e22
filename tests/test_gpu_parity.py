"""GPU parity: the CUDA path (libfc.so through its C ABI) against the oracle on the same seeded
inputs.  Bars (BASELINE.json north_star):
  * ghost rings and index tables: bit-exact;
  * state after the configured number of steps: max|dq_k| <= 1e-12 max|q_k| per component;
  * total mass: relative difference <= 1e-13; returned CFLs: relative <= 1e-12;
  * special cases (constant state, exact CFL-1 shifts): bitwise.
"""
import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads import forests as F
from workloads.configs import ADV_CONST, Workload, c1, c2, c3, c5

pytestmark = pytest.mark.gpu


def gpu_forest(w):
    return fc.forest_for(w, device=0)


def assert_parity(w, qg, qo, cg, co, mass_rtol=1e-13):
    for k in range(w.meqn):
        scale = np.abs(qo[:, k]).max()
        if scale == 0.0:
            scale = np.abs(qo).max()
        err = np.abs(qg[:, k] - qo[:, k]).max()
        assert err <= 1e-12 * scale, (w.name, k, err, scale)
        area = np.ldexp(1.0, -2 * w.forest.levels.astype(np.int64))[:, None, None]
        mg, mo = (qg[:, k] * area).sum(), (qo[:, k] * area).sum()
        assert abs(mg - mo) <= mass_rtol * max(abs(mo), (np.abs(qo[:, k]) * area).sum()), (w.name, k)
    np.testing.assert_allclose(cg, co, rtol=1e-12, atol=0)


# ---- ghost fill ---------------------------------------------------------------------------------
from workloads.cubed_sphere import c4_workload


def _ring_cases():
    rng = np.random.default_rng(1308147 + 11)
    out = [c1(), c2(), c3(level=2, m=8), c3(level=1, m=32), c5(level=2, m=16),
           c4_workload(base_level=2, m=8), c4_workload(base_level=2, m=8, uniform=True)]
    for name, conn in (("walls", F.walled_unit_square(F.WALL)), ("brick", F.brick(3, 2, bc=F.OUTFLOW)),
                       ("reversed", F.brick(2, 1, bc=F.OUTFLOW, reversed_x_links=(0,))),
                       ("periodic", F.periodic_unit_square())):
        fr = F.forest_refined(conn, 2, lambda t, x, y, h: rng.random(len(x)) < 0.4)
        meqn = 3 if name == "walls" else 1
        kind = 2 if meqn == 3 else ADV_CONST
        q0 = np.zeros((fr.num_patches, meqn, 8, 8))
        out.append(Workload(f"rand_{name}", fr, 8, meqn, 0, kind, (1.0, 0.5), q0, None, 1, 1e-3, "fixed"))
    return out


@pytest.mark.parametrize("w", _ring_cases(), ids=lambda w: w.name)
def test_ghost_rings_bitwise(w, rng):
    q = rng.standard_normal(w.q0.shape)
    if w.meqn >= 3:
        q[:, 0] = np.abs(q[:, 0]) + 1.0
    f = gpu_forest(w)
    f.set_q(np.ascontiguousarray(q))
    f.ghost_fill()
    g = f.get_q_padded()
    of = oracle.forest_for(w)
    o = of.ghost_fill(of.pad(q))
    np.testing.assert_array_equal(g, o)
    np.testing.assert_array_equal(f.ghost_table(), of.ghost_table())


# ---- full runs vs the oracle ----------------------------------------------------------------------
RUNS = [c1(), c2(), c3(level=3, m=32), c5(level=3, m=16), c5(level=2, m=8),
        c4_workload(base_level=2, m=16, steps=100), c4_workload(base_level=2, m=8, uniform=True, steps=60),
        c1(level=2, m=24, steps=30), c1(level=1, m=20, steps=30), c1(level=1, m=6, steps=30),
        c1(level=0, m=16, steps=30), c1(level=3, m=4, steps=30), c5(level=0, m=8, steps=30)]


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", RUNS, ids=lambda w: w.name)
def test_parity_against_oracle(w, skip):
    qo, co, do = oracle.run(w)
    qg, cg, dg = fc.run(w, dt_list=do, skip_quiescent=skip)
    assert_parity(w, qg, qo, cg, co)


VARIANTS = [(1, 2, oracle.LIM_MC), (2, 1, oracle.LIM_MC), (2, 0, oracle.LIM_MC),
            (2, 2, oracle.LIM_MINMOD), (2, 2, oracle.LIM_NONE)]


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: f"m2_{v[0]}_m3_{v[1]}_lim{v[2]}")
@pytest.mark.parametrize("w", [c5(level=2, m=16, steps=20), c3(level=1, m=32, steps=20), c2(steps=20),
                               c4_workload(base_level=1, m=16, steps=20)], ids=lambda w: w.name)
def test_parity_method_variants(w, variant):
    """method2 = 1 (no F~), method3 = 1 (transverse of A-+dq alone) / 0 (none), minmod and no
    limiter: every variant of the update (SURVEY §8(b) fc_set_problem) against the
    oracle, full update and quiescent shortcut."""
    import dataclasses
    w = dataclasses.replace(w, method2=variant[0], method3=variant[1], limiter=variant[2])
    if variant[1] == 0:   # without transverse terms the unsplit scheme is stable only to CFL 1/2
        w = dataclasses.replace(w, dt0=0.5 * w.dt0, cfl_target=0.45)
    qo, co, do = oracle.run(w)
    for skip in (0, 1):
        qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
        assert_parity(w, qg, qo, cg, co)


@pytest.mark.parametrize("w", [c5(level=3, m=16, steps=40), c3(level=2, m=32, steps=40),
                               c4_workload(base_level=2, m=16, steps=40)], ids=lambda w: w.name)
def test_quiescent_shortcut_is_exact(w):
    """The quiescent-tile shortcut (uniform staged window -> q_new = q, CFL from the state) gives
    bitwise the same state as the full update, and the same CFLs up to rounding."""
    _, _, do = oracle.run(w, steps=w.steps)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=1)
    q0, c0_, _ = fc.run(w, dt_list=do, skip_quiescent=0)
    np.testing.assert_array_equal(q1, q0)
    np.testing.assert_allclose(c1_, c0_, rtol=1e-14, atol=0)


@pytest.mark.parametrize("w", [c5(level=3, m=16, steps=40), c5(level=4, m=16, steps=30), c3(level=2, m=32, steps=40)],
                         ids=lambda w: w.name)
def test_quiescent_shortcut_follows_the_same_dt_sequence(w):
    """under the workload's own variable-dt policy (no replayed dt list) the shortcut
    and the full update must take the same dt decisions -- a quiescent window's CFL is computed
    with the full update's own Roe arithmetic (step_ws.cuh, ws_quiescent_cfl), so the CFLs, hence
    the dt sequence and the states, are bitwise equal.  (C5 L4: 1024 patches, the copy / activity
    filter path; the others: the in-kernel uniform-window check.)"""
    q1, c1_, d1 = fc.run(w, skip_quiescent=1)
    q0, c0_, d0 = fc.run(w, skip_quiescent=0)
    np.testing.assert_array_equal(c1_, c0_)
    np.testing.assert_array_equal(d1, d0)
    np.testing.assert_array_equal(q1, q0)


def test_parity_c2_levels_and_dt_policy_on_gpu():
    """C2 with the GPU driving its own dt policy (fixed dt) equals the oracle's run."""
    w = c2()
    qo, co, do = oracle.run(w)
    qg, cg, dg = fc.run(w)
    np.testing.assert_array_equal(dg, do)
    assert_parity(w, qg, qo, cg, co)


# ---- exact cases -------------------------------------------------------------------------------
@pytest.mark.parametrize("uv", [(1, 0), (0, -1), (1, 1), (-1, 1)])
@pytest.mark.parametrize("method2", [1, 2])
def test_exact_cfl1_shift_bitwise(rng, uv, method2):
    fr = F.forest_uniform(F.brick(2, 1, periodic_x=True, periodic_y=True), 2)
    m = 8
    G = rng.integers(0, 256, size=(1, 32, 64)).astype(np.float64)
    q0 = np.zeros((fr.num_patches, 1, m, m))
    for p in range(fr.num_patches):
        t, x0, y0 = int(fr.tree_ids[p]), int(fr.ix[p]) * m, int(fr.iy[p]) * m
        q0[p, 0] = G[0, y0:y0 + m, t * 32 + x0:t * 32 + x0 + m]
    w = Workload("shift", fr, m, 1, 0, ADV_CONST, (float(uv[0]), float(uv[1])), q0, None, 3,
                 1.0 / 32, "fixed", method2=method2)
    qg, cg, _ = fc.run(w)
    expect = np.roll(G, shift=(3 * uv[1], 3 * uv[0]), axis=(1, 2))
    for p in range(fr.num_patches):
        t, x0, y0 = int(fr.tree_ids[p]), int(fr.ix[p]) * m, int(fr.iy[p]) * m
        np.testing.assert_array_equal(qg[p, 0], expect[0, y0:y0 + m, t * 32 + x0:t * 32 + x0 + m])
    assert (cg == 1.0).all()


def test_constant_state_bitwise():
    w = c5(level=2, m=16)
    rho, u, v, p = 1.2, 0.7, -0.3, 2.0
    w.q0[:, 0], w.q0[:, 1], w.q0[:, 2] = rho, rho * u, rho * v
    w.q0[:, 3] = p / 0.4 + 0.5 * rho * (u * u + v * v)
    qg, _, _ = fc.run(w, steps=3)
    np.testing.assert_array_equal(qg, w.q0)


# ---- step acceptance / errors ----------------------------------------------------------------------
def test_cfl_reject_keeps_state_and_errors():
    w = c1()
    f = gpu_forest(w)
    f.set_q(np.ascontiguousarray(w.q0))
    rc, cfl = f.step(10 * w.dt0, raise_on_reject=False)
    assert rc == fc.FC_ECFL and cfl == pytest.approx(9.0, rel=1e-12)
    np.testing.assert_array_equal(f.get_q(), w.q0)
    with pytest.raises(fc.FcError) as ei:
        f.step(-1.0)
    assert ei.value.code == fc.FC_EINVAL
    bad = w.q0.copy()
    bad[3, 0, 2, 2] = np.nan
    f.set_q(np.ascontiguousarray(bad))
    with pytest.raises(fc.FcError) as ei:
        f.step(w.dt0)
    assert ei.value.code == fc.FC_ENONFINITE


def test_device_pointers_roundtrip():
    import torch
    w = c3(level=2, m=8)
    f = gpu_forest(w)
    qd = torch.from_numpy(np.ascontiguousarray(w.q0)).cuda()
    f.set_q(qd)
    out = torch.empty_like(qd)
    f.get_q(out)
    assert torch.equal(out.cpu(), torch.from_numpy(w.q0))


# ---- full-size launch configuration, sampled -------------------------------------------------------
def _sample_ids(w, rng, extra):
    P = w.num_patches
    ids = set(rng.choice(P, size=min(P, 96), replace=False).tolist())
    ids.update(extra)
    return np.array(sorted(i for i in ids if 0 <= i < P), np.int64)


@pytest.mark.parametrize("name", ["C5", "C3", "C4"])
def test_full_size_first_step_sampled(name, rng):
    """BASELINE.json's full sizes in the launch configuration bench.py times: one step from the IC
    on the GPU, checked on sampled patches (random + shock/bubble/wall-adjacent ones) against
    the oracle's per-patch step built from the same IC."""
    w = {"C5": c5, "C3": c3, "C4": c4_workload}[name]()
    f = gpu_forest(w)
    f.set_q(np.ascontiguousarray(w.q0))
    rc, cfl = f.step(w.dt0)
    qg = f.get_q()
    x0, y0, h = w.forest.origin()
    X = x0 + w.forest.tree_ids
    if name == "C5":
        extra = np.nonzero((np.abs(X + h / 2 - 1.29) < 0.01) | (np.abs(X + h / 2 - 1.3) < 0.02) |
                           (y0 == 0) | (x0 + h >= 1.0 - 1e-12))[0][:64]
    elif name == "C4":   # patches at tree corners / faces and at level jumps
        corner = ((x0 == 0) | (x0 + h >= 1 - 1e-12)) & ((y0 == 0) | (y0 + h >= 1 - 1e-12))
        extra = np.concatenate([np.nonzero(corner)[0], np.nonzero(np.diff(w.forest.levels) != 0)[0][:40]])
    else:
        extra = np.nonzero((x0 == 0) | (y0 == 0) | (np.abs(np.hypot(x0 + h / 2 - 0.5, y0 + h / 2 - 0.5) - 0.2) < 0.03))[0][:64]
    ids = _sample_ids(w, rng, extra.tolist())
    of = oracle.forest_for(w)
    qo, co = of.step_sample(oracle.problem_for(w), w.q0, w.dt0, 1.0 / w.m, ids, aux=w.aux)
    for k in range(w.meqn):
        scale = max(np.abs(qo[:, k]).max(), 1e-300)
        err = np.abs(qg[ids, k] - qo[:, k]).max()
        assert err <= 1e-12 * max(scale, np.abs(qo).max() if scale == 1e-300 else scale), (k, err)
    assert cfl >= co.max() * (1 - 1e-12) and cfl <= 1.0


def test_zero_velocity_is_a_fixed_point():
    """Degenerate advection u = v = 0: no wave moves, the state is unchanged bitwise and every CFL
    is 0 (both kernels: constant velocity and capacity form with zero edge velocities)."""
    import dataclasses
    from workloads.cubed_sphere import c4_workload
    w = dataclasses.replace(c2(steps=5), params=(0.0, 0.0))
    q, c, _ = fc.run(w)
    np.testing.assert_array_equal(q, w.q0)
    assert (c == 0.0).all()
    s = c4_workload(base_level=1, m=8, steps=3)
    s.aux[:, 1:] = 0.0
    q, c, _ = fc.run(s)
    np.testing.assert_array_equal(q, s.q0)
    assert (c == 0.0).all()


@pytest.mark.parametrize("uv", [(-0.7, 0.45), (0.3, -0.9), (-0.6, -0.8)])
@pytest.mark.parametrize("m", [8, 16])
@pytest.mark.parametrize("reflux", [0, 1])
def test_constant_velocity_signs_against_oracle(uv, m, reflux):
    """The register-sweep kernel is instantiated per sign of (u, v): every sign combination on an AMR
    forest (C2 rule) at m = 8 and 16, with and without the reflux records, both update modes."""
    import dataclasses
    w = dataclasses.replace(c2(base_level=2, m=m, steps=12), params=uv, reflux=reflux)
    qo, co, do = oracle.run(w)
    for skip in (1, 0):
        qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
        assert_parity(w, qg, qo, cg, co)


@pytest.mark.parametrize("w", [c5(level=1, m=4, steps=10), c5(level=1, m=12, steps=10), c5(level=0, m=24, steps=10),
                               c3(level=1, m=6, steps=10), c3(level=1, m=20, steps=10)], ids=lambda w: w.name)
def test_systems_ragged_tilings_against_oracle(w):
    """Systems on patch sizes that tile as 4 x 4 (m = 4), 3 x 3 tiles of 4 (m = 12), 3 x 3 of 8
    (m = 24), 3 x 3 of 2 (m = 6) and 5 x 5 of 4 (m = 20), with walls (SWE) and outflow (Euler):
    both update modes against the oracle."""
    qo, co, do = oracle.run(w)
    for skip in (1, 0):
        qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
        assert_parity(w, qg, qo, cg, co)


@pytest.mark.parametrize("bc", ["outflow", "wall"])
@pytest.mark.parametrize("m", [8, 16])
def test_constant_velocity_physical_boundaries_against_oracle(bc, m):
    """The register-sweep kernel's physical-boundary ghosts on the fused path (ring BC codes applied
    in shared memory, uniform forests) and on the AMR fused path: outflow and (scalar) wall
    boundaries, a uniform and a refined forest, both modes, against the oracle."""
    conn = F.brick(2, 1, bc=F.OUTFLOW) if bc == "outflow" else F.walled_unit_square(F.WALL)
    for fr in (F.forest_uniform(conn, 2),
               F.forest_refined(conn, 2, lambda t, x, y, h: (x + t - 0.6) ** 2 + (y - 0.5) ** 2 < 0.1)):
        X, Y = F.cell_centres(fr, m)
        X = X + fr.tree_ids[:, None, None]
        q0 = np.exp(-20.0 * ((X - 0.45) ** 2 + (Y - 0.4) ** 2))[:, None]
        dt = 0.8 * (0.5 ** int(fr.levels.max()) / m) / 1.0
        w = Workload(f"bc_{bc}_m{m}", fr, m, 1, 0, ADV_CONST, (0.9, -0.6), q0, None, 12, dt, "fixed")
        qo, co, do = oracle.run(w)
        for skip in (1, 0):
            qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
            assert_parity(w, qg, qo, cg, co, mass_rtol=1.0)   # (outflow: mass leaves the domain)


def _amr_euler_m16(steps=10):
    import dataclasses as _dc
    import sys as _sys
    import os as _os
    _sys.path.insert(0, _os.path.dirname(__file__))
    from test_gpu_subcycle import amr_euler
    from workloads import forests as _F
    from workloads.configs import EULER_ROE
    r = np.random.default_rng(1308147 + 77)
    fr = _F.forest_refined(_F.brick(2, 1, periodic_x=True, periodic_y=True), 1, lambda t, x, y, h: r.random(len(x)) < 0.5)
    m = 16
    X, Y = _F.cell_centres(fr, m)
    X = X + fr.tree_ids[:, None, None]
    rho = 1.0 + 0.5 * np.exp(-20 * ((X - 1.0) ** 2 + (Y - 0.5) ** 2))
    u, v, p = 0.3 + 0 * X, -0.2 + 0 * X, 1.0 + 0.3 * np.sin(2 * np.pi * X)
    g = 1.4
    q0 = np.stack([rho, rho * u, rho * v, p / (g - 1) + 0.5 * rho * (u * u + v * v)], 1)
    return Workload("amr_euler_m16", fr, m, 4, 0, EULER_ROE, (g, 1.0), q0, None, steps, 1e-3, "cfl")


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("w", [_amr_euler_m16(), c3(level=1, m=48, steps=20)], ids=lambda w: w.name)
def test_warp_sweep_kernel_on_amr_and_3x3_tiles(w, skip):
    """The warp-sweep kernel with the fused two-hop AMR gather (computed ghosts: ring owner code
    255) on an m = 16 AMR Euler brick, and on m = 48 patches (3 x 3 tiles of 16), against the
    oracle."""
    qo, co, do = oracle.run(w)
    f = gpu_forest(w)
    if w.name.startswith("amr"):
        assert f.stats()["uniform_fast_path"] == 2
    qg, cg, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
    assert_parity(w, qg, qo, cg, co)
