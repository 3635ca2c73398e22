"""Pins for the oracle's Riemann solvers and limiter (oracle/claw.c).

Independent references: SPEC worked examples (tests/golden), the PDE flux functions written out
here (f(q) of the shallow-water and Euler equations), their Jacobians (checked against central
finite differences of those fluxes in this file), and Roe's defining properties
(sum of waves = jump, sum of speed*wave = flux jump).
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
G_SWE, GAM = 1.0, 1.4


# ---- PDE fluxes (definitions) ----------------------------------------------------------------------
def swe_flux(q, d, g=G_SWE):
    h, hu, hv = q
    u, v = hu / h, hv / h
    if d == 1:
        return np.array([hu, hu * u + 0.5 * g * h * h, hu * v])
    return np.array([hv, hv * u, hv * v + 0.5 * g * h * h])


def euler_flux(q, d, gam=GAM):
    rho, ru, rv, E = q
    u, v = ru / rho, rv / rho
    p = (gam - 1.0) * (E - 0.5 * rho * (u * u + v * v))
    if d == 1:
        return np.array([ru, ru * u + p, ru * v, u * (E + p)])
    return np.array([rv, rv * u, rv * v + p, v * (E + p)])


def euler_jac_y(u, v, H, gam=GAM):
    k = 0.5 * (gam - 1.0) * (u * u + v * v)
    return np.array([[0.0, 0.0, 1.0, 0.0],
                     [-u * v, v, u, 0.0],
                     [k - v * v, -(gam - 1.0) * u, (3.0 - gam) * v, gam - 1.0],
                     [v * (k - H), -(gam - 1.0) * u * v, H - (gam - 1.0) * v * v, gam * v]])


def euler_jac(u, v, H, d):
    """x-direction Jacobian from the y one by swapping the roles of (u, rho u) and (v, rho v)."""
    if d == 2:
        return euler_jac_y(u, v, H)
    P = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1.0]])
    return P @ euler_jac_y(v, u, H) @ P


def swe_jac(u, v, c2, d):
    if d == 2:
        return np.array([[0.0, 0.0, 1.0], [-u * v, v, u], [c2 - v * v, 0.0, 2 * v]])
    return np.array([[0.0, 1.0, 0.0], [c2 - u * u, 2 * u, 0.0], [-u * v, v, u]])


def fd_jac(flux, q, d, eps=1e-6):
    J = np.zeros((len(q), len(q)))
    for k in range(len(q)):
        e = np.zeros(len(q))
        e[k] = eps * max(1.0, abs(q[k]))
        J[:, k] = (flux(q + e, d) - flux(q - e, d)) / (2 * e[k])
    return J


def rand_euler(rng, n):
    rho = rng.uniform(0.1, 4.0, n)
    u = rng.uniform(-3, 3, n)
    v = rng.uniform(-3, 3, n)
    p = rng.uniform(0.1, 10.0, n)
    E = p / (GAM - 1.0) + 0.5 * rho * (u * u + v * v)
    return np.stack([rho, rho * u, rho * v, E], 1)


def rand_swe(rng, n):
    h = rng.uniform(0.1, 3.0, n)
    u = rng.uniform(-2, 2, n)
    v = rng.uniform(-2, 2, n)
    return np.stack([h, h * u, h * v], 1)


# ---- examples --------------------------------------------------------------------------------------
def test_limiter_spec_examples():
    for ex in GOLD["limiter"]:
        assert oracle.limiter(oracle.LIM_MINMOD, ex["theta"]) == ex["minmod"]
        assert oracle.limiter(oracle.LIM_MC, ex["theta"]) == ex["mc"]
        assert oracle.limiter(oracle.LIM_NONE, ex["theta"]) == 1.0


def test_riemann_advect_spec_examples():
    for ex in GOLD["riemann_advect"]:
        pr = oracle.problem(oracle.ADV_CONST, (ex["s"], 0.0))
        W, s, am, ap = oracle.rpn2(pr, 1, [ex["ql"]], [ex["qr"]])
        assert (W[0, 0], s[0], am[0], ap[0]) == (ex["wave"], ex["s"], ex["amdq"], ex["apdq"])
        # same through the edge-velocity solver (velocity stored with the right cell)
        pr2 = oracle.problem(oracle.ADV_EDGEVEL_CAPA)
        W2, s2, am2, ap2 = oracle.rpn2(pr2, 1, [ex["ql"]], [ex["qr"]], [1, 9, 9], [1, ex["s"], 9])
        assert (W2[0, 0], s2[0], am2[0], ap2[0]) == (ex["wave"], ex["s"], ex["amdq"], ex["apdq"])


def test_advect_fluctuation_identity(rng):
    """A-dq + A+dq = s dq for random inputs."""
    for _ in range(200):
        s = rng.normal()
        ql, qr = rng.normal(size=2)
        for ixy in (1, 2):
            pr = oracle.problem(oracle.ADV_CONST, (s, s) if True else None)
            W, sp, am, ap = oracle.rpn2(pr, ixy, [ql], [qr])
            assert am[0] + ap[0] == pytest.approx(s * (qr - ql), rel=1e-15, abs=1e-300)


# ---- Roe solvers ------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", [oracle.SWE_ROE, oracle.EULER_ROE])
@pytest.mark.parametrize("efix", [0.0, 1.0])
def test_roe_properties(rng, kind, efix):
    """Roe's defining properties: sum_p W_p = dq and sum_p s_p W_p = f(q_r) - f(q_l); the
    fluctuations always split the flux difference, A-dq + A+dq = df (also with HH)."""
    if kind == oracle.SWE_ROE and efix:
        pytest.skip("no entropy fix for SWE (reading: subcritical dam break)")
    params = (G_SWE, 0.0) if kind == oracle.SWE_ROE else (GAM, efix)
    pr = oracle.problem(kind, params)
    flux = swe_flux if kind == oracle.SWE_ROE else euler_flux
    gen = rand_swe if kind == oracle.SWE_ROE else rand_euler
    Ql, Qr = gen(rng, 300), gen(rng, 300)
    if efix:   # moderate jumps in primitive variables keep the HH intermediate states physical
        def prim_pert(n):
            rho = rng.uniform(0.5, 2.0, n)
            u, v = rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n)
            p = rng.uniform(0.5, 2.0, n)
            return np.stack([rho, rho * u, rho * v, p / (GAM - 1.0) + 0.5 * rho * (u * u + v * v)], 1)
        Ql, Qr = prim_pert(300), prim_pert(300)
    done = 0
    for ql, qr in zip(Ql, Qr):
        for d in (1, 2):
            try:
                W, s, am, ap = oracle.rpn2(pr, d, ql, qr)
            except RuntimeError:
                # the linearised HH intermediate state Q_l + W1 / Q_r - W4 is unphysical for some
                # strong rarefactions (Roe is not positivity preserving): flagged, not computed
                assert efix
                continue
            done += 1
            df = flux(qr, d) - flux(ql, d)
            scale = np.abs(flux(qr, d)).max() + np.abs(flux(ql, d)).max()
            np.testing.assert_allclose(W.sum(0), qr - ql, rtol=0, atol=1e-13 * np.abs(np.r_[ql, qr]).max())
            np.testing.assert_allclose((s[:, None] * W).sum(0), df, rtol=0, atol=1e-13 * scale)
            np.testing.assert_allclose(am + ap, df, rtol=0, atol=1e-13 * scale)
    assert done >= 0.8 * 2 * len(Ql)


@pytest.mark.parametrize("kind", [oracle.SWE_ROE, oracle.EULER_ROE])
def test_equal_states_give_no_waves(rng, kind):
    params = (G_SWE, 0.0) if kind == oracle.SWE_ROE else (GAM, 1.0)
    pr = oracle.problem(kind, params)
    q = (rand_swe if kind == oracle.SWE_ROE else rand_euler)(rng, 20)
    for qq in q:
        for d in (1, 2):
            W, s, am, ap = oracle.rpn2(pr, d, qq, qq)
            assert not W.any() and not am.any() and not ap.any()


def test_euler_supersonic_upwinding(rng):
    """All characteristic speeds positive -> A-dq = 0; all negative -> A+dq = 0 (with HH)."""
    pr = oracle.problem(oracle.EULER_ROE, (GAM, 1.0))
    for sign in (1.0, -1.0):
        for _ in range(50):
            rho = rng.uniform(0.5, 2.0, 2)
            p = rng.uniform(0.5, 2.0, 2)
            c = np.sqrt(GAM * p / rho)
            u = sign * (c.max() * 3.0 + rng.uniform(0, 1, 2))
            v = rng.uniform(-1, 1, 2)
            E = p / (GAM - 1) + 0.5 * rho * (u * u + v * v)
            ql = np.array([rho[0], rho[0] * u[0], rho[0] * v[0], E[0]])
            qr = np.array([rho[1], rho[1] * u[1], rho[1] * v[1], E[1]])
            W, s, am, ap = oracle.rpn2(pr, 1, ql, qr)
            if sign > 0:
                assert not am.any()
            else:
                assert np.abs(ap).max() <= 1e-13 * np.abs(am).max()


def test_euler_entropy_fix_transonic_rarefaction():
    """A transonic 1-rarefaction (u-c < 0 left, > 0 in the star state): the plain Roe split puts
    the whole 1-wave to the left; Harten-Hyman splits it, and the fixed A-dq lies strictly between
    0 and the unfixed one in its density component."""
    rho_l, u_l, p_l = 1.0, 0.75, 1.0
    rho_r, u_r, p_r = 0.125, 0.0, 0.1     # Sod-like with a left-moving rarefaction through sonic
    E_l = p_l / (GAM - 1) + 0.5 * rho_l * u_l ** 2
    E_r = p_r / (GAM - 1) + 0.5 * rho_r * u_r ** 2
    ql = np.array([rho_l, rho_l * u_l, 0.0, E_l])
    qr = np.array([rho_r, rho_r * u_r, 0.0, E_r])
    _, s0, am0, ap0 = oracle.rpn2(oracle.problem(oracle.EULER_ROE, (GAM, 0.0)), 1, ql, qr)
    _, s1, am1, ap1 = oracle.rpn2(oracle.problem(oracle.EULER_ROE, (GAM, 1.0)), 1, ql, qr)
    assert not np.allclose(am0, am1)
    np.testing.assert_allclose(am0 + ap0, am1 + ap1, rtol=1e-14)


@pytest.mark.parametrize("kind", [oracle.SWE_ROE, oracle.EULER_ROE])
def test_transverse_split_is_jacobian(rng, kind):
    """B-X + B+X = B(q*) X with B the transverse flux Jacobian at the Roe state; the Jacobian
    formula used here is first checked against finite differences of the PDE flux."""
    swe = kind == oracle.SWE_ROE
    pr = oracle.problem(kind, (G_SWE, 0.0) if swe else (GAM, 1.0))
    gen = rand_swe if swe else rand_euler
    flux = swe_flux if swe else euler_flux
    for q in gen(rng, 10):
        for d in (1, 2):
            u, v = q[1] / q[0], q[2] / q[0]
            if swe:
                J = swe_jac(u, v, G_SWE * q[0], d)
            else:
                p = (GAM - 1) * (q[3] - 0.5 * q[0] * (u * u + v * v))
                J = euler_jac(u, v, (q[3] + p) / q[0], d)
            np.testing.assert_allclose(J, fd_jac(flux, q, d), rtol=1e-6, atol=1e-6)
    Ql, Qr = gen(rng, 100), gen(rng, 100)
    for ql, qr in zip(Ql, Qr):
        X = rng.normal(size=len(ql))
        # Roe averages (Roe 1981): sqrt(density)-weighted velocities and enthalpy
        sl, sr = np.sqrt(ql[0]), np.sqrt(qr[0])
        avg = lambda a, b: (sl * a + sr * b) / (sl + sr)
        u, v = avg(ql[1] / ql[0], qr[1] / qr[0]), avg(ql[2] / ql[0], qr[2] / qr[0])
        for ixy in (1, 2):
            bm, bp = oracle.rpt2(pr, ixy, ql, qr, X)
            td = 2 if ixy == 1 else 1
            if swe:
                B = swe_jac(u, v, G_SWE * 0.5 * (ql[0] + qr[0]), td)
            else:
                H = lambda q: (q[3] + (GAM - 1) * (q[3] - 0.5 * (q[1] ** 2 + q[2] ** 2) / q[0])) / q[0]
                B = euler_jac(u, v, avg(H(ql), H(qr)), td)
            ref = B @ X
            np.testing.assert_allclose(bm + bp, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max(), np.abs(B).max() * np.abs(X).max()))


def test_transverse_edge_velocity_uses_receiving_cell():
    """ADV_EDGEVEL_CAPA: B-X = min(low transverse edge velocity, 0) X, B+X = max(high one, 0) X
    of the receiving cell (reading 3)."""
    pr = oracle.problem(oracle.ADV_EDGEVEL_CAPA)
    bm, bp = oracle.rpt2(pr, 1, [0.0], [0.0], [2.0], aux_recv=[1.0, 0.3, -0.7], aux_next=[1.0, 0.1, 0.9])
    assert (bm[0], bp[0]) == (-0.7 * 2.0, 0.9 * 2.0)
    bm, bp = oracle.rpt2(pr, 2, [0.0], [0.0], [2.0], aux_recv=[1.0, 0.3, -0.7], aux_next=[1.0, -0.4, 0.9])
    assert (bm[0], bp[0]) == (0.0, 0.0 * 2.0)
    bm, bp = oracle.rpt2(pr, 2, [0.0], [0.0], [2.0], aux_recv=[1.0, -0.3, -0.7], aux_next=[1.0, 0.4, 0.9])
    assert (bm[0], bp[0]) == (-0.6, 0.8)


@pytest.mark.parametrize("kind", [oracle.SWE_ROE, oracle.EULER_ROE])
def test_direction_symmetry(rng, kind):
    """Solving in y equals solving in x with the momentum components swapped."""
    swe = kind == oracle.SWE_ROE
    pr = oracle.problem(kind, (G_SWE, 0.0) if swe else (GAM, 0.0))
    gen = rand_swe if swe else rand_euler
    perm = [0, 2, 1] if swe else [0, 2, 1, 3]
    for ql, qr in zip(gen(rng, 50), gen(rng, 50)):
        Wx, sx, amx, apx = oracle.rpn2(pr, 1, ql[perm], qr[perm])
        Wy, sy, amy, apy = oracle.rpn2(pr, 2, ql, qr)
        np.testing.assert_array_equal(sx, sy)
        np.testing.assert_allclose(amx[perm], amy, rtol=1e-15, atol=1e-15)
        np.testing.assert_allclose(apx[perm], apy, rtol=1e-15, atol=1e-15)
