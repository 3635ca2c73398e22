"""Pins for the oracle's Euler HLLE solver (oracle/claw.c rp_hlle; Einfeldt's
two-wave solver in LeVeque 2002 §15.3.7; reading 25).

Independent references: (1) conservation -- A-dq + A+dq = f(Q_r) - f(Q_l) for any states (the
physical flux is evaluated here from its definition, not by the oracle); (2) the HLLE speed bounds
s1 <= min(u_l - c_l, u^ - c^) and s2 >= max(u_r + c_r, u^ + c^), with equality for one of each,
u^ and c^ the Roe averages computed here; (3) supersonic upwinding: all speeds positive ->
A-dq = 0 and A+dq = the flux difference; (4) consistency: equal states give zero waves; (5) the
middle state of a strong two-rarefaction problem has positive density and pressure (HLLE is
positively conservative, where the Roe linearisation's intermediate state is not); (6) the whole
step with HLLE on Sod's shock tube converges to the exact solution (an exact Riemann solver written
here from the textbook formulas, Newton on the pressure), and conserves mass exactly on a closed
domain.
"""
import math

import numpy as np
import pytest

import oracle
from workloads import forests as F
from workloads.configs import EULER_HLLE, EULER_ROE, Workload

G = 1.4


def cons(rho, u, v, p):
    return np.array([rho, rho * u, rho * v, p / (G - 1) + 0.5 * rho * (u * u + v * v)])


def prim(q):
    rho = q[0]
    u, v = q[1] / rho, q[2] / rho
    return rho, u, v, (G - 1) * (q[3] - 0.5 * rho * (u * u + v * v))


def flux(q, ixy):
    rho, u, v, p = prim(q)
    un = u if ixy == 1 else v
    f = q * un
    f[ixy] += p
    f[3] += p * un
    return f


def random_states(rng, n):
    out = []
    for _ in range(n):
        a = cons(rng.uniform(0.2, 3), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.1, 5))
        b = cons(rng.uniform(0.2, 3), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.1, 5))
        out.append((a, b))
    return out


PR = oracle.problem(EULER_HLLE, (G, 0.0))


def test_two_waves_and_conservation(rng):
    assert oracle.mwaves(EULER_HLLE) == 2 and oracle.meqn(EULER_HLLE) == 4
    for ql, qr in random_states(rng, 200):
        for ixy in (1, 2):
            W, s, am, ap = oracle.rpn2(PR, ixy, ql, qr)
            df = flux(qr, ixy) - flux(ql, ixy)
            assert np.allclose(am + ap, df, rtol=0, atol=1e-13 * (1 + np.abs(df).max()))
            assert np.allclose(W.sum(0), qr - ql, rtol=0, atol=1e-13 * (1 + np.abs(qr - ql).max()))
            assert np.allclose(s[0] * W[0] + s[1] * W[1], df, rtol=0, atol=1e-12 * (1 + np.abs(df).max()))


def test_speed_bounds(rng):
    for ql, qr in random_states(rng, 200):
        for ixy in (1, 2):
            W, s, am, ap = oracle.rpn2(PR, ixy, ql, qr)
            rl, ul, vl, pl = prim(ql)
            rr, ur, vr, pr = prim(qr)
            unl, unr = (ul, ur) if ixy == 1 else (vl, vr)
            cl, cr = math.sqrt(G * pl / rl), math.sqrt(G * pr / rr)
            wl, wr = math.sqrt(rl), math.sqrt(rr)
            Hl, Hr = (ql[3] + pl) / rl, (qr[3] + pr) / rr
            uh = (wl * ul + wr * ur) / (wl + wr)
            vh = (wl * vl + wr * vr) / (wl + wr)
            Hh = (wl * Hl + wr * Hr) / (wl + wr)
            ch = math.sqrt((G - 1) * (Hh - 0.5 * (uh * uh + vh * vh)))
            unh = uh if ixy == 1 else vh
            assert s[0] == pytest.approx(min(unl - cl, unh - ch), rel=1e-13, abs=1e-13)
            assert s[1] == pytest.approx(max(unr + cr, unh + ch), rel=1e-13, abs=1e-13)
            assert s[0] < s[1]


def test_supersonic_upwinding_and_consistency(rng):
    ql, qr = cons(1.0, 3.0, 0.2, 1.0), cons(0.8, 2.8, -0.1, 0.9)     # u - c > 0 on both sides
    W, s, am, ap = oracle.rpn2(PR, 1, ql, qr)
    assert s[0] > 0 and (am == 0).all()
    np.testing.assert_allclose(ap, flux(qr, 1) - flux(ql, 1), rtol=0, atol=1e-13)
    for _ in range(20):
        q = cons(rng.uniform(0.2, 3), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.1, 5))
        W, s, am, ap = oracle.rpn2(PR, 2, q, q)
        assert (W == 0).all() and (am == 0).all() and (ap == 0).all()


def test_strong_rarefaction_middle_state_positive():
    """The 1-2-3-1 problem (Einfeldt et al.): states moving apart at Mach ~1.7.  HLLE's middle
    state keeps rho* > 0 and p* > 0; the Roe linearisation's intermediate density goes negative."""
    ql, qr = cons(1.0, -2.0, 0.0, 0.4), cons(1.0, 2.0, 0.0, 0.4)
    W, s, am, ap = oracle.rpn2(PR, 1, ql, qr)
    qs = ql + W[0]
    rho, u, v, p = prim(qs)
    assert rho > 0 and p > 0
    Wr, sr, _, _ = oracle.rpn2(oracle.problem(EULER_ROE, (G, 0.0)), 1, ql, qr)
    assert (ql + Wr[0])[0] < 0


def exact_sod(x, t, x0=2.0, L=(1.0, 0.0, 1.0), R=(0.125, 0.0, 0.1)):
    """Exact density of the Riemann problem (rho, u, p) L | R at x0 (textbook wave curves; Newton
    on p*; left rarefaction / right shock structure of Sod's data)."""
    rl, ul, pl = L
    rr, ur, pr = R
    cl, cr = math.sqrt(G * pl / rl), math.sqrt(G * pr / rr)

    def fk(p, rk, pk, ck):
        if p > pk:
            A, B = 2 / ((G + 1) * rk), (G - 1) / (G + 1) * pk
            return (p - pk) * math.sqrt(A / (p + B)), math.sqrt(A / (p + B)) * (1 - 0.5 * (p - pk) / (p + B))
        return (2 * ck / (G - 1)) * ((p / pk) ** ((G - 1) / (2 * G)) - 1), (p / pk) ** (-(G + 1) / (2 * G)) / (rk * ck)

    p = 0.5 * (pl + pr)
    for _ in range(60):
        f1, d1 = fk(p, rl, pl, cl)
        f2, d2 = fk(p, rr, pr, cr)
        p = max(1e-12, p - (f1 + f2 + ur - ul) / (d1 + d2))
    f1, _ = fk(p, rl, pl, cl)
    f2, _ = fk(p, rr, pr, cr)
    us = 0.5 * (ul + ur) + 0.5 * (f2 - f1)
    rls = rl * (p / pl) ** (1 / G)                                    # behind the rarefaction
    rrs = rr * ((p / pr + (G - 1) / (G + 1)) / ((G - 1) / (G + 1) * p / pr + 1))   # behind the shock
    cls = cl * (p / pl) ** ((G - 1) / (2 * G))
    sshock = ur + cr * math.sqrt((G + 1) / (2 * G) * p / pr + (G - 1) / (2 * G))
    out = np.empty_like(x)
    for i, xi in enumerate(x):
        xi = (xi - x0) / t
        if xi < ul - cl:
            out[i] = rl
        elif xi < us - cls:                                            # inside the fan
            c = 2 / (G + 1) * (cl + (G - 1) / 2 * (ul - xi))
            out[i] = rl * (c / cl) ** (2 / (G - 1))
        elif xi < us:
            out[i] = rls
        elif xi < sshock:
            out[i] = rrs
        else:
            out[i] = rr
    return out


def sod_workload(level, m=8, t_end=0.4, kind=EULER_HLLE):
    f = F.forest_uniform(F.brick(4, 1, bc=F.OUTFLOW), level)
    X, Y = F.cell_centres(f, m)
    X = X + f.tree_ids[:, None, None]
    left = X < 2.0
    q0 = np.stack([np.where(left, 1.0, 0.125), 0 * X, 0 * X, np.where(left, 1.0, 0.1) / (G - 1)], 1)
    dx = 0.5 ** level / m
    steps = int(math.ceil(t_end / (0.5 * dx)))
    return Workload(f"sod_L{level}", f, m, 4, 0, kind, (G, 0.0), q0, None, steps, t_end / steps, "fixed"), X


def test_hlle_step_converges_on_sod_and_conserves_mass():
    errs = []
    for level in (1, 2):
        w, X = sod_workload(level)
        q, cfl, dts = oracle.run(w)
        t = sum(dts)
        rho = q[:, 0]
        ex = exact_sod(X.ravel(), t).reshape(X.shape)
        dx = 0.5 ** level / w.m
        errs.append(np.abs(rho - ex).mean())
        assert np.ptp(rho, axis=1).max() < 1e-12          # one-dimensional: y-independent rows
        mass = rho.sum() * dx * dx
        assert mass == pytest.approx(w.q0[:, 0].sum() * dx * dx, rel=1e-13)   # waves stay inside
    assert errs[1] < 0.7 * errs[0] and errs[1] < 0.02
