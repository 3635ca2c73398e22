"""Pin (SURVEY §8(c.8) "update, 1D reduction"): the oracle's 2D unsplit step (oracle/claw.c,
orc_step_patch) on data that vary along x only equals an independent 1D wave-propagation code
written here in numpy from LeVeque's algorithm, which PAPER.md:168-171 [§3] cites ("the wave
propagation algorithm ... LeVeque"): J. Comput. Phys. 131 (1997); Finite Volume Methods for
Hyperbolic Problems (2002) -- §6.15-6.16 (capacity-form differencing, (dt/dx)_avg in the
correction flux), §9.5 (the limiter acts on the wave by the projection theta = W_I.W / W.W),
§15.3.2 (Roe linearisation), §15.3.5 (Harten-Hyman entropy fix).

Why the reduction is exact: with no jump along y every y-edge Riemann problem has zero waves, so
the y-sweep contributes nothing; the x-sweep's transverse terms G~ are identical on every row, so
G~(j+1/2) - G~(j-1/2) vanishes bitwise.  What is left is 1D wave propagation along each row.

The 1D code below is deliberately built differently from the oracle: Roe wave strengths come from
a numerical solve R alpha = dq with the eigenvector matrix (not closed-form strengths); the
Harten-Hyman fix evaluates the eigenvalues of the intermediate states with divisions and square
roots; the update is vectorised over cells.  A plausible mistake in the oracle -- the correction
flux scaled by one cell's dt/(kappa dx) instead of the average, a per-component limiter ratio
instead of the wave projection, the other cell's kappa in the CFL, a wrong Roe eigenvector or
wave speed, a dropped Harten-Hyman case -- fails one of these tests (DESIGN.md §9 records which
mutations were checked).

Also here: the capacity form with kappa = c, u~ = c u, v~ = c v reproduces ADV_CONST(u, v)
(genuinely 2D data), and the transverse (corner-transport) part of the capacity form, pinned by
the CTU mass budget of one fluctuation (test_capacity_transverse_moves_the_receiving_cells_share).
"""
import numpy as np
import pytest

import oracle

GAM = 1.4
G = 1.0
RNG = 1308147 + 41


# ------------------------------------------------------------------------------------------------
# independent 1D wave propagation (LeVeque 2002), x-direction, padded arrays with 2 ghost cells
# ------------------------------------------------------------------------------------------------
def roe_swe(ql, qr, g):
    """Roe eigen-system of the x-split shallow-water system with a passive tangential momentum
    (h, hu, hv): returns (waves [3][3], speeds [3]); strengths from a linear solve."""
    hl, hr = ql[0], qr[0]
    sl, sr = np.sqrt(hl), np.sqrt(hr)
    u = (sl * ql[1] / hl + sr * qr[1] / hr) / (sl + sr)
    v = (sl * ql[2] / hl + sr * qr[2] / hr) / (sl + sr)
    c = np.sqrt(g * 0.5 * (hl + hr))
    R = np.array([[1.0, u - c, v], [0.0, 0.0, 1.0], [1.0, u + c, v]]).T   # columns r1, r2, r3
    alpha = np.linalg.solve(R, qr - ql)
    return (R * alpha).T, np.array([u - c, u, u + c])


def euler_prim(q, gam):
    rho = q[0]
    u, v = q[1] / rho, q[2] / rho
    p = (gam - 1.0) * (q[3] - 0.5 * rho * (u * u + v * v))
    return rho, u, v, p


def roe_euler(ql, qr, gam):
    """Roe eigen-system of the x-split Euler equations (rho, rho u, rho v, E): waves [4][4],
    speeds [4], the Roe normal velocity; strengths from a linear solve."""
    rl, ul, vl, pl = euler_prim(ql, gam)
    rr, ur, vr, pr = euler_prim(qr, gam)
    Hl, Hr = (ql[3] + pl) / rl, (qr[3] + pr) / rr
    sl, sr = np.sqrt(rl), np.sqrt(rr)
    u = (sl * ul + sr * ur) / (sl + sr)
    v = (sl * vl + sr * vr) / (sl + sr)
    H = (sl * Hl + sr * Hr) / (sl + sr)
    c = np.sqrt((gam - 1.0) * (H - 0.5 * (u * u + v * v)))
    R = np.array([[1.0, u - c, v, H - u * c],
                  [1.0, u, v, 0.5 * (u * u + v * v)],
                  [0.0, 0.0, 1.0, v],
                  [1.0, u + c, v, H + u * c]]).T
    alpha = np.linalg.solve(R, qr - ql)
    return (R * alpha).T, np.array([u - c, u, u, u + c]), u


def sound(q, gam):
    rho, u, _, p = euler_prim(q, gam)
    # the Roe-linearised intermediate states must stay physical (else the config is invalid:
    # the oracle stops with ORC_EPHYS, reading 19) -- the test data are chosen so
    assert rho > 0.0 and p > 0.0, "unphysical intermediate state"
    return u, np.sqrt(gam * p / rho)


def lam1(q, gam):
    u, c = sound(q, gam)
    return u - c


def lam4(q, gam):
    u, c = sound(q, gam)
    return u + c


HH_TRANSONIC = [0]   # how often the Harten-Hyman transonic branch fired (coverage of the tests)


def euler_amdq_hh(ql, qr, W, s, ubar, gam):
    """A-dq with the Harten-Hyman entropy fix, in the order SURVEY §8(c.5) (i)-(iv) states
    (LeVeque 2002 §15.3.5): eigenvalues of the intermediate states by direct evaluation."""
    l1l = lam1(ql, gam)
    if l1l >= 0.0 and s[0] > 0.0:                           # (i) fully supersonic to the right
        return np.zeros(4)
    l1r = lam1(ql + W[0], gam)                              # (ii) 1-wave
    if l1l < 0.0 < l1r:
        HH_TRANSONIC[0] += 1
        beta1 = l1l * (l1r - s[0]) / (l1r - l1l)
    elif s[0] < 0.0:
        beta1 = s[0]
    else:
        beta1 = 0.0
    am = beta1 * W[0]
    if ubar >= 0.0:                                         # (iii)
        return am
    am = am + ubar * (W[1] + W[2])
    l4l, l4r = lam4(qr - W[3], gam), lam4(qr, gam)          # (iv) 4-wave
    if l4l < 0.0 < l4r:
        HH_TRANSONIC[0] += 1
        am = am + l4l * (l4r - s[3]) / (l4r - l4l) * W[3]
    elif s[3] < 0.0:
        am = am + s[3] * W[3]
    return am


def mc(theta):
    return max(0.0, min(0.5 * (1.0 + theta), 2.0, 2.0 * theta))


def minmod_lim(theta):
    return max(0.0, min(1.0, theta))


def wave_prop_1d(kind, q, dt, dx, kappa=None, uedge=None, u=0.0, limiter=mc, efix=True):
    """One step of LeVeque's 1D wave-propagation method on a padded row q [meqn][N+4] (cells
    0, 1 and N+2, N+3 are ghosts).  Edge c lies between cells c-1 and c.  Returns the updated
    interior [meqn][N] and the CFL number max over the corrected edges of max(r_c s, -r_{c-1} s)
    (the cell the wave enters).  kind: 'adv' (constant u), 'capa' (kappa per cell, u~ per edge,
    edge c's velocity stored at cell c), 'swe', 'euler'."""
    meqn, NP = q.shape
    N = NP - 4
    kap = np.ones(NP) if kappa is None else kappa
    r = dt / (kap * dx)                                     # capacity-form dt / (kappa dx)
    waves, speeds, amdq, apdq = {}, {}, {}, {}
    for c in range(1, N + 4):                               # all edges of the padded row
        ql, qr = q[:, c - 1], q[:, c]
        if kind in ("adv", "capa"):
            s = np.array([u if kind == "adv" else uedge[c]])
            W = (qr - ql).reshape(1, 1)
            am = min(s[0], 0.0) * W[0]
        elif kind == "swe":
            W, s = roe_swe(ql, qr, G)
            am = sum(min(sp, 0.0) * Wp for sp, Wp in zip(s, W))
        else:
            W, s, ubar = roe_euler(ql, qr, GAM)
            am = euler_amdq_hh(ql, qr, W, s, ubar, GAM) if efix else \
                sum(min(sp, 0.0) * Wp for sp, Wp in zip(s, W))
        waves[c], speeds[c] = W, s
        amdq[c] = am
        apdq[c] = sum(sp * Wp for sp, Wp in zip(s, W)) - am  # A+dq = sum s W - A-dq
    Ft = {}
    cfl = 0.0
    for c in range(2, N + 3):                               # edges with corrections
        W, s = waves[c], speeds[c]
        rav = 0.5 * (r[c - 1] + r[c])                       # (dt/dx)_avg of the capacity form
        F = np.zeros(meqn)
        for p in range(len(s)):
            cfl = max(cfl, r[c] * s[p], -r[c - 1] * s[p])
            nn = float(W[p] @ W[p])
            if nn == 0.0:
                continue
            WI = waves[c - 1 if s[p] > 0.0 else c + 1][p]   # upwind neighbour, same family
            phi = limiter(float(WI @ W[p]) / nn)            # projection of W_I onto W
            F += 0.5 * abs(s[p]) * (1.0 - rav * abs(s[p])) * phi * W[p]
        Ft[c] = F
    qn = np.empty((meqn, N))
    for c in range(2, N + 2):                               # interior cells
        qn[:, c - 2] = q[:, c] - r[c] * (apdq[c] + amdq[c + 1]) - r[c] * (Ft[c + 1] - Ft[c])
    return qn, cfl


# ------------------------------------------------------------------------------------------------
def embed_rows(row, m):
    """[meqn][m+4] row -> padded patch [meqn][m+4][m+4] constant along y (ghost rows included)."""
    return np.ascontiguousarray(np.repeat(row[:, None, :], m + 4, axis=1))


def normal_first(q, meqn):
    """The y-sweep's normal momentum is component 2: swap components 1 and 2 for the 1D code."""
    return q[[0, 2, 1] + list(range(3, meqn))] if meqn >= 3 else q


def check_reduction(kind_id, params, row, dt, dx, aux=None, limiter=oracle.LIM_MC, cfl_expected=None,
                    kind=None, axis="x", **kw):
    """2D step of data varying along `axis` only == the 1D step along that axis, on every row
    (axis x) or column (axis y).  aux = [kappa, u~, v~] as 1D arrays along the axis."""
    meqn, n = row.shape
    m = n - 4
    pr = oracle.problem(kind_id, params, limiter=limiter)
    q2d = embed_rows(row, m)
    auxpad = None
    if aux is not None:
        auxpad = np.stack([np.repeat(a[None, :], n, axis=0) for a in aux])
    if axis == "y":                                          # transpose the data: vary along y
        q2d = np.ascontiguousarray(np.swapaxes(q2d, 1, 2))
        if meqn >= 3:
            q2d = np.ascontiguousarray(q2d[[0, 2, 1] + list(range(3, meqn))])
        if auxpad is not None:
            auxpad = np.stack([auxpad[0].T, auxpad[2].T, auxpad[1].T])
    if auxpad is not None:
        auxpad = np.ascontiguousarray(auxpad)
    q2, cfl2 = oracle.step_patch(pr, np.ascontiguousarray(q2d), dt, dx, dx, auxpad)
    if axis == "y":                                          # back to the row frame
        q2 = np.swapaxes(q2, 1, 2)
        if meqn >= 3:
            q2 = q2[[0, 2, 1] + list(range(3, meqn))]
    lim = {oracle.LIM_MC: mc, oracle.LIM_MINMOD: minmod_lim}[limiter]
    q1, cfl1 = wave_prop_1d(kind, row, dt, dx, limiter=lim, **kw)
    scale = np.abs(row[:, 2:-2]).max(axis=1)
    for j in range(2, m + 2):                                # every interior row equals the 1D step
        err = np.abs(q2[:, j, 2:-2] - q1).max(axis=1)
        assert np.all(err <= 1e-14 * scale), (axis, j, err / scale)
    if cfl_expected == "1d":
        assert abs(cfl2 - cfl1) <= 1e-14 * cfl1, (cfl2, cfl1)
    return q1, cfl1, cfl2


AXES = pytest.mark.parametrize("axis", ["x", "y"])


@AXES
def test_capacity_form_reduces_to_1d_capacity_differencing(axis):
    """ADV_EDGEVEL_CAPA with kappa and u~ varying along x (v~ = 0): q and the CFL (the entered
    cell's kappa) equal the 1D capacity-form code; the correction uses (dt/dx)_avg."""
    rng = np.random.default_rng(RNG)
    m = 16
    for trial in range(6):
        q = rng.uniform(0.0, 1.0, (1, m + 4))
        kap = rng.uniform(0.4, 2.5, m + 4)
        ue = rng.uniform(-1.0, 1.0, m + 4) if trial % 2 else rng.uniform(0.2, 1.0, m + 4)
        dx = 1.0 / m
        dt = 0.8 * dx * kap.min() / np.abs(ue).max()
        check_reduction(oracle.ADV_EDGEVEL_CAPA, (0.0, 0.0), q, dt, dx,
                        aux=[kap, ue, np.zeros(m + 4)], kind="capa", kappa=kap, uedge=ue,
                        cfl_expected="1d", axis=axis)
    # minmod as well
    q = rng.uniform(0.0, 1.0, (1, m + 4))
    kap = rng.uniform(0.4, 2.5, m + 4)
    ue = rng.uniform(-1.0, 1.0, m + 4)
    dt = 0.7 * kap.min() / m
    check_reduction(oracle.ADV_EDGEVEL_CAPA, (0.0, 0.0), q, dt, 1.0 / m, aux=[kap, ue, np.zeros(m + 4)],
                    limiter=oracle.LIM_MINMOD, kind="capa", kappa=kap, uedge=ue, cfl_expected="1d",
                    axis=axis)


@AXES
def test_constant_velocity_reduces_to_1d_with_transverse_cancelling(axis):
    """ADV_CONST(u, v) with v != 0: the transverse terms of the x-sweep cancel row by row."""
    rng = np.random.default_rng(RNG + 1)
    m = 16
    for u, v in [(0.9, 0.7), (-0.6, 0.3), (0.5, -1.1)]:
        q = rng.uniform(-1.0, 1.0, (1, m + 4))
        dx = 1.0 / m
        dt = 0.85 * dx / max(abs(u), abs(v))
        if axis == "y":
            u, v = v, u                                     # the normal speed is v
        check_reduction(oracle.ADV_CONST, (u, v), q, dt, dx, kind="adv", u=u if axis == "x" else v,
                        axis=axis)


def swe_row(rng, m):
    h = rng.uniform(1.0, 2.0, m + 4)
    h[(m + 4) // 2:] *= 0.6                                   # a jump
    u = rng.uniform(-0.4, 0.4, m + 4)
    v = rng.uniform(-0.5, 0.5, m + 4)
    return np.stack([h, h * u, h * v])


@AXES
def test_swe_roe_reduces_to_1d_roe(axis):
    """SWE_ROE with a tangential momentum (shear wave r2 carried at u~): 3-wave 1D Roe."""
    rng = np.random.default_rng(RNG + 2)
    m = 16
    for trial in range(4):
        q = swe_row(rng, m)
        dx = 1.0 / m
        dt = 0.8 * dx / (np.abs(q[1] / q[0]).max() + np.sqrt(G * q[0].max()))
        lim = oracle.LIM_MC if trial < 3 else oracle.LIM_MINMOD
        check_reduction(oracle.SWE_ROE, (G, 0.0), q, dt, dx, limiter=lim, kind="swe", axis=axis)


def euler_state(rho, u, v, p):
    return np.array([rho, rho * u, rho * v, p / (GAM - 1.0) + 0.5 * rho * (u * u + v * v)])


def euler_rows(rng, m):
    rows = []
    while len(rows) < 3:                                    # smooth random data with a jump,
        rho = rng.uniform(0.8, 1.6, m + 4)                  # kept when every Roe-linearised
        u = rng.uniform(-1.2, 1.2, m + 4)                   # intermediate state is physical
        v = rng.uniform(-0.5, 0.5, m + 4)
        p = rng.uniform(0.8, 1.6, m + 4)
        rho[m // 2:] *= 0.5
        q = np.stack([euler_state(*s) for s in zip(rho, u, v, p)], axis=1)
        try:
            wave_prop_1d("euler", q, 1e-3, 1.0 / m)
        except AssertionError:
            continue
        rows.append(q)
    # Toro's test 1 (sonic point in the left rarefaction), variants, and the mirror images
    # (right-facing: the 4-wave branch of the fix)
    for ul, vt in [(0.75, 0.2), (0.6, -0.3), (0.9, 0.0)]:
        L, R = euler_state(1.0, ul, vt, 1.0), euler_state(0.125, 0.0, -0.1, 0.1)
        rows.append(np.stack([L if i < (m + 4) // 2 else R for i in range(m + 4)], axis=1))
        Lm, Rm = euler_state(0.125, 0.0, 0.1, 0.1), euler_state(1.0, -ul, -vt, 1.0)
        rows.append(np.stack([Lm if i < (m + 4) // 2 else Rm for i in range(m + 4)], axis=1))
    return rows


@AXES
def test_euler_roe_harten_hyman_reduces_to_1d_roe_with_entropy_fix(axis):
    """EULER_ROE with the Harten-Hyman fix (p1 = 1) and a tangential momentum: 4-wave 1D Roe,
    including transonic rarefactions (the fix fires; counted)."""
    rng = np.random.default_rng(RNG + 3)
    m = 16
    rows = euler_rows(rng, m)
    HH_TRANSONIC[0] = 0
    for q in rows:
        rho, u, v, p = euler_prim(q, GAM)
        dx = 1.0 / m
        dt = 0.7 * dx / (np.abs(u).max() + np.sqrt(GAM * p / rho).max())
        check_reduction(oracle.EULER_ROE, (GAM, 1.0), q, dt, dx, kind="euler", axis=axis)
    assert HH_TRANSONIC[0] >= 3, HH_TRANSONIC[0]   # both branches (1-wave, 4-wave) fire


@AXES
def test_euler_roe_without_fix_reduces_to_plain_roe(axis):
    rng = np.random.default_rng(RNG + 4)
    m = 16
    for q in euler_rows(rng, m)[:3]:
        rho, u, v, p = euler_prim(q, GAM)
        dx = 1.0 / m
        dt = 0.7 * dx / (np.abs(u).max() + np.sqrt(GAM * p / rho).max())
        check_reduction(oracle.EULER_ROE, (GAM, 0.0), q, dt, dx, kind="euler", efix=False,
                        axis=axis)


def test_systems_cfl_is_max_of_x_and_y_sweeps():
    """The 2D CFL is max(x-sweep, y-sweep) (reading 4): here the x part is the 1D code's and the
    y part, with no jump along y, is r (|v| + c) of the cells of columns 0..m+1."""
    rng = np.random.default_rng(RNG + 5)
    m = 16
    q = swe_row(rng, m)
    dx = 1.0 / m
    dt = 0.5 * dx
    _, cfl1, cfl2 = check_reduction(oracle.SWE_ROE, (G, 0.0), q, dt, dx, kind="swe")
    h = q[0, 1:m + 3]
    cy = (dt / dx) * (np.abs(q[2, 1:m + 3] / h) + np.sqrt(G * h)).max()
    assert abs(cfl2 - max(cfl1, cy)) <= 1e-14 * cfl2


# ------------------------------------------------------------------------------------------------
def test_capacity_with_constant_kappa_is_adv_const():
    """kappa = c, u~ = c u, v~ = c v is ADV_CONST(u, v) on genuinely 2D data (bitwise for a power
    of two, to rounding otherwise)."""
    rng = np.random.default_rng(RNG + 6)
    m = 16
    n = m + 4
    dx = 1.0 / m
    for u, v in [(0.9, 0.6), (-0.7, 0.4), (0.3, -0.8)]:
        q = np.ascontiguousarray(rng.uniform(0.0, 1.0, (1, n, n)))
        dt = 0.8 * dx / max(abs(u), abs(v))
        qa, ca = oracle.step_patch(oracle.problem(oracle.ADV_CONST, (u, v)), q, dt, dx, dx)
        for c, tol in [(2.0, 0.0), (1.7, 1e-14)]:
            aux = np.ascontiguousarray(np.stack([np.full((n, n), c), np.full((n, n), c * u),
                                                 np.full((n, n), c * v)]))
            qc, cc = oracle.step_patch(oracle.problem(oracle.ADV_EDGEVEL_CAPA), q, dt, dx, dx, aux)
            err = np.abs(qc[:, 2:-2, 2:-2] - qa[:, 2:-2, 2:-2]).max()
            assert err <= tol * np.abs(q).max(), (c, err)
            assert abs(cc - ca) <= tol * ca + (0.0 if tol == 0.0 else 1e-15), (c, cc, ca)


def test_capacity_transverse_moves_the_receiving_cells_share():
    """Corner transport in the capacity form (LeVeque 2002 §20.5 with §6.16's capacity; reading
    3): a fluctuation entering cell C raises C's mass by dt dy |fluctuation|; the transverse
    correction then moves the fraction 1/2 (|v~| dt / (kappa_C dy)) -- half of C's *own*
    transverse Courant number -- of that mass across C's edge in the direction of v~.  Data: one
    unit cell C0 in zero surroundings, first order with method3 = 1 (fluctuations only), all four
    sign patterns of (u~, v~).  The diagonal cell D downstream of C0 receives exactly two such
    shares: from the x-fluctuation entering C1 (D's neighbour across y) and from the
    y-fluctuation entering C2 (D's neighbour across x).  kappa varies strongly from cell to cell,
    so scaling a share by the other cell's kappa changes the value."""
    rng = np.random.default_rng(RNG + 7)
    m = 8
    n = m + 4
    dx = 1.0 / m
    I = lambda c: (c[1] + 1, c[0] + 1)   # (row, column) of 1-based cell (i, j) in the padded array
    xe = lambda a, b: (max(a[0], b[0]), a[1])      # storage cell of the x-edge between a and b
    ye = lambda a, b: (a[0], max(a[1], b[1]))      # storage cell of the y-edge between a and b
    for trial in range(8):
        sx, sy = (1, 1, -1, -1)[trial % 4], (1, -1, 1, -1)[trial % 4]
        kap = rng.uniform(0.3, 3.0, (n, n))
        ut = sx * rng.uniform(0.2, 1.0, (n, n))
        vt = sy * rng.uniform(0.2, 1.0, (n, n))
        aux = np.ascontiguousarray(np.stack([kap, ut, vt]))
        dt = 0.4 * dx * kap.min() / max(np.abs(ut).max(), np.abs(vt).max())
        i0, j0 = 4, 4
        C0, C1 = (i0 - sx, j0), (i0, j0)
        C2, D = (i0 - sx, j0 + sy), (i0, j0 + sy)
        q = np.zeros((1, n, n))
        q[(0,) + I(C0)] = 1.0
        pr = oracle.problem(oracle.ADV_EDGEVEL_CAPA, limiter=oracle.LIM_NONE, method2=1, method3=1)
        qn, _ = oracle.step_patch(pr, np.ascontiguousarray(q), dt, dx, dx, aux)
        # the fluctuation entering C1 through the x-edge C0|C1 is -|u~| (mass dt dy times it);
        # its share across C1's y-edge towards D
        mass1 = dt * dx * -abs(ut[I(xe(C0, C1))])
        share1 = 0.5 * abs(vt[I(ye(C1, D))]) * dt / (kap[I(C1)] * dx) * mass1
        # the fluctuation entering C2 through the y-edge C0|C2; its share across C2's x-edge to D
        mass2 = dt * dx * -abs(vt[I(ye(C0, C2))])
        share2 = 0.5 * abs(ut[I(xe(C2, D))]) * dt / (kap[I(C2)] * dx) * mass2
        # D gains the moved mass (negative here): its value is -(share1 + share2) / (kappa_D dx dy)
        expect = -(share1 + share2) / (kap[I(D)] * dx * dx)
        got = qn[(0,) + I(D)]
        assert abs(got - expect) <= 1e-14 * abs(expect), (sx, sy, got, expect)
