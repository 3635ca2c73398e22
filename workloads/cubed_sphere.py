"""C4 inputs: the six-tree cubed sphere (PAPER.md:230-236 [Fig. 1 right], PAPER.md:374-384 [§5
Example 2: rigid rotation on the sphere]).  Input generation only -- geometry and velocity data
the method consumes (capacity kappa and edge velocities), no ghost fill and no update.

Readings:
  * trees are cube faces +x, +y, -x, -y, +z, -z with right-handed frames (e_xi, e_eta, n);
    the connectivity is derived by matching the faces' shared 3D edges;
  * equiangular map: alpha, beta = (xi - 1/2) pi/2, (eta - 1/2) pi/2, point ~ n + tan(alpha) e_xi
    + tan(beta) e_eta, normalised to the unit sphere;
  * solid-body rotation about n_hat = (sin pi/4, 0, cos pi/4), omega = 2 pi, from the stream
    function psi = -omega n_hat . x: the flux through a cell edge is the psi difference of its end
    points, so the discrete velocity field is exactly divergence free; u~ = flux / d_eta,
    v~ = flux / d_xi (sign checked against (omega n_hat x X) . normal in the tests);
  * kappa = spherical area of the cell / (d_xi d_eta), two Van Oosterom-Strackee triangles;
  * ghost-cell aux = the true geometry of the region the ghost covers, reached through the
    connectivity and expressed (signed) in the patch's own frame; at the 8 three-tree corners the
    patch's own mapping is extended past its faces;
  * two cosine bells of radius 0.5 rad at (lambda, phi) = (5 pi/6, 0), (7 pi/6, 0):
    q = 0.1 + 0.9 sum_b 1/2 (1 + cos(pi d_b / r0)) [d_b < r0];
  * mesh: level `base` everywhere, refined by one level where the n_hat-latitude of a patch centre
    is within `band` rad of the bells' common n_hat-latitude (-0.6591).
"""
from __future__ import annotations

import math

import numpy as np

from .forests import Connectivity, Forest, forest_refined, forest_uniform

# (n, e_xi, e_eta) per tree: +x, +y, -x, -y, +z, -z
FRAMES = np.array([
    [[1, 0, 0], [0, 1, 0], [0, 0, 1]],
    [[0, 1, 0], [-1, 0, 0], [0, 0, 1]],
    [[-1, 0, 0], [0, -1, 0], [0, 0, 1]],
    [[0, -1, 0], [1, 0, 0], [0, 0, 1]],
    [[0, 0, 1], [1, 0, 0], [0, 1, 0]],
    [[0, 0, -1], [0, 1, 0], [1, 0, 0]],
], dtype=np.float64)

AXIS = np.array([math.sin(math.pi / 4), 0.0, math.cos(math.pi / 4)])
OMEGA = 2.0 * math.pi
BELLS = [(5 * math.pi / 6, 0.0), (7 * math.pi / 6, 0.0)]
R0 = 0.5


def cube_point(t: int, xi, eta):
    """Point on the cube [-1, 1]^3 of tree t at computational (xi, eta) (may lie past an edge)."""
    n, ex, ey = FRAMES[t]
    xi = np.asarray(xi, np.float64)[..., None]
    eta = np.asarray(eta, np.float64)[..., None]
    return n + (2 * xi - 1) * ex + (2 * eta - 1) * ey


def cube_connectivity() -> Connectivity:
    """Match each tree face (0: xi = 0, 1: xi = 1, 2: eta = 0, 3: eta = 1) with the face of another
    tree sharing the same 3D edge; reversed iff their tangential coordinates (eta on xi-faces, xi
    on eta-faces) run in opposite directions along the edge."""
    def edge(t, f):
        if f in (0, 1):
            xi = float(f)
            a, b = cube_point(t, xi, 0.0), cube_point(t, xi, 1.0)
        else:
            eta = float(f - 2)
            a, b = cube_point(t, 0.0, eta), cube_point(t, 1.0, eta)
        return np.round(a).astype(int), np.round(b).astype(int)
    T = 6
    t2t = np.zeros(4 * T, np.int32)
    t2f = np.zeros(4 * T, np.int8)
    for t in range(T):
        for f in range(4):
            a, b = edge(t, f)
            found = None
            for u in range(T):
                if u == t:
                    continue
                for g in range(4):
                    c, d = edge(u, g)
                    if (a == c).all() and (b == d).all():
                        found = (u, g, 0)
                    elif (a == d).all() and (b == c).all():
                        found = (u, g, 1)
            assert found is not None, (t, f)
            t2t[4 * t + f] = found[0]
            t2f[4 * t + f] = found[1] + 4 * found[2]
    return Connectivity(t2t, t2f, np.zeros(4 * T, np.int8))


def sphere_point(t: int, xi, eta):
    """Equiangular map of tree t (valid also slightly past the tree for ghost regions)."""
    n, ex, ey = FRAMES[t]
    a = (np.asarray(xi, np.float64) - 0.5) * (math.pi / 2)
    b = (np.asarray(eta, np.float64) - 0.5) * (math.pi / 2)
    p = n + np.tan(a)[..., None] * ex + np.tan(b)[..., None] * ey
    return p / np.linalg.norm(p, axis=-1, keepdims=True)


def psi(x):
    return -OMEGA * (x @ AXIS)


def tri_area(a, b, c):
    """Solid angle of the spherical triangle (a, b, c) of unit vectors (Van Oosterom-Strackee)."""
    num = np.abs(np.einsum("...i,...i->...", a, np.cross(b, c)))
    den = 1.0 + np.einsum("...i,...i->...", a, b) + np.einsum("...i,...i->...", b, c) + \
        np.einsum("...i,...i->...", c, a)
    return 2.0 * np.arctan2(num, den)


# ---- continuous face crossing (the connectivity's meaning) ---------------------
def _cross(conn: Connectivity, t: int, f: int, X, Y):
    nt = int(conn.tree_to_tree[4 * t + f])
    code = int(conn.tree_to_face[4 * t + f])
    nf, rev = code & 3, code >> 2
    if f == 0:
        d, tau = -X, Y
    elif f == 1:
        d, tau = X - 1.0, Y
    elif f == 2:
        d, tau = -Y, X
    else:
        d, tau = Y - 1.0, X
    if rev:
        tau = 1.0 - tau
    if nf == 0:
        return nt, d, tau
    if nf == 1:
        return nt, 1.0 - d, tau
    if nf == 2:
        return nt, tau, d
    return nt, tau, 1.0 - d


def _corner_route(conn, t, fx, fy, xc, yc):
    """Tree and composed crossing for a corner region outside both faces, or None at a 3-tree
    corner (the two routes x-then-y and y-then-x disagree)."""
    def route(f1):
        t1, a, b = _cross(conn, t, f1, np.array([xc]), np.array([yc]))
        f2 = (0 if a[0] < 0 else 1) if (a[0] < 0 or a[0] > 1) else (2 if b[0] < 0 else 3)
        t2, a2, b2 = _cross(conn, t1, f2, a, b)
        return f1, f2, t1, t2, a2[0], b2[0]
    ra, rb = route(fx), route(fy)
    if ra[3] == rb[3] and abs(ra[4] - rb[4]) < 1e-12 and abs(ra[5] - rb[5]) < 1e-12:
        return ra
    return None


def _map_points(conn, t, region, X, Y):
    """Sphere points of coordinates (X, Y) given in tree t's frame that belong to a ghost region:
    region = None (inside), ("x", f), ("y", f) or ("c", fx, fy) for corner blocks."""
    if region is None:
        return sphere_point(t, X, Y)
    if region[0] in ("x", "y"):
        nt, A, B = _cross(conn, t, region[1], X, Y)
        return sphere_point(nt, A, B)
    r = region[3]
    if r is None:                      # three-tree cube corner: extend p's own mapping
        return sphere_point(t, X, Y)
    f1, f2, t1 = r[0], r[1], r[2]
    _, A, B = _cross(conn, t, f1, X, Y)
    t2, A2, B2 = _cross(conn, t1, f2, A, B)
    return sphere_point(t2, A2, B2)


def patch_geometry(conn, t, x0, y0, h, m):
    """aux [3][m+4][m+4] = (kappa, u~ at the left edge, v~ at the bottom edge) of every padded cell
    of the patch with origin (x0, y0) and size h in tree t, plus the sphere points of the cell
    centres [m+4][m+4][3].  Each cell's 4 corners (and its centre) are mapped through the face
    crossing(s) of the region the cell lies in."""
    n = m + 4
    d = h / m
    kk = np.arange(n) - 2
    XA = x0 + kk[None, :] * d + 0 * kk[:, None]
    YA = y0 + kk[:, None] * d + 0 * kk[None, :]
    XC, YC = XA + 0.5 * d, YA + 0.5 * d
    ox = np.where(XC < 0, -1, np.where(XC > 1, 1, 0))
    oy = np.where(YC < 0, -1, np.where(YC > 1, 1, 0))
    aux = np.zeros((3, n, n))
    centres = np.zeros((n, n, 3))
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            sel = (ox == sx) & (oy == sy)
            if not sel.any():
                continue
            if sx == 0 and sy == 0:
                region = None
            elif sy == 0:
                region = ("x", 0 if sx < 0 else 1)
            elif sx == 0:
                region = ("y", 2 if sy < 0 else 3)
            else:
                fx, fy = (0 if sx < 0 else 1), (2 if sy < 0 else 3)
                jj, ii = np.argwhere(sel)[0]
                region = ("c", fx, fy, _corner_route(conn, t, fx, fy, XC[jj, ii], YC[jj, ii]))
            xa, ya = XA[sel], YA[sel]
            bl = _map_points(conn, t, region, xa, ya)
            br = _map_points(conn, t, region, xa + d, ya)
            tl = _map_points(conn, t, region, xa, ya + d)
            tr = _map_points(conn, t, region, xa + d, ya + d)
            area = tri_area(bl, br, tr) + tri_area(bl, tr, tl)
            aux[0][sel] = area / (d * d)
            aux[1][sel] = (psi(bl) - psi(tl)) / d      # flux through the left edge, +xi normal
            aux[2][sel] = (psi(br) - psi(bl)) / d      # flux through the bottom edge, +eta normal
            centres[sel] = _map_points(conn, t, region, xa + 0.5 * d, ya + 0.5 * d)
    return aux, centres


def bells(x):
    q = np.full(x.shape[:-1], 0.1)
    for lam, phi in BELLS:
        c = np.array([math.cos(phi) * math.cos(lam), math.cos(phi) * math.sin(lam), math.sin(phi)])
        dist = np.arccos(np.clip(x @ c, -1.0, 1.0))
        q = q + np.where(dist < R0, 0.9 * 0.5 * (1.0 + np.cos(math.pi * dist / R0)), 0.0)
    return q


def band_latitude():
    lam, phi = BELLS[0]
    c = np.array([math.cos(phi) * math.cos(lam), math.cos(phi) * math.sin(lam), math.sin(phi)])
    return math.asin(float(c @ AXIS))


def c4_forest(base_level: int = 4, band: float = 0.6, uniform: bool = False) -> Forest:
    conn = cube_connectivity()
    if uniform:
        return forest_uniform(conn, base_level)
    phib = band_latitude()

    def refine(t, xc, yc, h):
        p = sphere_point(t, xc, yc)
        lat = np.arcsin(np.clip(p @ AXIS, -1.0, 1.0))
        return np.abs(lat - phib) < band
    return forest_refined(conn, base_level, refine)


def _sphere_point_t(torch, t: int, xi, eta):
    """sphere_point in torch (float64)."""
    n, ex, ey = (torch.as_tensor(v, dtype=torch.float64, device=xi.device) for v in FRAMES[t])
    a = (xi - 0.5) * (math.pi / 2)
    b = (eta - 0.5) * (math.pi / 2)
    p = n + torch.tan(a)[..., None] * ex + torch.tan(b)[..., None] * ey
    return p / torch.linalg.vector_norm(p, dim=-1, keepdim=True)


def _map_points_t(torch, conn, t, region, X, Y):
    if region is None or (region[0] == "c" and region[3] is None):
        return _sphere_point_t(torch, t, X, Y)
    if region[0] in ("x", "y"):
        nt, A, B = _cross(conn, t, region[1], X, Y)
        return _sphere_point_t(torch, nt, A, B)
    r = region[3]
    _, A, B = _cross(conn, t, r[0], X, Y)
    t2, A2, B2 = _cross(conn, r[2], r[1], A, B)
    return _sphere_point_t(torch, t2, A2, B2)


def _tri_area_t(torch, a, b, c):
    num = torch.abs((a * torch.linalg.cross(b, c)).sum(-1))
    den = 1.0 + (a * b).sum(-1) + (b * c).sum(-1) + (c * a).sum(-1)
    return 2.0 * torch.atan2(num, den)


def all_patch_geometry(conn, tree_ids, x0, y0, h, m, chunk=8192):
    """patch_geometry for every patch, vectorised: aux [P][3][m+4][m+4] and interior cell-centre
    sphere points [P][m][m][3].  Same mapping, face crossings and formulas as patch_geometry, per
    cell corner.  With a GPU the arithmetic runs in torch fp64 on it (the T4 variant has 92 M padded
    cells: ~2 min in numpy); otherwise numpy on chunks of patches.  The two agree to ~1e-12
    (transcendental implementations); a run uses one of them for both the oracle and the GPU."""
    import torch
    if not torch.cuda.is_available():
        return _all_patch_geometry_np(conn, tree_ids, x0, y0, h, m)
    dev = torch.device("cuda")
    P = len(tree_ids)
    n = m + 4
    aux = np.zeros((P, 3, n, n))
    centres = np.zeros((P, m, m, 3))
    axis = torch.as_tensor(AXIS, dtype=torch.float64, device=dev)
    psi_t = lambda x: -OMEGA * (x @ axis)
    routes = {}
    for a0 in range(0, P, chunk):
        sl = slice(a0, min(P, a0 + chunk))
        T = torch.as_tensor(np.asarray(tree_ids[sl]), device=dev)
        X0 = torch.as_tensor(np.asarray(x0[sl], np.float64), device=dev)
        Y0 = torch.as_tensor(np.asarray(y0[sl], np.float64), device=dev)
        d = torch.as_tensor(np.asarray(h[sl], np.float64), device=dev)[:, None, None] / m
        kk = torch.arange(n, device=dev, dtype=torch.float64) - 2
        XA = X0[:, None, None] + kk[None, None, :] * d + 0 * kk[None, :, None]
        YA = Y0[:, None, None] + kk[None, :, None] * d + 0 * kk[None, None, :]
        XC, YC = XA + 0.5 * d, YA + 0.5 * d
        ox = torch.where(XC < 0, -1, torch.where(XC > 1, 1, 0))
        oy = torch.where(YC < 0, -1, torch.where(YC > 1, 1, 0))
        DD = d.expand_as(XA)
        TT = T[:, None, None].expand_as(XA)
        A = torch.zeros((XA.shape[0], 3, n, n), dtype=torch.float64, device=dev)
        Cn = torch.zeros(XA.shape + (3,), dtype=torch.float64, device=dev)
        for t in range(conn.num_trees):
            for sx in (-1, 0, 1):
                for sy in (-1, 0, 1):
                    sel = (TT == t) & (ox == sx) & (oy == sy)
                    idx = torch.nonzero(sel, as_tuple=True)
                    if idx[0].numel() == 0:
                        continue
                    if sx == 0 and sy == 0:
                        region = None
                    elif sy == 0:
                        region = ("x", 0 if sx < 0 else 1)
                    elif sx == 0:
                        region = ("y", 2 if sy < 0 else 3)
                    else:
                        fx, fy = (0 if sx < 0 else 1), (2 if sy < 0 else 3)
                        if (t, fx, fy) not in routes:
                            p_, j_, i_ = (int(v[0]) for v in idx)
                            routes[(t, fx, fy)] = _corner_route(conn, t, fx, fy, float(XC[p_, j_, i_]),
                                                                float(YC[p_, j_, i_]))
                        region = ("c", fx, fy, routes[(t, fx, fy)])
                    xa, ya, dd = XA[idx], YA[idx], DD[idx]
                    bl = _map_points_t(torch, conn, t, region, xa, ya)
                    br = _map_points_t(torch, conn, t, region, xa + dd, ya)
                    tl = _map_points_t(torch, conn, t, region, xa, ya + dd)
                    tr = _map_points_t(torch, conn, t, region, xa + dd, ya + dd)
                    area = _tri_area_t(torch, bl, br, tr) + _tri_area_t(torch, bl, tr, tl)
                    A[idx[0], 0, idx[1], idx[2]] = area / (dd * dd)
                    A[idx[0], 1, idx[1], idx[2]] = (psi_t(bl) - psi_t(tl)) / dd   # left edge, +xi normal
                    A[idx[0], 2, idx[1], idx[2]] = (psi_t(br) - psi_t(bl)) / dd   # bottom edge, +eta
                    Cn[idx] = _map_points_t(torch, conn, t, region, xa + 0.5 * dd, ya + 0.5 * dd)
        aux[sl] = A.cpu().numpy()
        centres[sl] = Cn[:, 2:m + 2, 2:m + 2].cpu().numpy()
    return aux, centres


def _all_patch_geometry_np(conn, tree_ids, x0, y0, h, m, chunk=2048):
    P = len(tree_ids)
    if P > chunk:
        parts = [_all_patch_geometry_np(conn, tree_ids[a:a + chunk], x0[a:a + chunk], y0[a:a + chunk],
                                        h[a:a + chunk], m, chunk) for a in range(0, P, chunk)]
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
    n = m + 4
    d = (h / m)[:, None, None]
    kk = np.arange(n) - 2
    XA = x0[:, None, None] + kk[None, None, :] * d + 0 * kk[None, :, None]
    YA = y0[:, None, None] + kk[None, :, None] * d + 0 * kk[None, None, :]
    XC, YC = XA + 0.5 * d, YA + 0.5 * d
    ox = np.where(XC < 0, -1, np.where(XC > 1, 1, 0))
    oy = np.where(YC < 0, -1, np.where(YC > 1, 1, 0))
    DD = np.broadcast_to(d, XA.shape)
    TT = np.broadcast_to(np.asarray(tree_ids)[:, None, None], XA.shape)
    aux = np.zeros((P, 3, n, n))
    centres = np.zeros((P, n, n, 3))
    for t in range(conn.num_trees):
        for sx in (-1, 0, 1):
            for sy in (-1, 0, 1):
                sel = (TT == t) & (ox == sx) & (oy == sy)
                if not sel.any():
                    continue
                if sx == 0 and sy == 0:
                    region = None
                elif sy == 0:
                    region = ("x", 0 if sx < 0 else 1)
                elif sx == 0:
                    region = ("y", 2 if sy < 0 else 3)
                else:
                    fx, fy = (0 if sx < 0 else 1), (2 if sy < 0 else 3)
                    pp, jj, ii = np.argwhere(sel)[0]
                    region = ("c", fx, fy, _corner_route(conn, t, fx, fy, XC[pp, jj, ii], YC[pp, jj, ii]))
                xa, ya, dd = XA[sel], YA[sel], DD[sel]
                bl = _map_points(conn, t, region, xa, ya)
                br = _map_points(conn, t, region, xa + dd, ya)
                tl = _map_points(conn, t, region, xa, ya + dd)
                tr = _map_points(conn, t, region, xa + dd, ya + dd)
                area = tri_area(bl, br, tr) + tri_area(bl, tr, tl)
                idx = np.nonzero(sel)
                aux[idx[0], 0, idx[1], idx[2]] = area / (dd * dd)
                aux[idx[0], 1, idx[1], idx[2]] = (psi(bl) - psi(tl)) / dd
                aux[idx[0], 2, idx[1], idx[2]] = (psi(br) - psi(bl)) / dd
                centres[idx] = _map_points(conn, t, region, xa + 0.5 * dd, ya + 0.5 * dd)
    return aux, np.ascontiguousarray(centres[:, 2:m + 2, 2:m + 2])


def c4_workload(base_level: int = 4, m: int = 16, steps: int = 500, band: float = 0.6,
                uniform: bool = False):
    from .configs import ADV_EDGEVEL_CAPA, Workload
    f = c4_forest(base_level, band, uniform)
    P = f.num_patches
    x0, y0, h = f.origin()
    aux, centres = all_patch_geometry(f.conn, f.tree_ids, np.asarray(x0, np.float64),
                                      np.asarray(y0, np.float64), np.asarray(h, np.float64), m)
    q0 = bells(centres)[:, None]
    # dt = 0.9 / max over edges of |s| / (kappa_entered dxi)  (the CFL with dt factored out)
    dxi = (h / m)[:, None, None]
    kap = aux[:, 0]
    cmax = 0.0
    us = aux[:, 1, 2:m + 2, 2:m + 3]            # left edges of cells i = 1..m+1, rows 1..m
    ent = np.where(us > 0, kap[:, 2:m + 2, 2:m + 3], kap[:, 2:m + 2, 1:m + 2])
    cmax = max(cmax, float((np.abs(us) / (ent * dxi)).max()))
    vs = aux[:, 2, 2:m + 3, 2:m + 2]
    ent = np.where(vs > 0, kap[:, 2:m + 3, 2:m + 2], kap[:, 1:m + 2, 2:m + 2])
    cmax = max(cmax, float((np.abs(vs) / (ent * dxi)).max()))
    dt = 0.9 / cmax
    name = "C4" if (base_level, m, band, uniform) == (4, 16, 0.6, False) else \
        f"C4_L{base_level}_m{m}" + ("_uniform" if uniform else "")
    w = Workload(name, f, m, 1, 3, ADV_EDGEVEL_CAPA, (0.0, 0.0), np.ascontiguousarray(q0), aux, steps, dt,
                 "fixed")
    w.info["refined_parents"] = int((f.levels > base_level).sum() // 4)
    w.info["centres"] = centres          # sphere points of the interior cell centres (tests)
    return w
