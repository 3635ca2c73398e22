"""ctypes binding of the CPU oracle (liboracle.so, plain C in this directory).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  The product path never does, and the oracle
shares no code with it.  Every function cites the passage it follows in the C sources.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["forest.c", "ghost.c", "claw.c", "subcycle.c", "regrid.c", "forest3.c"]
LIB = os.path.join(HERE, "liboracle.so")

OK, EINVAL, ETILING, ECONN, EBALANCE, ENOMEM, EUNSUP, EPHYS = 0, -1, -2, -3, -4, -5, -6, -7
OP_NONE, OP_COPY, OP_AVG4, OP_INTERP, OP_BCX, OP_BCY, OP_CORNER3 = range(7)
ADV_CONST, ADV_EDGEVEL_CAPA, SWE_ROE, EULER_ROE, EULER_HLLE = 0, 1, 2, 3, 4
LIM_NONE, LIM_MINMOD, LIM_MC = 0, 1, 2
REC = 8


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -ffp-contract=off (plain C, optional OpenMP)."""
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    hdrs = [os.path.join(HERE, h) for h in ("oracle.h", "oracle_internal.h")]
    flags = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-fopenmp", "-Wall"]
    h = hashlib.sha256("\0".join(flags).encode())
    for s in srcs + hdrs:   # content-hash stamp (not mtimes): a shipped .so is rebuilt if stale
        with open(s, "rb") as f:
            h.update(f.read())
    stamp, stamp_file = h.hexdigest(), LIB + ".stamp"
    if not force and os.path.exists(LIB) and os.path.exists(stamp_file):
        with open(stamp_file) as f:
            if f.read().strip() == stamp:
                return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.run(flags + ["-o", tmp] + srcs + ["-lm"], check=True)
    os.replace(tmp, LIB)
    with open(stamp_file, "w") as f:
        f.write(stamp + "\n")
    return LIB


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int), ("p0", C.c_double), ("p1", C.c_double), ("limiter", C.c_int),
                ("method2", C.c_int), ("method3", C.c_int), ("reflux", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.c_void_p
        L.orc_forest_create.argtypes = [C.c_int64, P, P, C.c_int32, P, P, P, C.c_int, C.POINTER(P)]
        L.orc_forest_destroy.argtypes = [P]
        L.orc_forest_coords.argtypes = [P, P, P, C.POINTER(C.c_int)]
        L.orc_ring_count.argtypes = [C.c_int]
        L.orc_ghost_records.argtypes = [P, C.c_int64, P]
        L.orc_ghost_table.argtypes = [P, P]
        L.orc_ghost_fill.argtypes = [P, P, C.c_int]
        L.orc_step.argtypes = [P, C.POINTER(Problem), P, P, C.c_double, C.c_double, P,
                               C.POINTER(C.c_double), C.c_int]
        L.orc_step_sample.argtypes = [P, C.POINTER(Problem), P, P, C.c_double, C.c_double, P,
                                      C.c_int64, P, P]
        L.orc_build_padded_sample.argtypes = [P, P, C.c_int, C.c_int64, P]
        L.orc_step_patch.argtypes = [C.POINTER(Problem), C.c_int, C.c_int, P, P, C.c_double,
                                     C.c_double, C.c_double, P]
        L.orc_step_patch.restype = C.c_double
        L.orc_step_patch_faces.argtypes = [C.POINTER(Problem), C.c_int, C.c_int, P, P, C.c_double,
                                           C.c_double, C.c_double, P, P]
        L.orc_step_patch_faces.restype = C.c_double
        L.orc_flux.argtypes = [C.POINTER(Problem), C.c_int, P, C.c_double, P]
        L.orc_regrid.argtypes = [P, P, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, P, P, P, P, P]
        L.orc_step_subcycled.argtypes = [P, C.POINTER(Problem), P, P, C.c_double, C.c_double, P,
                                         C.POINTER(C.c_double)]
        L.orc_limiter.argtypes = [C.c_int, C.c_double]
        L.orc_limiter.restype = C.c_double
        L.orc_meqn.argtypes = [C.c_int]
        L.orc_mwaves.argtypes = [C.c_int]
        L.orc_rpn2.argtypes = [C.POINTER(Problem), C.c_int, P, P, P, P, P, P, P, P]
        L.orc_rpt2.argtypes = [C.POINTER(Problem), C.c_int, P, P, P, P, P, P, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def problem(kind, params=(0.0, 0.0), limiter=LIM_MC, method2=2, method3=2, reflux=0) -> Problem:
    return Problem(int(kind), float(params[0]), float(params[1]), int(limiter), int(method2),
                   int(method3), int(reflux))


def meqn(kind: int) -> int:
    return lib().orc_meqn(kind)


def mwaves(kind: int) -> int:
    return lib().orc_mwaves(kind)


def limiter(kind: int, theta: float) -> float:
    return lib().orc_limiter(kind, theta)


def rpn2(pr: Problem, ixy: int, ql, qr, auxl=None, auxr=None):
    me, mw = lib().orc_meqn(pr.kind), lib().orc_mwaves(pr.kind)
    ql = np.ascontiguousarray(ql, np.float64)
    qr = np.ascontiguousarray(qr, np.float64)
    al = np.ascontiguousarray(auxl if auxl is not None else [1.0, 0.0, 0.0], np.float64)
    ar = np.ascontiguousarray(auxr if auxr is not None else [1.0, 0.0, 0.0], np.float64)
    W = np.zeros((mw, me))
    s = np.zeros(mw)
    am = np.zeros(me)
    ap = np.zeros(me)
    rc = lib().orc_rpn2(C.byref(pr), ixy, _p(ql), _p(qr), _p(al), _p(ar), _p(W), _p(s), _p(am), _p(ap))
    if rc:
        raise RuntimeError(f"orc_rpn2 -> {rc}")
    return W, s, am, ap


def rpt2(pr: Problem, ixy: int, ql, qr, asdq, aux_recv=None, aux_next=None):
    me = lib().orc_meqn(pr.kind)
    ql = np.ascontiguousarray(ql, np.float64)
    qr = np.ascontiguousarray(qr, np.float64)
    X = np.ascontiguousarray(asdq, np.float64)
    a1 = np.ascontiguousarray(aux_recv if aux_recv is not None else [1.0, 0.0, 0.0], np.float64)
    a2 = np.ascontiguousarray(aux_next if aux_next is not None else [1.0, 0.0, 0.0], np.float64)
    bm = np.zeros(me)
    bp = np.zeros(me)
    rc = lib().orc_rpt2(C.byref(pr), ixy, _p(ql), _p(qr), _p(a1), _p(a2), _p(X), _p(bm), _p(bp))
    if rc:
        raise RuntimeError(f"orc_rpt2 -> {rc}")
    return bm, bp


def step_patch(pr: Problem, qpad: np.ndarray, dt: float, dx: float, dy: float, auxpad=None):
    """One update of a single padded patch [meqn][n][n] (ring filled) -> (qnew padded, cfl)."""
    meq, n, _ = qpad.shape
    m = n - 4
    qp = np.ascontiguousarray(qpad, np.float64)
    out = qp.copy()
    ap = None if auxpad is None else np.ascontiguousarray(auxpad, np.float64)
    cfl = lib().orc_step_patch(C.byref(pr), m, meq, _p(qp), None if ap is None else _p(ap), dt,
                               dx, dy, _p(out))
    return out, cfl


class OracleForest:
    """A decoded forest with brute-force ghost tables (forest.c) and the stepping driver."""

    def __init__(self, levels, tree_ids, conn, m: int):
        self.levels = np.ascontiguousarray(levels, np.int8)
        self.tree_ids = np.ascontiguousarray(tree_ids, np.int32)
        self.t2t = np.ascontiguousarray(conn.tree_to_tree, np.int32)
        self.t2f = np.ascontiguousarray(conn.tree_to_face, np.int8)
        self.fbc = np.ascontiguousarray(conn.face_bc, np.int8)
        self.m = m
        self.P = len(self.levels)
        h = C.c_void_p()
        rc = lib().orc_forest_create(self.P, _p(self.levels), _p(self.tree_ids), len(self.t2t) // 4,
                                     _p(self.t2t), _p(self.t2f), _p(self.fbc), m, C.byref(h))
        if rc:
            raise ValueError(f"orc_forest_create -> {rc}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_forest_destroy(self.h)
            self.h = None

    @property
    def n(self) -> int:
        return self.m + 4

    @property
    def G(self) -> int:
        return lib().orc_ring_count(self.m)

    def coords(self):
        x = np.zeros(self.P, np.int64)
        y = np.zeros(self.P, np.int64)
        lm = C.c_int()
        lib().orc_forest_coords(self.h, _p(x), _p(y), C.byref(lm))
        return x, y, lm.value

    def ghost_records(self, p: int) -> np.ndarray:
        rec = np.zeros((self.G, REC), np.int32)
        rc = lib().orc_ghost_records(self.h, p, _p(rec))
        if rc:
            raise ValueError(f"orc_ghost_records -> {rc}")
        return rec

    def ghost_table(self) -> np.ndarray:
        rec = np.zeros((self.P, self.G, REC), np.int32)
        rc = lib().orc_ghost_table(self.h, _p(rec))
        if rc:
            raise ValueError(f"orc_ghost_table -> {rc}")
        return rec

    def pad(self, q: np.ndarray) -> np.ndarray:
        """[P][meqn][m][m] interiors -> [P][meqn][n][n] with a NaN ring (unfilled)."""
        P, meq, m, _ = q.shape
        qp = np.full((P, meq, m + 4, m + 4), np.nan)
        qp[:, :, 2:m + 2, 2:m + 2] = q
        return qp

    def ghost_fill(self, qpad: np.ndarray) -> np.ndarray:
        assert qpad.flags.c_contiguous and qpad.dtype == np.float64
        rc = lib().orc_ghost_fill(self.h, _p(qpad), qpad.shape[1])
        if rc:
            raise ValueError(f"orc_ghost_fill -> {rc}")
        return qpad

    def step(self, pr: Problem, qpad: np.ndarray, dt: float, dx0: float, aux=None, nthreads=1):
        """Ghost fill of qpad (in place) + one update -> (qout padded, cfl)."""
        out = np.empty_like(qpad)
        cfl = C.c_double()
        ap = None if aux is None else np.ascontiguousarray(aux, np.float64)
        rc = lib().orc_step(self.h, C.byref(pr), _p(qpad), None if ap is None else _p(ap), dt, dx0,
                            _p(out), C.byref(cfl), nthreads)
        if rc:
            raise RuntimeError(f"orc_step -> {rc}")
        return out, cfl.value

    def step_subcycled(self, pr: Problem, qpad: np.ndarray, dt_coarse: float, dx0: float, aux=None):
        """One sub-cycled step (per-level dt, time-interpolated coarse ghosts; subcycle.c) of the
        coarsest level by dt_coarse -> (qout padded, interiors valid; cfl)."""
        qpad = np.ascontiguousarray(qpad, np.float64)
        out = np.empty_like(qpad)
        cfl = C.c_double()
        ap = None if aux is None else np.ascontiguousarray(aux, np.float64)
        rc = lib().orc_step_subcycled(self.h, C.byref(pr), _p(qpad), None if ap is None else _p(ap),
                                      dt_coarse, dx0, _p(out), C.byref(cfl))
        if rc:
            raise RuntimeError(f"orc_step_subcycled -> {rc}")
        return out, cfl.value

    def regrid(self, qpad: np.ndarray, refine_threshold: float, coarsen_threshold: float,
               min_level: int, max_level: int):
        """Regrid (regrid.c) from a ghost-filled padded state -> (levels, tree_ids, q interiors, src)."""
        qpad = np.ascontiguousarray(qpad, np.float64)
        P, meq = qpad.shape[0], qpad.shape[1]
        m = self.m
        nl = np.zeros(4 * P, np.int8)
        nt = np.zeros(4 * P, np.int32)
        qo = np.zeros((4 * P, meq, m, m))
        src = np.zeros((4 * P, 6), np.int32)
        npn = C.c_int64()
        rc = lib().orc_regrid(self.h, _p(qpad), meq, refine_threshold, coarsen_threshold, min_level, max_level,
                              C.byref(npn), _p(nl), _p(nt), _p(qo), _p(src))
        if rc:
            raise RuntimeError(f"orc_regrid -> {rc}")
        k = npn.value
        return nl[:k].copy(), nt[:k].copy(), qo[:k].copy(), src[:k].copy()

    def step_sample(self, pr: Problem, q: np.ndarray, dt: float, dx0: float, ids, aux=None):
        q = np.ascontiguousarray(q, np.float64)
        ids = np.ascontiguousarray(ids, np.int64)
        P, meq, m, _ = q.shape
        out = np.zeros((len(ids), meq, m, m))
        cfl = np.zeros(len(ids))
        ap = None if aux is None else np.ascontiguousarray(aux, np.float64)
        rc = lib().orc_step_sample(self.h, C.byref(pr), _p(q), None if ap is None else _p(ap), dt,
                                   dx0, _p(ids), len(ids), _p(out), _p(cfl))
        if rc:
            raise RuntimeError(f"orc_step_sample -> {rc}")
        return out, cfl

    def padded_sample(self, q: np.ndarray, p: int) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float64)
        meq, m = q.shape[1], q.shape[2]
        out = np.zeros((meq, m + 4, m + 4))
        rc = lib().orc_build_padded_sample(self.h, _p(q), meq, p, _p(out))
        if rc:
            raise RuntimeError(f"orc_build_padded_sample -> {rc}")
        return out


def forest_for(w) -> OracleForest:
    return OracleForest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m)


def problem_for(w) -> Problem:
    return problem(w.kind, w.params, w.limiter, w.method2, w.method3, getattr(w, "reflux", 0))


def run(w, steps: int | None = None, dt_list=None, nthreads: int = 1, forest=None):
    """Run the workload's dt policy for `steps` steps on the oracle.
    Returns (q [P][meqn][m][m], cfls, dts).  With dt_list the dt sequence is replayed."""
    f = forest or forest_for(w)
    pr = problem_for(w)
    steps = w.steps if steps is None else steps
    qp = f.pad(w.q0)
    dx0 = 1.0 / w.m
    dt = w.dt0
    cfls, dts = [], []
    for n in range(steps):
        if dt_list is not None:
            dt = dt_list[n]
        out, cfl = f.step(pr, qp, dt, dx0, w.aux, nthreads)
        if cfl > w.cfl_reject and dt_list is None:
            # Clawpack retake with dt * target / cfl (state unchanged)
            dt = dt * w.cfl_target / cfl
            out, cfl = f.step(pr, qp, dt, dx0, w.aux, nthreads)
        cfls.append(cfl)
        dts.append(dt)
        qp = out
        if dt_list is None:
            dt = w.next_dt(dt, cfl)
    m = w.m
    return np.ascontiguousarray(qp[:, :, 2:m + 2, 2:m + 2]), np.array(cfls), np.array(dts)


def run_subcycled(w, steps: int | None = None, dt_list=None, forest=None):
    """Sub-cycled driver (subcycle.c): each step advances the coarsest level by dt_coarse and every
    finer level l by dt_coarse 2^-(l - lmin).  dt_coarse starts at w.dt0 * 2^(lmax - lmin) (the
    workload's dt0 is the finest level's) and follows the workload's policy on the returned CFL.
    Returns (q [P][meqn][m][m], cfls, dt_coarse list)."""
    f = forest or forest_for(w)
    pr = problem_for(w)
    steps = w.steps if steps is None else steps
    qp = f.pad(w.q0)
    dx0 = 1.0 / w.m
    lv = w.forest.levels
    dt = w.dt0 * 2.0 ** (int(lv.max()) - int(lv.min()))
    cfls, dts = [], []
    for n in range(steps):
        if dt_list is not None:
            dt = dt_list[n]
        out, cfl = f.step_subcycled(pr, qp, dt, dx0, w.aux)
        if cfl > w.cfl_reject and dt_list is None:
            dt = dt * w.cfl_target / cfl
            out, cfl = f.step_subcycled(pr, qp, dt, dx0, w.aux)
        cfls.append(cfl)
        dts.append(dt)
        qp = out
        if dt_list is None:
            dt = w.next_dt(dt, cfl)
    m = w.m
    return np.ascontiguousarray(qp[:, :, 2:m + 2, 2:m + 2]), np.array(cfls), np.array(dts)
