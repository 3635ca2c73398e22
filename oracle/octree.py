"""ctypes binding of the octree oracle (forest3.c).  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).
Cites: the C sources (reading 26)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import lib as _lib, _p

OP_COPY, OP_AVG8, OP_INTERP, OP_BCX, OP_BCY, OP_BCZ = 1, 2, 3, 4, 5, 6
_init = False


def lib():
    global _init
    L = _lib()
    if not _init:
        P = C.c_void_p
        L.orc3_forest_create.argtypes = [C.c_int64, P, P, C.c_int32, P, P, C.c_int, C.POINTER(P)]
        L.orc3_forest_destroy.argtypes = [P]
        L.orc3_forest_coords.argtypes = [P, P, P, P, C.POINTER(C.c_int)]
        L.orc3_ring_count.argtypes = [C.c_int]
        L.orc3_ghost_records.argtypes = [P, C.c_int64, P]
        L.orc3_ghost_table.argtypes = [P, P]
        L.orc3_ghost_fill.argtypes = [P, P]
        L.orc3_step_patch.argtypes = [P, P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                      C.c_double, P]
        L.orc3_step_patch.restype = C.c_double
        L.orc3_step.argtypes = [P, P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                C.c_double, P, C.POINTER(C.c_double)]
        _init = True
    return L


class OracleForest3:
    def __init__(self, forest, m: int):
        self.levels = np.ascontiguousarray(forest.levels, np.int8)
        self.tree_ids = np.ascontiguousarray(forest.tree_ids, np.int32)
        self.t2t = np.ascontiguousarray(forest.t2t, np.int32)
        self.fbc = np.ascontiguousarray(forest.fbc, np.int8)
        self.m = m
        self.P = len(self.levels)
        self.h = C.c_void_p()
        rc = lib().orc3_forest_create(self.P, _p(self.levels), _p(self.tree_ids), len(self.t2t) // 6,
                                      _p(self.t2t), _p(self.fbc), m, C.byref(self.h))
        if rc:
            raise ValueError(f"orc3_forest_create -> {rc}")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc3_forest_destroy(self.h)
            self.h = None

    @property
    def n(self):
        return self.m + 4

    @property
    def G(self):
        return lib().orc3_ring_count(self.m)

    def coords(self):
        x, y, z = (np.zeros(self.P, np.int64) for _ in range(3))
        lm = C.c_int()
        lib().orc3_forest_coords(self.h, _p(x), _p(y), _p(z), C.byref(lm))
        return x, y, z, lm.value

    def ghost_table(self) -> np.ndarray:
        rec = np.zeros((self.P, self.G, 8), np.int32)
        rc = lib().orc3_ghost_table(self.h, _p(rec))
        if rc:
            raise ValueError(f"orc3_ghost_table -> {rc}")
        return rec

    def pad(self, q: np.ndarray) -> np.ndarray:
        """[P][m][m][m] interiors (index [p][k][j][i]) -> [P][n][n][n] with a NaN ring."""
        m, n = self.m, self.n
        out = np.full((self.P, n, n, n), np.nan)
        out[:, 2:m + 2, 2:m + 2, 2:m + 2] = q
        return out

    def ghost_fill(self, qpad: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(qpad, np.float64).copy()
        rc = lib().orc3_ghost_fill(self.h, _p(q))
        if rc:
            raise ValueError(f"orc3_ghost_fill -> {rc}")
        return q

    def step(self, qpad, vel, dt, dx0, limiter=2, method2=2):
        q = np.ascontiguousarray(qpad, np.float64).copy()
        out = np.empty_like(q)
        cfl = C.c_double()
        rc = lib().orc3_step(self.h, _p(q), float(vel[0]), float(vel[1]), float(vel[2]), limiter, method2, dt, dx0,
                             _p(out), C.byref(cfl))
        if rc:
            raise ValueError(f"orc3_step -> {rc}")
        return out, cfl.value


def run3(forest, m, q0, vel, dt, steps, dx0=None, limiter=2, method2=2):
    """steps fixed-dt split steps from interiors q0 [P][m][m][m] -> (interiors, cfls)."""
    f = OracleForest3(forest, m)
    dx0 = 1.0 / m if dx0 is None else dx0
    qp = f.pad(q0)
    cfls = []
    for _ in range(steps):
        qp, c = f.step(qp, vel, dt, dx0, limiter, method2)
        cfls.append(c)
    return np.ascontiguousarray(qp[:, 2:m + 2, 2:m + 2, 2:m + 2]), np.array(cfls)
