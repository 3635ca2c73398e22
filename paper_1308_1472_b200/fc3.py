"""ctypes binding of the octree ABI (include/fc3.h): argument marshalling only -- every step of the
path runs in libfc.so's kernels (there is no CPU fallback; the import raises without the library).
Names follow fc3.h; `Forest3` bundles the calls of one handle."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .fc import FC_LIM_MC, FC_OK, _check, _ptr, lib as _lib

EXPORTS3 = ["fc3_forest_create", "fc3_forest_destroy", "fc3_set_problem", "fc3_set_q", "fc3_ghost_fill",
            "fc3_step", "fc3_get_q", "fc3_get_q_padded", "fc3_get_ghost_table", "fc3_set_stream"]


class Forest3Desc(C.Structure):
    _fields_ = [("num_patches", C.c_int64), ("levels", C.c_void_p), ("tree_ids", C.c_void_p),
                ("m", C.c_int32), ("num_trees", C.c_int32), ("tree_to_tree", C.c_void_p),
                ("face_bc", C.c_void_p), ("tree_dx0", C.c_double), ("device", C.c_int32)]


_init = False


def lib():
    global _init
    L = _lib()
    if not _init:
        P = C.c_void_p
        L.fc3_forest_create.argtypes = [C.POINTER(Forest3Desc), C.POINTER(P)]
        L.fc3_forest_destroy.argtypes = [P]
        L.fc3_set_problem.argtypes = [P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double]
        L.fc3_set_q.argtypes = [P, P, C.c_int]
        L.fc3_ghost_fill.argtypes = [P]
        L.fc3_step.argtypes = [P, C.c_double, C.POINTER(C.c_double)]
        L.fc3_get_q.argtypes = [P, P, C.c_int]
        L.fc3_get_q_padded.argtypes = [P, P, C.c_int]
        L.fc3_get_ghost_table.argtypes = [P, P, C.c_int64, C.POINTER(C.c_int64)]
        L.fc3_set_stream.argtypes = [P, P]
        _init = True
    return L


class Forest3:
    def __init__(self, forest, m: int, device: int = 0, tree_dx0: float = 1.0):
        self._keep = [np.ascontiguousarray(forest.levels, np.int8), np.ascontiguousarray(forest.tree_ids, np.int32),
                      np.ascontiguousarray(forest.t2t, np.int32), np.ascontiguousarray(forest.fbc, np.int8)]
        lv, tr, t2t, fbc = self._keep
        d = Forest3Desc(len(lv), lv.ctypes.data, tr.ctypes.data, m, len(t2t) // 6, t2t.ctypes.data,
                        fbc.ctypes.data, tree_dx0, device)
        self.h = C.c_void_p()
        _check(lib().fc3_forest_create(C.byref(d), C.byref(self.h)), "fc3_forest_create")
        self.P, self.m = len(lv), m

    def close(self):
        if self.h:
            lib().fc3_forest_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_problem(self, vel, limiter=FC_LIM_MC, method2=2, cfl_reject=1.0):
        _check(lib().fc3_set_problem(self.h, float(vel[0]), float(vel[1]), float(vel[2]), limiter, method2,
                                     cfl_reject), "fc3_set_problem")

    def set_q(self, q):
        p, where = _ptr(q)
        _check(lib().fc3_set_q(self.h, p, where), "fc3_set_q")

    def set_stream(self, stream_ptr):
        _check(lib().fc3_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None), "fc3_set_stream")

    def ghost_fill(self):
        _check(lib().fc3_ghost_fill(self.h), "fc3_ghost_fill")

    def step(self, dt: float, raise_on_reject: bool = True):
        c = C.c_double(0.0)
        rc = lib().fc3_step(self.h, dt, C.byref(c))
        if rc != FC_OK and raise_on_reject:
            _check(rc, "fc3_step")
        return rc, c.value

    def get_q(self):
        m = self.m
        out = np.empty((self.P, m, m, m))
        _check(lib().fc3_get_q(self.h, out.ctypes.data_as(C.c_void_p), 0), "fc3_get_q")
        return out

    def get_q_padded(self):
        n = self.m + 4
        out = np.empty((self.P, n, n, n))
        _check(lib().fc3_get_q_padded(self.h, out.ctypes.data_as(C.c_void_p), 0), "fc3_get_q_padded")
        return out

    def ghost_table(self):
        n = C.c_int64()
        lib().fc3_get_ghost_table(self.h, None, 0, C.byref(n))
        buf = np.empty(n.value, np.int32)
        _check(lib().fc3_get_ghost_table(self.h, buf.ctypes.data_as(C.c_void_p), n.value, C.byref(n)),
               "fc3_get_ghost_table")
        G = (self.m + 4) ** 3 - self.m ** 3
        return buf.reshape(self.P, G, 8)


def run3(forest, m, q0, vel, dt, steps, device=0, limiter=FC_LIM_MC, method2=2):
    """fixed-dt steps on the GPU -> (interiors [P][m][m][m], cfls)."""
    f = Forest3(forest, m, device)
    f.set_problem(vel, limiter, method2)
    f.set_q(np.ascontiguousarray(q0, np.float64))
    cfls = [f.step(dt)[1] for _ in range(steps)]
    q = f.get_q()
    f.close()
    return q, np.array(cfls)
