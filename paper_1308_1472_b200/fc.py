"""Thin ctypes binding of libfc.so (include/fc.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  There is no fallback: if libfc.so is missing or a
call fails, an exception is raised.

Names follow the C ABI: fc_forest_create, fc_set_problem, fc_set_aux, fc_set_q, fc_ghost_fill,
fc_step, fc_get_q, fc_get_q_padded, fc_get_ghost_table, ... ; `Forest` bundles them per handle.
Host buffers are numpy arrays; device buffers are torch CUDA tensors (passed by data_ptr()).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FC_LIB_PATH") or os.path.join(HERE, "libfc.so")   # (override: tuning builds)

FC_OK, FC_EINVAL, FC_ETILING, FC_ECONN, FC_EBALANCE, FC_ECUDA, FC_ENCCL, FC_ENOMEM, FC_ESTATE, \
    FC_ECFL, FC_ENONFINITE, FC_EUNSUP = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9, -10, -11
FC_HOST, FC_DEVICE = 0, 1
FC_ADV_CONST, FC_ADV_EDGEVEL_CAPA, FC_SWE_ROE, FC_EULER_ROE, FC_EULER_HLLE = 0, 1, 2, 3, 4
FC_LIM_NONE, FC_LIM_MINMOD, FC_LIM_MC = 0, 1, 2
FC_TABLE_EXPANDED = 1
FC_TABLE_COMPACT = 2

ERRNAMES = {0: "FC_OK", -1: "FC_EINVAL", -2: "FC_ETILING", -3: "FC_ECONN", -4: "FC_EBALANCE",
            -5: "FC_ECUDA", -6: "FC_ENCCL", -7: "FC_ENOMEM", -8: "FC_ESTATE", -9: "FC_ECFL",
            -10: "FC_ENONFINITE", -11: "FC_EUNSUP"}

# every symbol include/fc.h declares (checked by the CPU test suite)
EXPORTS = ["fc_forest_create", "fc_forest_destroy", "fc_set_problem", "fc_set_aux", "fc_set_q",
           "fc_ghost_fill", "fc_step", "fc_get_q", "fc_get_q_padded", "fc_get_ghost_table",
           "fc_set_stream", "fc_set_timing", "fc_get_stats", "fc_reset_stats", "fc_local_range",
           "fc_halo_counts", "fc_halo_requests", "fc_halo_set_requests", "fc_halo_finalize",
           "fc_halo_buffers", "fc_halo_pack", "fc_halo_unpack", "fc_step_local", "fc_commit",
           "fc_nccl_unique_id", "fc_last_error", "fc_step_subcycled", "fc_regrid", "fc_get_leaves",
           "fc_p2p_buffers", "fc_p2p_set_peer", "fc_run", "fc_reflux_requests", "fc_reflux_set_requests",
           "fc_reflux_finalize", "fc_reflux_buffers", "fc_regrid_fill", "fc_regrid_tags", "fc_regrid_begin",
           "fc_regrid_buffers", "fc_regrid_finish"]


class FcError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where} -> {ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class ForestDesc(C.Structure):
    _fields_ = [("num_patches", C.c_int64), ("levels", C.c_void_p), ("tree_ids", C.c_void_p),
                ("num_trees", C.c_int32), ("tree_to_tree", C.c_void_p), ("tree_to_face", C.c_void_p),
                ("face_bc", C.c_void_p), ("m", C.c_int32), ("mbc", C.c_int32), ("meqn", C.c_int32),
                ("maux", C.c_int32), ("tree_dx0", C.c_double), ("device", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id", C.c_void_p),
                ("halo_p2p", C.c_int32), ("partition", C.c_void_p)]


class Problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p0", C.c_double), ("p1", C.c_double), ("limiter", C.c_int32),
                ("method2", C.c_int32), ("method3", C.c_int32), ("cfl_reject", C.c_double),
                ("skip_quiescent", C.c_int32), ("reflux", C.c_int32)]


class RegridParams(C.Structure):
    _fields_ = [("refine_threshold", C.c_double), ("coarsen_threshold", C.c_double),
                ("min_level", C.c_int32), ("max_level", C.c_int32), ("level_weights", C.c_int32),
                ("pad_", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("steps", C.c_int64), ("ms_ghost", C.c_double),
                ("ms_step", C.c_double), ("ms_comm", C.c_double), ("step_kernel_launches", C.c_int64),
                ("local_patches", C.c_int64), ("halo_cells", C.c_int64),
                ("uniform_fast_path", C.c_int32), ("pad_", C.c_int32), ("ms_copy", C.c_double),
                ("copy_launches", C.c_int64), ("regular_patches", C.c_int64),
                ("quad_blocks", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


_lib = None


def lib():
    """Load libfc.so (raises if it has not been built -- there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1308_1472_b200.build` "
                              "(the product path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.fc_forest_create.argtypes = [C.POINTER(ForestDesc), C.POINTER(P)]
        L.fc_forest_destroy.argtypes = [P]
        L.fc_set_problem.argtypes = [P, C.POINTER(Problem)]
        L.fc_set_aux.argtypes = [P, P, C.c_int]
        L.fc_set_q.argtypes = [P, P, C.c_int]
        L.fc_ghost_fill.argtypes = [P]
        L.fc_step.argtypes = [P, C.c_double, C.POINTER(C.c_double)]
        L.fc_step_subcycled.argtypes = [P, C.c_double, C.POINTER(C.c_double)]
        L.fc_regrid.argtypes = [P, C.POINTER(RegridParams), C.POINTER(P)]
        L.fc_get_leaves.argtypes = [P, P, P, C.c_int64, C.POINTER(C.c_int64)]
        L.fc_p2p_buffers.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_int32)]
        L.fc_p2p_set_peer.argtypes = [P, C.c_int32, P, P]
        L.fc_run.argtypes = [P, C.c_double, C.c_int64, P, C.POINTER(C.c_double)]
        L.fc_get_q.argtypes = [P, P, C.c_int]
        L.fc_get_q_padded.argtypes = [P, P, C.c_int]
        L.fc_get_ghost_table.argtypes = [P, C.c_int, P, C.c_int64, C.POINTER(C.c_int64)]
        L.fc_set_stream.argtypes = [P, P]
        L.fc_set_timing.argtypes = [P, C.c_int]
        L.fc_get_stats.argtypes = [P, C.POINTER(Stats)]
        L.fc_reset_stats.argtypes = [P]
        L.fc_local_range.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.fc_halo_counts.argtypes = [P, P]
        L.fc_halo_requests.argtypes = [P, C.c_int, C.c_int, P, C.c_int64, C.POINTER(C.c_int64)]
        L.fc_halo_set_requests.argtypes = [P, C.c_int, C.c_int, P, C.c_int64]
        L.fc_halo_finalize.argtypes = [P]
        L.fc_halo_buffers.argtypes = [P, C.c_int, C.POINTER(P), C.POINTER(P), P, P]
        L.fc_reflux_requests.argtypes = [P, C.c_int, P, C.c_int64, C.POINTER(C.c_int64)]
        L.fc_reflux_set_requests.argtypes = [P, C.c_int, P, C.c_int64]
        L.fc_reflux_finalize.argtypes = [P]
        L.fc_reflux_buffers.argtypes = [P, C.POINTER(P), C.POINTER(P), P, P]
        L.fc_regrid_fill.argtypes = [P, C.c_int]
        L.fc_regrid_tags.argtypes = [P, P]
        L.fc_regrid_begin.argtypes = [P, P, C.POINTER(RegridParams), C.POINTER(P)]
        L.fc_regrid_buffers.argtypes = [P, P, C.POINTER(P), C.POINTER(P), P, P]
        L.fc_regrid_finish.argtypes = [P]
        L.fc_halo_pack.argtypes = [P, C.c_int]
        L.fc_halo_unpack.argtypes = [P, C.c_int]
        L.fc_step_local.argtypes = [P, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.fc_commit.argtypes = [P, C.c_double]
        L.fc_nccl_unique_id.argtypes = [P]
        L.fc_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != FC_OK:
        raise FcError(rc, where, lib().fc_last_error().decode())


def _ptr(a):
    """numpy array -> (ptr, FC_HOST); torch tensor -> (data_ptr, FC_HOST/FC_DEVICE)."""
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous and a.dtype == np.float64
        return a.ctypes.data_as(C.c_void_p), FC_HOST
    import torch
    assert a.is_contiguous() and a.dtype == torch.float64
    return C.c_void_p(a.data_ptr()), (FC_DEVICE if a.is_cuda else FC_HOST)


def fc_nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().fc_nccl_unique_id(buf), "fc_nccl_unique_id")
    return bytes(buf)


class Forest:
    """One libfc handle (one per process / GPU)."""

    def __init__(self, levels, tree_ids, conn, m: int, meqn: int, maux: int = 0,
                 tree_dx0: float = 1.0, device: int = 0, rank: int = 0, nranks: int = 1,
                 nccl_id: bytes | None = None, halo_p2p: int = 0, partition=None):
        self._keep = [np.ascontiguousarray(levels, np.int8), np.ascontiguousarray(tree_ids, np.int32),
                      np.ascontiguousarray(conn.tree_to_tree, np.int32),
                      np.ascontiguousarray(conn.tree_to_face, np.int8),
                      np.ascontiguousarray(conn.face_bc, np.int8)]
        lv, tr, t2t, t2f, fbc = self._keep
        part = None if partition is None else np.ascontiguousarray(partition, np.int64)
        self._keep.append(part)
        self._nid = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        d = ForestDesc(len(lv), lv.ctypes.data, tr.ctypes.data, len(t2t) // 4, t2t.ctypes.data,
                       t2f.ctypes.data, fbc.ctypes.data, m, 2, meqn, maux, tree_dx0, device, rank,
                       nranks, C.cast(self._nid, C.c_void_p) if self._nid else None, halo_p2p,
                       part.ctypes.data if part is not None else None)
        h = C.c_void_p()
        _check(lib().fc_forest_create(C.byref(d), C.byref(h)), "fc_forest_create")
        self.h = h
        self.m, self.meqn, self.maux, self.n = m, meqn, maux, m + 4
        first, count = C.c_int64(), C.c_int64()
        _check(lib().fc_local_range(h, C.byref(first), C.byref(count)), "fc_local_range")
        self.first, self.count = first.value, count.value
        self.nranks = nranks

    def close(self):
        if getattr(self, "h", None):
            lib().fc_forest_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- calls -----------------------------------------------------------------------------------
    def set_problem(self, kind, p0=0.0, p1=0.0, limiter=FC_LIM_MC, method2=2, method3=2,
                    cfl_reject=1.0, skip_quiescent=1, reflux=0):
        pr = Problem(kind, p0, p1, limiter, method2, method3, cfl_reject, skip_quiescent, reflux)
        _check(lib().fc_set_problem(self.h, C.byref(pr)), "fc_set_problem")

    def set_aux(self, aux):
        p, where = _ptr(aux)
        _check(lib().fc_set_aux(self.h, p, where), "fc_set_aux")

    def set_q(self, q):
        p, where = _ptr(q)
        _check(lib().fc_set_q(self.h, p, where), "fc_set_q")

    def ghost_fill(self):
        _check(lib().fc_ghost_fill(self.h), "fc_ghost_fill")

    def step(self, dt: float, raise_on_reject: bool = True):
        """Returns (rc, cfl).  rc is FC_OK, or FC_ECFL / FC_ENONFINITE when not committed."""
        cfl = C.c_double(0.0)
        rc = lib().fc_step(self.h, dt, C.byref(cfl))
        if rc not in (FC_OK, FC_ECFL) or (raise_on_reject and rc != FC_OK):
            _check(rc, "fc_step")
        return rc, cfl.value

    def run(self, dt: float, nsteps: int, raise_on_reject: bool = True):
        """fc_run: nsteps fixed-dt steps replayed as CUDA graphs -> (rc, cfls[nsteps])."""
        cfls = np.zeros(max(1, nsteps))
        mx = C.c_double(0.0)
        rc = lib().fc_run(self.h, dt, nsteps, cfls.ctypes.data_as(C.c_void_p), C.byref(mx))
        if rc not in (FC_OK, FC_ECFL) or (raise_on_reject and rc != FC_OK):
            _check(rc, "fc_run")
        return rc, cfls[:nsteps]

    def step_subcycled(self, dt_coarse: float, raise_on_reject: bool = True):
        """One sub-cycled step (coarsest level by dt_coarse, finer levels by halves); (rc, cfl)."""
        cfl = C.c_double(0.0)
        rc = lib().fc_step_subcycled(self.h, dt_coarse, C.byref(cfl))
        if rc not in (FC_OK, FC_ECFL) or (raise_on_reject and rc != FC_OK):
            _check(rc, "fc_step_subcycled")
        return rc, cfl.value

    def regrid(self, refine_threshold: float, coarsen_threshold: float, min_level: int, max_level: int,
               level_weights: int = 0):
        """Dynamic regrid (fc_regrid) -> a new Forest on the new mesh (problem and q carried over;
        aux must be set again for the capacity form).  This handle stays valid."""
        rp = RegridParams(refine_threshold, coarsen_threshold, min_level, max_level, level_weights)
        h = C.c_void_p()
        _check(lib().fc_regrid(self.h, C.byref(rp), C.byref(h)), "fc_regrid")
        return self._wrap(h)

    def p2p_buffers(self):
        """(buf0, buf1, parity): this rank's two state buffers (device addresses) and which is q_old."""
        b0, b1, par = C.c_void_p(), C.c_void_p(), C.c_int32()
        _check(lib().fc_p2p_buffers(self.h, C.byref(b0), C.byref(b1), C.byref(par)), "fc_p2p_buffers")
        return b0.value, b1.value, par.value

    def p2p_set_peer(self, peer: int, buf0: int, buf1: int):
        _check(lib().fc_p2p_set_peer(self.h, peer, C.c_void_p(buf0), C.c_void_p(buf1)), "fc_p2p_set_peer")

    def leaves(self):
        """(levels int8[P], tree_ids int32[P]) of the forest in global Morton order."""
        n = C.c_int64()
        _check(lib().fc_get_leaves(self.h, None, None, 0, C.byref(n)), "fc_get_leaves")
        lv = np.zeros(n.value, np.int8)
        tr = np.zeros(n.value, np.int32)
        _check(lib().fc_get_leaves(self.h, lv.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p),
                                   n.value, C.byref(n)), "fc_get_leaves")
        return lv, tr

    def get_q(self, out=None):
        if out is None:
            out = np.empty((self.count, self.meqn, self.m, self.m))
        p, where = _ptr(out)
        _check(lib().fc_get_q(self.h, p, where), "fc_get_q")
        return out

    def get_q_padded(self, out=None):
        if out is None:
            out = np.empty((self.count, self.meqn, self.n, self.n))
        p, where = _ptr(out)
        _check(lib().fc_get_q_padded(self.h, p, where), "fc_get_q_padded")
        return out

    def ghost_table(self, which: int = FC_TABLE_EXPANDED) -> np.ndarray:
        """EXPANDED: [P_local][G][8] per ring cell; COMPACT: [P_local][8 directions][5]."""
        n = C.c_int64()
        lib().fc_get_ghost_table(self.h, which, None, 0, C.byref(n))
        buf = np.empty(n.value, np.int32)
        _check(lib().fc_get_ghost_table(self.h, which, buf.ctypes.data_as(C.c_void_p),
                                        n.value, C.byref(n)), "fc_get_ghost_table")
        if which == FC_TABLE_COMPACT:
            return buf.reshape(self.count, 8, 5)
        G = self.n * self.n - self.m * self.m
        return buf.reshape(self.count, G, 8)

    def set_stream(self, stream_ptr: int | None):
        _check(lib().fc_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None), "fc_set_stream")

    def set_timing(self, on: bool):
        _check(lib().fc_set_timing(self.h, 1 if on else 0), "fc_set_timing")

    def stats(self) -> dict:
        s = Stats()
        _check(lib().fc_get_stats(self.h, C.byref(s)), "fc_get_stats")
        return s.as_dict()

    def reset_stats(self):
        _check(lib().fc_reset_stats(self.h), "fc_reset_stats")

    def halo_requests(self, peer: int, round_: int) -> np.ndarray:
        n = C.c_int64()
        lib().fc_halo_requests(self.h, peer, round_, None, 0, C.byref(n))
        buf = np.empty(max(1, n.value), np.int64)
        _check(lib().fc_halo_requests(self.h, peer, round_, buf.ctypes.data_as(C.c_void_p), n.value,
                                      C.byref(n)), "fc_halo_requests")
        return buf[:n.value]

    # -- manual halo transport (staged step) --------------------------------------------------
    def halo_set_requests(self, round_: int, peer: int, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, np.int64)
        _check(lib().fc_halo_set_requests(self.h, round_, peer, keys.ctypes.data_as(C.c_void_p), len(keys)),
               "fc_halo_set_requests")

    def halo_finalize(self):
        _check(lib().fc_halo_finalize(self.h), "fc_halo_finalize")

    def _wrap(self, h):
        g = Forest.__new__(Forest)
        g.h = h
        g._keep, g._nid = [], None
        g.m, g.meqn, g.maux, g.n = self.m, self.meqn, self.maux, self.n
        first, count = C.c_int64(), C.c_int64()
        _check(lib().fc_local_range(h, C.byref(first), C.byref(count)), "fc_local_range")
        g.first, g.count, g.nranks = first.value, count.value, self.nranks
        return g

    def regrid_fill(self, phase: int):
        _check(lib().fc_regrid_fill(self.h, phase), "fc_regrid_fill")

    def regrid_tags(self) -> np.ndarray:
        t = np.zeros(max(1, self.count))
        _check(lib().fc_regrid_tags(self.h, t.ctypes.data_as(C.c_void_p)), "fc_regrid_tags")
        return t[:self.count]

    def regrid_begin(self, global_tags: np.ndarray, refine_threshold: float, coarsen_threshold: float,
                     min_level: int, max_level: int, level_weights: int = 0):
        gt = np.ascontiguousarray(global_tags, np.float64)
        rp = RegridParams(refine_threshold, coarsen_threshold, min_level, max_level, level_weights)
        h = C.c_void_p()
        _check(lib().fc_regrid_begin(self.h, gt.ctypes.data_as(C.c_void_p), C.byref(rp), C.byref(h)),
               "fc_regrid_begin")
        return self._wrap(h)

    def regrid_buffers(self, new):
        s, r = C.c_void_p(), C.c_void_p()
        so = np.zeros(self.nranks + 1, np.int64)
        ro = np.zeros(self.nranks + 1, np.int64)
        _check(lib().fc_regrid_buffers(self.h, new.h, C.byref(s), C.byref(r), so.ctypes.data_as(C.c_void_p),
                                       ro.ctypes.data_as(C.c_void_p)), "fc_regrid_buffers")
        return s.value, r.value, so, ro

    def regrid_finish(self):
        _check(lib().fc_regrid_finish(self.h), "fc_regrid_finish")

    def reflux_requests(self, peer: int) -> np.ndarray:
        n = C.c_int64()
        _check(lib().fc_reflux_requests(self.h, peer, None, 0, C.byref(n)), "fc_reflux_requests")
        buf = np.zeros(max(1, n.value), np.int64)
        _check(lib().fc_reflux_requests(self.h, peer, buf.ctypes.data_as(C.c_void_p), len(buf), C.byref(n)),
               "fc_reflux_requests")
        return buf[:n.value]

    def reflux_set_requests(self, peer: int, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, np.int64)
        _check(lib().fc_reflux_set_requests(self.h, peer, keys.ctypes.data_as(C.c_void_p), len(keys)),
               "fc_reflux_set_requests")

    def reflux_finalize(self):
        _check(lib().fc_reflux_finalize(self.h), "fc_reflux_finalize")

    def reflux_buffers(self):
        s, r = C.c_void_p(), C.c_void_p()
        so = np.zeros(self.nranks + 1, np.int64)
        ro = np.zeros(self.nranks + 1, np.int64)
        _check(lib().fc_reflux_buffers(self.h, C.byref(s), C.byref(r), so.ctypes.data_as(C.c_void_p),
                                       ro.ctypes.data_as(C.c_void_p)), "fc_reflux_buffers")
        return s.value, r.value, so, ro

    def halo_buffers(self, round_: int):
        s, r = C.c_void_p(), C.c_void_p()
        so = np.zeros(self.nranks + 1, np.int64)
        ro = np.zeros(self.nranks + 1, np.int64)
        _check(lib().fc_halo_buffers(self.h, round_, C.byref(s), C.byref(r), so.ctypes.data_as(C.c_void_p),
                                     ro.ctypes.data_as(C.c_void_p)), "fc_halo_buffers")
        return s.value, r.value, so, ro

    def halo_pack(self, round_: int):
        _check(lib().fc_halo_pack(self.h, round_), "fc_halo_pack")

    def halo_unpack(self, round_: int):
        _check(lib().fc_halo_unpack(self.h, round_), "fc_halo_unpack")

    def step_local(self, dt: float, phase: int) -> float:
        c = C.c_double(0.0)
        _check(lib().fc_step_local(self.h, dt, phase, C.byref(c)), "fc_step_local")
        return c.value

    def commit(self, global_cfl: float) -> int:
        rc = lib().fc_commit(self.h, global_cfl)
        if rc not in (FC_OK, FC_ECFL):
            _check(rc, "fc_commit")
        return rc

    def halo_counts(self) -> np.ndarray:
        out = np.zeros(self.nranks, np.int64)
        _check(lib().fc_halo_counts(self.h, out.ctypes.data_as(C.c_void_p)), "fc_halo_counts")
        return out


def forest_for(w, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id=None,
               skip_quiescent: int = 1) -> Forest:
    """Handle for a workloads.Workload, with its problem (and aux, for local patches) set."""
    f = Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0,
               device, rank, nranks, nccl_id)
    if device >= 0:
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject,
                      skip_quiescent, getattr(w, "reflux", 0))
        if w.aux is not None:
            f.set_aux(np.ascontiguousarray(w.aux[f.first:f.first + f.count]))
    return f


def run(w, steps: int | None = None, dt_list=None, device: int = 0, f: Forest | None = None,
        skip_quiescent: int = 1):
    """Run the workload's dt policy on the GPU (same policy as the oracle's driver).
    Returns (q [P][meqn][m][m], cfls, dts)."""
    f = f or forest_for(w, device, skip_quiescent=skip_quiescent)
    f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    steps = w.steps if steps is None else steps
    dt = w.dt0
    cfls, dts = [], []
    for n in range(steps):
        if dt_list is not None:
            dt = dt_list[n]
        rc, cfl = f.step(dt, raise_on_reject=dt_list is not None)
        if rc == FC_ECFL:
            dt = dt * w.cfl_target / cfl
            rc, cfl = f.step(dt)
        cfls.append(cfl)
        dts.append(dt)
        if dt_list is None:
            dt = w.next_dt(dt, cfl)
    return f.get_q(), np.array(cfls), np.array(dts)


def run_subcycled(w, steps: int | None = None, dt_list=None, device: int = 0, f: Forest | None = None,
                  skip_quiescent: int = 1):
    """Sub-cycled driver (same policy as oracle.run_subcycled): dt_coarse starts at
    w.dt0 * 2^(lmax - lmin).  Returns (q, cfls, dt_coarse list)."""
    f = f or forest_for(w, device, skip_quiescent=skip_quiescent)
    f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    steps = w.steps if steps is None else steps
    lv = w.forest.levels
    dt = w.dt0 * 2.0 ** (int(lv.max()) - int(lv.min()))
    cfls, dts = [], []
    for n in range(steps):
        if dt_list is not None:
            dt = dt_list[n]
        rc, cfl = f.step_subcycled(dt, raise_on_reject=dt_list is not None)
        if rc == FC_ECFL:
            dt = dt * w.cfl_target / cfl
            rc, cfl = f.step_subcycled(dt)
        cfls.append(cfl)
        dts.append(dt)
        if dt_list is None:
            dt = w.next_dt(dt, cfl)
    return f.get_q(), np.array(cfls), np.array(dts)
