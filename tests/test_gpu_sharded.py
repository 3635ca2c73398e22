"""The sharded (multi-GPU) data path on one GPU: R rank handles in one process with the manual
halo transport (include/fc.h "staged step"), halo buffers moved between the ranks with plain
device copies in place of ncclSend/ncclRecv, the CFL max taken over the ranks.  Everything else --
request exchange, pack / unpack lists, halo slots in virtual patches, round-2 exchange of coarse
ring cells for interpolation, the fused ring gather through halo slots, remote neighbours in the
quiescent filter -- is the production code.  The concatenated result must equal the one-rank run
bitwise (shard-count invariance) and the oracle within tolerance."""
import ctypes as C
import glob
import os

import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads.configs import c1, c2, c3, c5
from workloads.cubed_sphere import c4_workload

pytestmark = pytest.mark.gpu

_cudart = None


def d2d(dst: int, src: int, nbytes: int):
    global _cudart
    if _cudart is None:
        import nvidia.cuda_runtime as cr
        path = sorted(glob.glob(os.path.join(os.path.dirname(cr.__file__), "lib", "libcudart.so*")))[0]
        _cudart = C.CDLL(path)
        _cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    if nbytes:
        assert _cudart.cudaMemcpy(C.c_void_p(int(dst)), C.c_void_p(int(src)), int(nbytes), 3) == 0


def run_sharded(w, R, dts, skip, reflux=0, partition=None):
    hs = []
    for r in range(R):
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0, 0, r, R, None,
                      partition=partition)
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject, skip, reflux)
        if w.aux is not None:
            f.set_aux(np.ascontiguousarray(w.aux[f.first:f.first + f.count]))
        hs.append(f)
    for rnd in (1, 2):
        for r in range(R):
            for s in range(R):
                if s != r:
                    hs[s].halo_set_requests(rnd, r, hs[r].halo_requests(s, rnd))
    for f in hs:
        f.halo_finalize()
        f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    if reflux:   # fine faces of other ranks' coarse cells (fc_reflux_*)
        for r in range(R):
            for s in range(R):
                if s != r:
                    hs[s].reflux_set_requests(r, hs[r].reflux_requests(s))
        for f in hs:
            f.reflux_finalize()

    def move(bufs):
        for r in range(R):
            _, recv, _, roff = bufs[r]
            for s in range(R):
                if s == r:
                    continue
                send, _, soff, _ = bufs[s]
                n = roff[s + 1] - roff[s]
                assert n == soff[r + 1] - soff[r]
                d2d(recv + 8 * roff[s], send + 8 * soff[r], 8 * n)

    def exchange(rnd):
        for f in hs:
            f.halo_pack(rnd)
        bufs = [f.halo_buffers(rnd) for f in hs]
        for r in range(R):
            _, recv, _, roff = bufs[r]
            for s in range(R):
                if s == r:
                    continue
                send, _, soff, _ = bufs[s]
                n = roff[s + 1] - roff[s]
                assert n == soff[r + 1] - soff[r]
                d2d(recv + 8 * roff[s], send + 8 * soff[r], 8 * n)
        for f in hs:
            f.halo_unpack(rnd)

    cfls = []
    for dt in dts:
        exchange(1)
        for f in hs:
            f.step_local(dt, 1)
        exchange(2)
        c = max(f.step_local(dt, 2) for f in hs)
        if reflux:
            move([f.reflux_buffers() for f in hs])
            for f in hs:
                f.step_local(dt, 3)
        for f in hs:
            assert f.commit(c) == fc.FC_OK
        cfls.append(c)
    q = np.concatenate([f.get_q() for f in hs if f.count], axis=0)
    for f in hs:
        f.close()
    return q, np.array(cfls)


CASES = [c2(steps=30), c5(level=2, m=16, steps=30), c3(level=2, m=32, steps=30),
         c4_workload(base_level=2, m=8, steps=30)]


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("w", CASES, ids=lambda w: w.name)
def test_sharded_equals_single_rank_bitwise(w, R, skip):
    qo, co, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
    qr, cr = run_sharded(w, R, do, skip)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)
    for k in range(w.meqn):
        assert np.abs(qr[:, k] - qo[:, k]).max() <= 1e-12 * np.abs(qo[:, k]).max()


@pytest.mark.parametrize("R", [5, 8])
@pytest.mark.parametrize("w", [c1(), c5(level=2, m=16, steps=20),
                               c2(steps=20)], ids=lambda w: w.name)
def test_sharded_eight_ranks_bitwise(w, R):
    """8 shards (C1: 2 patches per rank, periodic wraps and corner-only peers) and an
    uneven 5-way cut, bitwise equal to one rank."""
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do)
    qr, cr = run_sharded(w, R, do, 1)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


# ---- peer-memory halo (halo_p2p): the fused gather reads other ranks' buffers directly -----------
def run_sharded_p2p(w, R, dts, skip=1):
    """R rank handles with halo_p2p = 1 wired to each other's state buffers (same device: the peer
    pointers are plain device pointers here, CUDA IPC mappings with NCCL); no halo pass at all."""
    hs = [fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0, 0, r, R, None,
                    halo_p2p=1) for r in range(R)]
    for f in hs:
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject, skip)
    bufs = [f.p2p_buffers() for f in hs]
    for r, f in enumerate(hs):
        for s in range(R):
            if s != r:
                f.p2p_set_peer(s, bufs[s][0], bufs[s][1])
        f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    cfls = []
    for dt in dts:
        for f in hs:
            f.step_local(dt, 1)
        c = max(f.step_local(dt, 2) for f in hs)
        for f in hs:
            assert f.commit(c) == fc.FC_OK
        cfls.append(c)
    assert len({f.p2p_buffers()[2] for f in hs}) == 1           # parities in lockstep
    q = np.concatenate([f.get_q() for f in hs if f.count], axis=0)
    for f in hs:
        f.close()
    return q, np.array(cfls)


@pytest.mark.parametrize("R", [2, 3, 4, 8])
@pytest.mark.parametrize("w", [c1(), c5(level=2, m=16, steps=30), c5(level=3, m=16, steps=10),
                               c5(level=4, m=16, steps=8)], ids=lambda w: w.name)
def test_peer_memory_halo_equals_single_rank_bitwise(w, R):
    """(C5 level 4 at 2 ranks: 512 patches per rank, so the quiescent filter runs with remote
    neighbours always active)"""
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do)
    qr, cr = run_sharded_p2p(w, R, do)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("w", [c5(level=3, m=16, steps=10), c3(level=2, m=32, steps=10)], ids=lambda w: w.name)
def test_peer_memory_halo_full_update_bitwise(w, R):
    """bench.py's multi-GPU mode: the full update (skip_quiescent = 0) with the peer-memory halo --
    the warp-sweep kernel gathers remote ring cells straight from the owners' buffers."""
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=0)
    qr, cr = run_sharded_p2p(w, R, do, skip=0)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


@pytest.mark.parametrize("R", [2, 3])
def test_empty_ranks_bitwise(R):
    """More ranks than patches (a one-patch periodic forest): the ranks past the patch count own
    empty Morton ranges and take part in every stage with nothing to do (Fig. 3's idle
    processors), for both halo transports."""
    w = c1(level=0, m=16, steps=10)
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do)
    qr, cr = run_sharded(w, R, do, 1)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)
    qp, cp = run_sharded_p2p(w, R, do)
    np.testing.assert_array_equal(qp, q1)
    np.testing.assert_array_equal(cp, c1_)


@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("w", [c2(steps=20), "amr_euler"], ids=lambda w: w if isinstance(w, str) else w.name)
def test_sharded_reflux_equals_single_rank_bitwise(w, R):
    """Reflux across rank cuts (fc_reflux_*): the fine-face records of other ranks' patches are
    requested once, packed after the update and moved between the ranks, then the correction is
    applied -- bitwise the one-rank result, which conserves sum q area exactly."""
    import dataclasses
    if w == "amr_euler":
        from test_gpu_subcycle import amr_euler
        w = amr_euler(steps=8)
    w = dataclasses.replace(w, reflux=1)
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do)
    qr, cr = run_sharded(w, R, do, 1, reflux=1)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


@pytest.mark.parametrize("w", [c2(steps=15), c5(level=2, m=16, steps=15)], ids=lambda w: w.name)
def test_sharded_custom_partition_bitwise(w):
    """fc_forest_desc.partition: uneven Morton cuts, one rank empty -- bitwise the one-rank run."""
    P = w.num_patches
    part = [0, P // 7, P // 7, P // 2 + 3, P]
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do)
    qr, cr = run_sharded(w, 4, do, 1, partition=part)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


def run_sharded_split(w, R, dts, skip):
    """The halo overlap's order (fc_step on NCCL handles): pack, interior update (phase 4) while
    the halo slots still hold the previous step's values, then the transport, unpack and the
    boundary update (phase 5).  An interior patch reading a halo slot would see stale data."""
    hs = []
    for r in range(R):
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0, 0, r, R, None)
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject, skip, 0)
        hs.append(f)
    for rnd in (1, 2):
        for r in range(R):
            for s in range(R):
                if s != r:
                    hs[s].halo_set_requests(rnd, r, hs[r].halo_requests(s, rnd))
    for f in hs:
        f.halo_finalize()
        f.set_q(np.ascontiguousarray(w.q0[f.first:f.first + f.count]))
    cfls = []
    for dt in dts:
        for f in hs:
            f.halo_pack(1)
        for f in hs:
            f.step_local(dt, 4)
        bufs = [f.halo_buffers(1) for f in hs]
        for r in range(R):
            _, recv, _, roff = bufs[r]
            for s in range(R):
                if s != r:
                    send, _, soff, _ = bufs[s]
                    d2d(recv + 8 * roff[s], send + 8 * soff[r], 8 * (roff[s + 1] - roff[s]))
        for f in hs:
            f.halo_unpack(1)
        c = max(f.step_local(dt, 5) for f in hs)
        for f in hs:
            assert f.commit(c) == fc.FC_OK
        cfls.append(c)
    q = np.concatenate([f.get_q() for f in hs if f.count], axis=0)
    for f in hs:
        f.close()
    return q, np.array(cfls)


@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("w", [c5(level=2, m=16, steps=20), c3(level=2, m=32, steps=20), c1(steps=20)],
                         ids=lambda w: w.name)
def test_split_update_halo_overlap_bitwise(w, R):
    """SURVEY §8(e) overlap: interior patches updated before the halo arrives, boundary patches
    after -- bitwise the one-rank run (full update: no filter)."""
    qo, co, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=0)
    qr, cr = run_sharded_split(w, R, do, 0)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)


@pytest.mark.parametrize("skip", [1, 0], ids=["quiescent_skip", "full_update"])
@pytest.mark.parametrize("R", [2, 3, 5])
@pytest.mark.parametrize("w", ["c2", "three_levels", "amr_euler_m16"])
def test_fused_amr_gather_on_shards_bitwise(w, R, skip):
    """The fused two-hop AMR gather on several ranks (verdict r1, What's missing #4): every remote
    cell a computed ghost reads -- the coarse patch's interior, the one-hop sources of its ring
    cells (copies, or the fine interiors of its averages, computed locally) -- arrives in a round-1
    halo slot, so one exchange round suffices; bitwise the one-rank run."""
    from test_gpu_subcycle import amr_euler, three_levels
    w = {"c2": lambda: c2(steps=12), "three_levels": lambda: three_levels(steps=6),
         "amr_euler_m16": lambda: amr_euler(steps=6, m=16)}[w]()
    f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0, 0, 0, R, None)
    assert f.stats()["uniform_fast_path"] == 2
    f.close()
    _, _, do = oracle.run(w)
    q1, c1_, _ = fc.run(w, dt_list=do, skip_quiescent=skip)
    qr, cr = run_sharded(w, R, do, skip)
    np.testing.assert_array_equal(qr, q1)
    np.testing.assert_array_equal(cr, c1_)
