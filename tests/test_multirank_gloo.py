"""The sharded (N > 1) path on the CPU: world-size-2 gloo process group.  Each rank builds its
host-only plan, the ranks exchange halo requests over torch.distributed (as libfc does over NCCL at
creation), each rank checks it owns what it is asked for, serves the requested cells from the
oracle's ghost-filled global state, and the requester verifies that every ghost record with a
remote source finds the oracle's value through its request list (rounds 1 and 2)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import torch
        import oracle
        from paper_1308_1472_b200 import fc
        from workloads.configs import c2, c5
        from workloads.cubed_sphere import c4_workload
        w = {"C2": c2, "C5": lambda: c5(level=2, m=8), "C4": lambda: c4_workload(base_level=2, m=8)}[name]()
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux,
                      device=-1, rank=rank, nranks=world)
        n = w.m + 4
        n2 = n * n
        rng = np.random.default_rng(1308147 + 5)
        q = rng.standard_normal(w.q0.shape)
        of = oracle.forest_for(w)
        qp = of.ghost_fill(of.pad(q))          # the global state after phases A, C, B, C
        flat = qp.reshape(w.num_patches, w.meqn, n2)
        # exchange requests (rounds 1 and 2) with the peer, serve them, get the values back
        got = {}
        for rnd in (1, 2):
            for peer in range(world):
                if peer == rank:
                    continue
                mine = f.halo_requests(peer, rnd)
                cnt = torch.tensor([len(mine)], dtype=torch.int64)
                other = torch.zeros(1, dtype=torch.int64)
                reqs = [dist.isend(cnt, peer), dist.irecv(other, peer)]
                for r in reqs:
                    r.wait()
                theirs = torch.zeros(int(other.item()), dtype=torch.int64)
                reqs = [dist.isend(torch.from_numpy(mine), peer) if len(mine) else None,
                        dist.irecv(theirs, peer) if len(theirs) else None]
                for r in reqs:
                    if r is not None:
                        r.wait()
                theirs = theirs.numpy()
                p0, p1 = f.first, f.first + f.count
                assert ((theirs // n2 >= p0) & (theirs // n2 < p1)).all(), "asked for a patch I do not own"
                serve = flat[theirs // n2, :, theirs % n2] if len(theirs) else np.zeros((0, w.meqn))
                back = torch.zeros((len(mine), w.meqn), dtype=torch.float64)
                reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(serve)), peer) if len(theirs) else None,
                        dist.irecv(back, peer) if len(mine) else None]
                for r in reqs:
                    if r is not None:
                        r.wait()
                for key, val in zip(mine, back.numpy()):
                    got[(rnd, int(key))] = val
        # every remote source of this rank's ghost records is served with the oracle's value
        tab = f.ghost_table()
        p0, p1 = f.first, f.first + f.count
        m = w.m
        used = 0
        for rec in tab.reshape(-1, 8):
            op, src = int(rec[0]), int(rec[1])
            if op not in (1, 2, 3) or p0 <= src < p1:
                continue
            cells = {1: [(rec[2], rec[3])],
                     2: [(rec[2] + a, rec[3] + b) for b in (0, 1) for a in (0, 1)],
                     3: [(rec[2], rec[3]), (rec[2] - 1, rec[3]), (rec[2] + 1, rec[3]),
                         (rec[2], rec[3] - 1), (rec[2], rec[3] + 1)]}[op]
            for (i, j) in cells:
                ring = not (1 <= i <= m and 1 <= j <= m)
                key = src * n2 + (j + 1) * n + (i + 1)
                val = got[(2 if ring else 1, key)]
                np.testing.assert_array_equal(val, flat[src, :, (j + 1) * n + (i + 1)])
                used += 1
        assert used > 0
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


@pytest.mark.parametrize("name", ["C2", "C5", "C4"])
def test_two_rank_halo_plan_over_gloo(name):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
