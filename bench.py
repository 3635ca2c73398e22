#!/usr/bin/env python
"""bench.py -- fp64 cell-updates/s of the ForestClaw hot path (ghost fill + wave-propagation
update + CFL reduction) on 1..8 B200s, plus roofline, end-to-end and oracle baselines.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl fc|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

One "step" = one fc_step: ghost fill (for N > 1 the remote ring cells are read inside the update
kernel from the owner GPU's memory over NVLink -- the peer-memory halo, `--halo nccl` for the NCCL
send/recv exchange instead), the full wave-propagation update of every local patch (skip_quiescent
= 0: every tile's Riemann solves, limiters and corrections), the global CFL max-allreduce and the
CFL read-back that drives the next dt (the Clawpack variable-dt rule of the workload).  The
workload is BASELINE.json configs[4] (C5: Euler shock-bubble on a 4-tree brick, level 8, m = 16,
262,144 patches, 67.1M cells) -- the config BASELINE's metric is quoted on at 1/2/4/8 GPUs --
Morton-sharded across ranks (strong scaling).  Its state (2 x 3.36 GB) is far larger than L2, so no
flush is needed between steps.

Extra keys: `value_quiescent_skip` (the library's exact, data-dependent shortcut for patches whose
window is one state), `variants_full_update` (SURVEY §8(d)'s T1-T4 on this GPU with their HBM
roofline fractions), `roofline_hbm` (the headline step against HBM).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec per step (ghost fill + update) at 1/2/4/8 B200; % HBM roofline"
UNIT = "cell-updates/s"
WORKLOADS = {
    "C5": ("C5: 2D Euler shock-bubble, Roe + Harten-Hyman, MC limiter, 4-tree brick [0,4]x[0,1] "
           "outflow, uniform level 8, m=16, mbc=2 (BASELINE.json configs[4])"),
    "C3": ("C3: shallow-water radial dam break, Roe, MC limiter, walls, uniform level 6, m=32 "
           "(BASELINE.json configs[2])"),
}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def make_workload(name: str):
    from workloads.configs import c3, c5
    if name == "C5":
        return c5(lazy=True)
    if name == "C3":
        return c3(lazy=True)
    raise SystemExit(f"unknown workload {name}")


def algorithmic_flops(name: str):
    """fp64 flops per cell-update of the method, counted on the oracle's own code
    (tools/count_flops.py -> profiles/algorithmic_flops.json)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "algorithmic_flops.json")))[name])
    except Exception:
        return None


def fp64_peak_tflops(pk) -> float:
    """B200 fp64 (non-tensor) peak from unit counts: 148 SMs x 64 FMA lanes x 2 flops x clock."""
    return 148 * 64 * 2 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12


def profile_summary(name: str):
    """Per-launch DRAM traffic of the update kernel from the committed ncu capture, if any."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "step_kernel_traffic.json")))[name]
    except Exception:
        return None


def bytes_per_cell_update(w) -> int:
    """Compulsory (algorithmic) HBM bytes per cell-update: q read + q written + aux read."""
    return 16 * w.meqn + 8 * w.maux


# ---------------------------------------------------------------------------------------------
class Clocks:
    """Clock / throttle sampling during the timed region (the B200_PROFILING.md clocks line:
    clocks.sm, clocks.max.sm, power.draw, clocks_event_reasons.{hw_slowdown, hw_thermal_slowdown,
    sw_thermal_slowdown, sw_power_cap}).  NVML is polled from a thread every `period` s: the timed
    region (~0.1-1 s) is shorter than nvidia-smi's own start-up, so `nvidia-smi -lms` saw nothing.
    Each rank samples its own GPU (found by UUID); rank 0 reports the samples of every rank."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int, period: float = 0.005):
        import threading
        import pynvml as nv
        import torch
        self.nv = nv
        nv.nvmlInit()
        self.h = None
        try:
            uid = str(torch.cuda.get_device_properties(device).uuid)
            self.h = nv.nvmlDeviceGetHandleByUUID(uid if uid.startswith("GPU-") else "GPU-" + uid)
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
        self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                     "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                     "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                     "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        self.period = period
        self.rows = []
        self.stop_ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
        except Exception:
            pw = None
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((sm, mx, pw, [k for k, b in self.bits.items() if rs & b]))

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def start(self):
        self.th.start()

    def stop(self):
        self.stop_ev.set()
        self.th.join(timeout=5)
        try:
            self._sample()           # at least one sample even for a very short region
        except Exception:
            pass
        return self.rows

    @staticmethod
    def summary(rows):
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [r[0] for r in rows]
        pw = [r[2] for r in rows if r[2] is not None]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows),
                "sm_mhz_min": min(sm), "reasons": sorted({x for r in rows for x in r[3]}),
                "samples": len(rows), "power_w_max": max(pw) if pw else None,
                "source": "NVML polled every 5 ms during the timed region (all ranks)"}


# ---------------------------------------------------------------------------------------------
def oracle_rate(w, seconds: float, sample_patches: int = 256, seed: int = 1308147):
    """The CPU oracle as it stands (oracle/*.c, gcc -O2, single thread) on a bounded sample of
    the same workload: repeated one-step updates of `sample_patches` patches from the IC (each
    patch's ghost ring built from its neighbours, then the update) until `seconds` elapsed."""
    import numpy as np
    import oracle
    f = oracle.forest_for(w)
    rng = np.random.default_rng(seed)
    ids = np.sort(rng.choice(w.num_patches, size=sample_patches, replace=False)).astype(np.int64)
    q = w.q0 if w.q0 is not None else None
    if q is None:   # the sampled patches' rings need their neighbours: materialise the IC once
        w.materialise()
        q = w.q0
    pr = oracle.problem_for(w)
    t0 = time.perf_counter()
    reps = 0
    while True:
        f.step_sample(pr, q, w.dt0, 1.0 / w.m, ids)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    cells = reps * len(ids) * w.m * w.m
    return cells / el, el, reps, len(ids)


def oracle_rate_openmp(seconds: float):
    """The oracle's whole-forest step (orc_step, its OpenMP loop over patches) on all host cores,
    on C5's physics and patch size at level 5 (4,096 patches, 1.05 M cells: the full C5 forest
    would take minutes per step): ghost fill + one update per repetition, until `seconds`."""
    import oracle
    from workloads.configs import c5
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    w = c5(level=5, m=16, steps=1)
    f = oracle.forest_for(w)
    pr = oracle.problem_for(w)
    qp = f.pad(w.q0)
    t0 = time.perf_counter()
    reps = 0
    while True:
        f.step(pr, qp, w.dt0, 1.0 / w.m, None, cores)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    cells = w.num_patches * w.m * w.m
    return {"value": cells * reps / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{reps} x whole-forest steps (ghost fill + update, OpenMP over patches) of C5 physics "
                      f"at level 5 ({w.num_patches} patches, {cells} cells), {el:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle timed on the host (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = make_workload(args.workload)
    import numpy as np
    import oracle
    w.materialise()
    f = oracle.forest_for(w)
    pr = oracle.problem_for(w)
    rng = np.random.default_rng(1308147)
    ids = np.sort(rng.choice(w.num_patches, size=args.ref_patches, replace=False)).astype(np.int64)
    for _ in range(args.warmup):
        f.step_sample(pr, w.q0, w.dt0, 1.0 / w.m, ids)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        f.step_sample(pr, w.q0, w.dt0, 1.0 / w.m, ids)
    el = time.perf_counter() - t0
    cells = len(ids) * w.m * w.m
    value = cells * args.steps / el
    sample = (f"{len(ids)} random patches of {w.name} ({cells} cells) per step: ghost ring from "
              f"neighbour interiors + one wave-propagation update, single thread, from the IC")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOADS[args.workload], "cells_per_step": cells},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def run_variants(args, fc, hbm_peak):
    """SURVEY §8(d)'s throughput variants on this GPU, full update (skip_quiescent = 0): T1 (C1
    physics, uniform L10, m = 8), T2 (C2 physics, L8/L9, m = 16), T3 (C3 physics, L8, m = 32),
    T4 (C4 physics, L7/L8 band, m = 16).  W warm-ups then K steps of each config's dt policy from
    its IC, CUDA events around the step loop (each step includes its CFL read-back); states >> L2.
    HBM fraction = compulsory bytes (16 meqn + 8 maux per cell-update) / measured copy peak."""
    import numpy as np
    import torch
    from workloads.configs import c1, c2, c3
    from workloads.cubed_sphere import c4_workload
    makers = {"T1": lambda: c1(level=10, m=8), "T2": lambda: c2(base_level=8, m=16),
              "T3": lambda: c3(level=8, m=32), "T4": lambda: c4_workload(base_level=7, m=16, steps=20)}
    stream = torch.cuda.current_stream()
    out = {}
    for name, mk in makers.items():
        t0 = time.perf_counter()
        w = mk()
        gen_s = time.perf_counter() - t0
        qd = torch.from_numpy(np.ascontiguousarray(w.q0)).cuda()
        f = fc.forest_for(w, torch.cuda.current_device(), skip_quiescent=0)
        f.set_stream(stream.cuda_stream)

        def run(n, dt):
            for _ in range(n):
                rc, cfl = f.step(dt, raise_on_reject=False)
                if rc == fc.FC_ECFL:
                    dt = dt * w.cfl_target / cfl
                    rc, cfl = f.step(dt)
                dt = w.next_dt(dt, cfl)
            return dt
        f.set_q(qd)
        dt = run(max(3, args.warmup), w.dt0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(args.variant_steps, dt)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.variant_steps
        # the same steps replayed as CUDA graphs (fc_run, fixed dt = the adaptive dt reached): no
        # host turnaround between steps; each step still reduces its CFL (read back per call)
        f.run(dt, 1)                                  # (graph capture outside the timed region)
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        rc_g, _ = f.run(dt, args.variant_steps, raise_on_reject=False)
        g1.record(stream)
        torch.cuda.synchronize()
        ms_g = g0.elapsed_time(g1) / args.variant_steps if rc_g == fc.FC_OK else None
        f.reset_stats()
        f.set_timing(True)
        run(3, dt)
        st = f.stats()
        f.set_timing(False)
        f.close()
        del qd
        rate = w.cells / (ms / 1e3)
        bpc = 16 * w.meqn + 8 * w.maux
        graph = None
        if ms_g:
            rg = w.cells / (ms_g / 1e3)
            graph = {"ms_per_step": ms_g, "value": rg, "hbm_roofline_frac": rg * bpc / (hbm_peak * 1e9),
                     "timing": "fc_run (CUDA graphs, fixed dt), CUDA events around one call of K steps, "
                               "including its state backup copy and the CFL read-back"}
        out[name] = {"workload": w.name, "patches": w.num_patches, "cells": w.cells,
                     "ms_per_step": ms, "value": rate, "unit": UNIT,
                     "bytes_per_cell_update": bpc, "hbm_roofline_frac": rate * bpc / (hbm_peak * 1e9),
                     "update_kernel_ms": st["ms_step"] / max(1, st["step_kernel_launches"]),
                     "ghost_ms": st["ms_ghost"] / max(1, st["steps"]),
                     "fused_path": st.get("uniform_fast_path"), "generate_s": gen_s,
                     "steps": args.variant_steps, "mode": "full update (skip_quiescent = 0)",
                     "graph": graph}
    out["O3"] = run_octree(args, hbm_peak)
    return out


def run_octree(args, hbm_peak):
    """The octree path (include/fc3.h; reading 26) on this GPU: a 2 x 1 x 1 periodic
    brick of octrees at uniform level 4, m = 16 (8192 patches, 33.6 M cells), a Gaussian bump,
    velocity (0.8, -0.45, 0.3), MC, fixed dt at Courant 0.9; K steps after W warm-ups, CUDA events
    around the step loop (each step reads its CFL back).  Bitwise the oracle (tests/test_gpu_octree.py)."""
    import numpy as np
    import torch
    from paper_1308_1472_b200 import fc3
    from workloads.octree import cell_centres, forest3
    t0 = time.perf_counter()
    f = forest3((2, 1, 1), 4)
    m = 16
    c = cell_centres(f, m)
    q0 = np.exp(-8.0 * ((c[:, 0] - 0.6) ** 2 + (c[:, 1] - 0.5) ** 2 + (c[:, 2] - 0.45) ** 2))
    gen_s = time.perf_counter() - t0
    g = fc3.Forest3(f, m, torch.cuda.current_device())
    vel = (0.8, -0.45, 0.3)
    dt = 0.9 / (m * 2 ** 4) / 0.8
    g.set_problem(vel)
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)
    g.set_q(np.ascontiguousarray(q0))
    for _ in range(max(3, args.warmup)):
        g.step(dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.variant_steps):
        g.step(dt)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.variant_steps
    g.close()
    cells = f.num_patches * m ** 3
    rate = cells / (ms / 1e3)
    return {"workload": "octree brick 2x1x1, uniform level 4, m = 16, scalar advection (Godunov split)",
            "patches": int(f.num_patches), "cells": int(cells), "ms_per_step": ms, "value": rate, "unit": UNIT,
            "bytes_per_cell_update": 16, "hbm_roofline_frac": rate * 16 / (hbm_peak * 1e9),
            "timing": "CUDA events on the library's stream around K fc3_step calls (each reads its CFL back)",
            "generate_s": gen_s, "steps": args.variant_steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="fc", choices=["fc", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-patches", type=int, default=256)
    ap.add_argument("--no-variants", dest="variants", action="store_false",
                    help="skip the T1-T4 throughput variants (extra keys)")
    ap.add_argument("--variant-steps", type=int, default=20)
    ap.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: peer-memory halo in the fused gather (default) or NCCL send/recv")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1308_1472_b200 import build as libbuild
    libbuild.build()
    from paper_1308_1472_b200 import fc

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = make_workload(args.workload)
    P = w.num_patches
    p0, p1 = (rank * P) // world, ((rank + 1) * P) // world
    nccl_id = None
    if world > 1:
        obj = [fc.fc_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # N > 1: peer-memory halo (the fused ring gather reads neighbours' cells from the owner GPU over
    # NVLink, CUDA IPC mapped at creation) unless --halo nccl; falls back to the NCCL halo exchange
    # if the IPC mapping is refused
    halo = "none"
    if world > 1:
        halo = args.halo
        f, why = None, ""
        try:
            f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0,
                          local, rank, world, nccl_id, halo_p2p=1 if halo == "p2p" else 0)
        except fc.FcError as e:
            if halo != "p2p":
                raise
            why = str(e)
        ok = torch.tensor([1 if f is not None else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)            # the decision is collective
        if int(ok.item()) == 0:
            print(f"[bench] rank {rank}: peer-memory halo unavailable ({why or 'on another rank'}); NCCL halo",
                  file=sys.stderr)
            if f is not None:
                f.close()
            halo = "nccl (p2p refused)"
            obj = [fc.fc_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0,
                          local, rank, world, obj[0], halo_p2p=0)
    else:
        f = fc.Forest(w.forest.levels, w.forest.tree_ids, w.forest.conn, w.m, w.meqn, w.maux, 1.0,
                      local, rank, world, nccl_id)
    assert (f.first, f.count) == (p0, p1 - p0)
    f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject)
    q0 = torch.from_numpy(w.q0_range(p0, p1)).pin_memory()
    qdev = q0.cuda()
    stream = torch.cuda.current_stream()
    f.set_stream(stream.cuda_stream)
    cells_total = w.cells
    local_cells = (p1 - p0) * w.m * w.m

    def steps(n, dt):
        cfls = []
        for _ in range(n):
            rc, cfl = f.step(dt, raise_on_reject=False)
            if rc == fc.FC_ECFL:             # Clawpack retake with the reduced dt
                dt = dt * w.cfl_target / cfl
                rc, cfl = f.step(dt)
            cfls.append(cfl)
            dt = w.next_dt(dt, cfl)
        return dt, cfls

    def set_mode(skip: int):
        f.set_problem(w.kind, w.params[0], w.params[1], w.limiter, w.method2, w.method3, w.cfl_reject, skip)

    def timed(skip: int, monitor: bool, instrument: bool):
        """W warm-up + K timed steps from the IC (device-resident inputs).  instrument: the
        library's own per-phase / per-kernel CUDA events on its stream (measured: they slow the C5
        default step by ~14 %, so the headline pass runs without them and an identical instrumented
        pass supplies the kernel durations)."""
        set_mode(skip)
        f.set_q(qdev)
        dt, _ = steps(args.warmup, w.dt0)
        f.reset_stats()
        f.set_timing(instrument)
        clocks = None
        if monitor:
            try:
                clocks = Clocks(local)
            except Exception as e:   # NVML unavailable: reported as no samples
                print(f"[bench] clock sampling unavailable: {e}", file=sys.stderr)
        barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        dt, cfls = steps(args.steps, dt)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        rows = clocks.stop() if clocks else []
        if world > 1 and monitor:
            allrows = [None] * world
            dist.all_gather_object(allrows, rows)
            rows = [r for rr in allrows for r in (rr or [])]
        clk = Clocks.summary(rows) if monitor else None
        ms = allmax(ev0.elapsed_time(ev1))
        st = f.stats()
        f.set_timing(False)
        return ms, st, clk, cfls

    # ---- device-resident timed runs.  Headline: the method's full update (every tile's Riemann
    # solves, limiters and corrections; skip_quiescent = 0).  Beside it, the exact quiescent
    # shortcut (data-dependent: it skips the arithmetic of patches whose window is one state).
    ms, _, clk, cfls = timed(0, True, False)
    value = cells_total * args.steps / (ms / 1000.0)
    ms_i, st, _, _ = timed(0, False, True)          # instrumented twin: kernel / phase durations
    ms_q, _, _, _ = timed(1, False, False)
    value_q = cells_total * args.steps / (ms_q / 1000.0)
    _, st_q, _, _ = timed(1, False, True)
    set_mode(0)

    pk, pk_src = peaks()
    bpc = bytes_per_cell_update(w)
    hbm_peak = float(pk["hbm_gbs"])
    flops = algorithmic_flops(args.workload)
    fp64_peak = fp64_peak_tflops(pk)
    prof = profile_summary(args.workload) or {}
    kernel = {"C5": "k_step<EulerRoe>", "C3": "k_step<SweRoe>"}[args.workload]
    # dominant kernel of the full step: the update kernel (ghost kernels fill the rings first),
    # its launch time from CUDA events around its launches on the library's stream
    step_ms = st["ms_step"] / max(1, st["step_kernel_launches"])
    ghost_ms = st["ms_ghost"] / max(1, st["steps"])
    step_share = step_ms / (ms_i / args.steps)
    ach_tf = local_cells * flops / (step_ms / 1000.0) / 1e12 if flops else None
    roofline = {"bound": "alu", "achieved": ach_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": (ach_tf / fp64_peak) if ach_tf else None,
                "traffic": prof.get("step_dram_bytes_per_launch"),
                "traffic_full_step": prof.get("full_step_dram_bytes"),
                "algorithmic_bytes_per_launch": local_cells * bpc,
                "kernel": kernel + " (full update; dominant kernel of the step)", "launch_ms": step_ms,
                "share_of_step": step_share,
                "algorithmic_flops_per_cell_update": flops,
                "peak_source": "derived (DESIGN.md §6): 148 SMs x 64 fp64 FMA lanes x 2 flops x sm_max_mhz "
                               f"({pk.get('sm_max_mhz', 1965.0)} MHz, {pk_src} MEASURED_PEAKS.json); the DFMA "
                               "microbenchmark measures 34.1 TF (profiles/r01/dfma_peak.json)",
                "flops_source": "profiles/algorithmic_flops.json (fp64 ops of the oracle's own code per "
                                "cell-update, tools/count_flops.py)",
                "traffic_source": prof.get("source"),
                "timing": "kernel duration from CUDA events on the library stream in an instrumented twin "
                          "of the timed region (same steps from the same state); the headline pass runs "
                          "without the library's events"}
    # the same full step against HBM: compulsory bytes per cell-update at the measured copy peak
    ach_gbs = local_cells * bpc / (ms / args.steps / 1000.0) / 1e9
    roofline_hbm = {"bound": "hbm", "achieved": ach_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach_gbs / hbm_peak, "frac_vs_nominal_8000": ach_gbs / 8000.0,
                    "what": "whole full step, compulsory bytes (q read + written once, 16 meqn B per "
                            "cell-update): fp64-bound for the Euler/SWE solvers (BASELINE.md §2)",
                    "algorithmic_bytes_per_cell_update": bpc,
                    "peak_source": f"{pk_src} MEASURED_PEAKS.json hbm_gbs (copy)"}
    # the data-dependent quiescent shortcut (exact, library default): per-kernel durations
    copy_ms = st_q["ms_copy"] / max(1, st_q["copy_launches"]) if st_q.get("copy_launches") else None
    quiescent = {"value": value_q, "unit": UNIT, "ms_per_step": ms_q / args.steps,
                 "what": "skip_quiescent = 1 (library default): patches whose staged window holds one "
                         "state skip the update arithmetic (bitwise exact: every jump is 0); their cells "
                         "are still read and written (k_copy_classify). DATA-DEPENDENT: it measures the "
                         "flow (C5: ~96 % of patches quiescent), not the method's arithmetic",
                 "copy_kernel_ms": copy_ms,
                 "copy_kernel_hbm_frac": (local_cells * bpc / (copy_ms / 1000.0) / 1e9 / hbm_peak) if copy_ms else None,
                 "update_phase_ms": st_q["ms_step"] / max(1, st_q["step_kernel_launches"])}
    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        qh = torch.empty_like(q0).pin_memory()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f.set_q(q0)                       # H2D from pinned host memory + scatter into q_old
        _, _ = steps(args.steps, w.dt0)
        f.get_q(qh)                       # gather + D2H into pinned host memory
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = allmax(e0.elapsed_time(e1))
        qbytes = q0.numel() * 8
        e2e = {"value": cells_total * args.steps / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": qbytes / args.steps, "d2h_bytes_per_step": (qbytes + 8 * args.steps) / args.steps,
               "ms_total": ems,
               "definition": "fc_set_q(pinned host) + K x fc_step (CFL to host each step) + fc_get_q(pinned host), per-rank bytes"}

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        w.q0 = q0.numpy()                 # the full IC is already on the host at N = 1
        rate, el, reps, ns = oracle_rate(w, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{reps} x one-step updates of {ns} random {w.name} patches ({ns * w.m * w.m} cells) "
                         f"from the IC, ring built from neighbours, {el:.1f} s single-threaded"}
        if args.workload == "C5":         # the oracle with OpenMP on all host cores too
            cpu["openmp"] = oracle_rate_openmp(max(1.0, args.cpu_seconds / 3))

    variants = run_variants(args, fc, hbm_peak) if (args.variants and world == 1) else None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS[args.workload], "patches": P, "cells": cells_total,
                           "mode": "full update of every patch (skip_quiescent = 0)",
                           "parallelism": f"morton-shard x{world}" + (f" (halo: {halo})" if world > 1 else ""),
                           "l2": "state 2 x %.2f GB >> 126 MB L2 (no flush needed)" % (P * w.meqn * (w.m + 4) ** 2 * 8 / 1e9),
                           "dt_policy": "Clawpack variable dt (0.9 / CFL)", "final_cfl": cfls[-1]},
                "roofline": roofline, "roofline_hbm": roofline_hbm,
                "value_quiescent_skip": quiescent,
                "variants_full_update": variants,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": st["kernel_launches"],
                "phase_ms_per_step": {"ghost": ghost_ms, "update": step_ms,
                                      "cfl_allreduce": st["ms_comm"] / max(1, st["steps"])},
                "clocks": clk}
        print(json.dumps(line), flush=True)
    f.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
