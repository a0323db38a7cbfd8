#!/usr/bin/env python
"""Benchmark of the Born-series sweep (BASELINE.json metric: Gpts/s, grid-point sweeps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "c1"): 64 independent seeded media on the 511^2 interior
grid of a 512-cell box (h = 1/512), contrast 0.5, 8 ppw, pointwise map gamma(x) = iV/eta,
rtol 1e-6.  A STEP is one bp::run call over the whole batch limited to --sweeps sweeps
(max_iters), i.e. --sweeps Born sweeps of every member plus the run's setup (||f||, ||G f||)
and result gather.  Work counted = sweeps actually executed (sum of iters) x 511^2 points.

* value   -- device-resident: f, u and the media live in HBM before the timed region;
             K steps timed with CUDA events on the library stream, max over ranks.
* e2e     -- the same steps through the public C ABI with PINNED HOST buffers: every step
             uploads the media (bp_problem_set_medium) and the sources, runs, and reads u and
             the traces back; H2D/D2H inside the timed region.
* roofline -- the fused row kernel (96 algorithmic B/pt) timed per launch with
             CUDA events on the launching stream (a second timed pass of the same K steps with
             the graph replaced by individually event-bracketed launches), vs MEASURED_PEAKS.
* cpu_baseline -- the reference's own code (oracle/_ref) on the host cores, bounded sample.

N > 1 (torchrun): the config's 64 members are split over the ranks (8 per GPU at N = 8, config
1's wording; "scaling": "strong"), independent members with no collective on the data path
(SURVEY.md 8(e)); --weak gives every rank its own N = 1 batch (global members [64 r, 64 r + 64)).
torch.distributed only for the barrier and the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Born-series sweeps x grid points per sec (Gpts/s); achieved HBM GB/s vs peak"
WORKLOADS = {
    "c0": "c0: 1 x 127^2 Dirichlet Helmholtz CBS, contrast 0.3, 10 ppw, sponge N/8, rtol 1e-6",
    "c1": "c1: 64 x 511^2 Dirichlet Helmholtz CBS batch, contrast 0.5, 8 ppw, sponge N/8, rtol 1e-6",
    "c2": "c2: 1 x 4095^2 Dirichlet Helmholtz CBS, contrast 0.5, 6 ppw, 16 point sources, rtol 1e-6",
    "c3": "c3: 1 x 255^3 Dirichlet Helmholtz CBS (seven-point, 3-D extension), contrast 0.4, 8 ppw, rtol 1e-5",
    "c4": "c4: 32 x 1024^2 Neumann convection-diffusion-reaction (upwind, DCT-II), real fp64, "
          "scalar gamma 1, rtol 1e-8",
}
# c4 (real fp64): RC_A T,u in + u out = 24 B/pt; RC_B u,bx,by,sigma,f in + T out = 48 B/pt;
# CC_GREEN T in + T out = 16 B/pt
CDR_ROW_BYTES_PER_PT = 72
CDR_COL_BYTES_PER_PT = 16
CDR_SWEEP_BYTES_PER_PT = 88
UNIT = "Gpts/s"
ROW_BYTES_PER_PT = 96     # row kernel: T in, u in, k2 in, f in, u out, T out (16 B each)
COL_BYTES_PER_PT = 32     # column kernel: T in, T out
SWEEP_BYTES_PER_PT = 128


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[2]))
            except ValueError:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "power_w": float(np.median(pw)) if pw else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(k2, f, k0, eta, sweeps, threads):
    """The reference's own code (oracle/_ref: proj/src sources + FFTW shim + restated run) on
    the host: OpenMP over members like proj/src/bench.cpp:143, each member iterated `sweeps`
    times.  Returns (Gpts/s, seconds, kind, sample)."""
    from oracle import MAP_POINTWISE, Reference, ReferenceBatch, Oracle, OracleProblem
    nd = k2.shape[1]
    if Reference.available():
        batch = ReferenceBatch(k2, k0, eta)  # Problem construction outside the timed sample
        t0 = time.perf_counter()
        _, _, _, info = batch.run(f, map_kind=MAP_POINTWISE, rtol=1e-6, max_iters=sweeps,
                                  nthreads=threads)
        dt = time.perf_counter() - t0
        batch.close()
        done = sum(i for i, _ in info)
        kind = "reference"
    else:  # the plain-C port
        Oracle.set_threads(threads)
        t0 = time.perf_counter()
        done = 0
        for b in range(k2.shape[0]):
            done += OracleProblem(k2[b], k0[b], eta[b]).run(f[b], map_kind=MAP_POINTWISE,
                                                            max_iters=sweeps).iters
        dt = time.perf_counter() - t0
        kind = "port"
    sample = (f"{k2.shape[0]} members x {sweeps} sweeps of {nd}x{nd} (bp::run incl. its setup, "
              f"Problem construction excluded), OpenMP over members, {threads} threads; transforms "
              f"through the project FFTW-API shim (radix-4 Stockham, not FFTW: FFTW is absent)")
    return done * nd * nd / dt / 1e9, dt, kind, sample


def cpu_oracle_parallel(k2, f, k0, eta, sweeps, threads):
    """SURVEY.md 8(d) mode (ii), "oracle-parallel": the plain-C port on ONE member with OpenMP
    inside every transform / element-wise pass (the reference never threads its FFTW plans,
    transforms.cpp:39-65).  Returns (Gpts/s, seconds, sample)."""
    from oracle import MAP_POINTWISE, Oracle, OracleProblem
    nd = k2.shape[1]
    Oracle.set_threads(threads)
    t0 = time.perf_counter()
    done = OracleProblem(k2[0], k0[0], eta[0]).run(f[0], map_kind=MAP_POINTWISE, rtol=1e-30,
                                                   max_iters=sweeps).iters
    dt = time.perf_counter() - t0
    return done * nd * nd / dt / 1e9, dt, (f"1 member x {done} sweeps of {nd}x{nd}, plain-C port, "
                                           f"OpenMP over transform lines, {threads} threads")


def cpu_baseline_cdr(bx, by, sigma, s0, f, sweeps, threads):
    """c4 has no reference problem family: the plain-C port (oracle/bp_oracle.c) on the host,
    OpenMP inside each transform / stencil, members one after another."""
    from oracle import Oracle, OracleProblem
    Oracle.set_threads(threads)
    n = bx.shape[1]
    t0 = time.perf_counter()
    done = 0
    for b in range(bx.shape[0]):
        done += OracleProblem.cdr(bx[b], by[b], sigma[b], s0[b]).run(
            f[b] + 0j, rtol=1e-8, max_iters=sweeps).iters
    dt = time.perf_counter() - t0
    sample = (f"{bx.shape[0]} c4 member(s) x {sweeps} sweeps of {n}x{n} (full bp::run incl. setup), "
              f"plain-C port, OpenMP over grid lines, {threads} threads")
    return done * n * n / dt / 1e9, dt, "port", sample


def workload_config(name: str, map_name: str, total: int, nd: int, dim: int = 2) -> dict:
    """The bench line's `config`: the workload only, identical in both arms (the arm-specific
    execution details go to the line's `step` / `parallelism` keys)."""
    grid = (f"{nd}x{nd} Neumann cell-centred (h=1/{nd})" if name == "c4" else
            "x".join([str(nd)] * dim) + f" (n={nd + 1}, h=1/{nd + 1})")
    return {"workload": WORKLOADS[name] + f"; map {map_name}", "grid": grid, "global_batch": total,
            "l2": "no flush needed: the per-step working set (>1 GB) >> 126 MB L2"}


def run_reference_arm(args):
    """The reference's own CPU path on the host cores: oracle/_ref --
    proj/src compiled in place with the project's FFTW-API shim (FFTW is absent) and the
    Eigen-free restatement of run / apply_correction.  Inputs come from the reference's own
    RngState / samplers (oracle/instances.py); nothing of the product package is imported.
    The members' Problem objects are built once before timing; a step is one bp::run of every
    member limited to --ref-sweeps sweeps, OpenMP over members (proj/src/bench.cpp:143-151)."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    from oracle import MAP_POINTWISE, Oracle, OracleProblem, Reference, ReferenceBatch
    from oracle.instances import cdr_c4, helmholtz_c1
    cores = os.cpu_count() or 1
    if args.config == "c4":
        # c4 has no reference problem family: the plain-C port stands in
        m = min(8, 32)
        bx, by, sg, s0, f = cdr_c4(0, m)
        sweeps = max(1, args.ref_sweeps)
        Oracle.set_threads(cores)
        probs = [OracleProblem.cdr(bx[b], by[b], sg[b], s0[b]) for b in range(m)]

        def step():
            return sum(probs[b].run(f[b] + 0j, rtol=1e-8, max_iters=sweeps).iters for b in range(m))
        n, kind = 1024, "port"
        sample = (f"{m} of the 32 c4 members x {sweeps} sweeps of 1024x1024 per step, plain-C port "
                  f"(oracle/bp_oracle.c; the reference has no CDR problem family), OpenMP over grid "
                  f"lines, {cores} threads")
        cfg = workload_config("c4", "scalar", 32, 1024)
    else:
        if not Reference.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbpref.so not built"}))
            return 0
        members = 64
        k2, f, k0, eta = helmholtz_c1(0, members)
        batch = ReferenceBatch(k2, k0, eta)  # Problem construction: outside the timed region
        sweeps = max(1, args.ref_sweeps)

        def step():
            _, _, _, info = batch.run(f, map_kind=MAP_POINTWISE, rtol=1e-6, max_iters=sweeps,
                                      nthreads=cores)
            return sum(i for i, _ in info)
        n, kind = 511, "reference"
        sample = (f"all 64 c1 members x {sweeps} sweeps of 511x511 per step (bp::run per member: "
                  f"its setup ||f||, ||G f|| included, Problem construction excluded), OpenMP over "
                  f"members, {cores} threads; transforms through the project FFTW-API shim "
                  f"(radix-4 Stockham, not FFTW: FFTW is absent)")
        cfg = workload_config("c1", "pointwise", 64, 511)
    for _ in range(args.warmup):
        step()
    done, times = 0, []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        done += step()
        times.append(time.perf_counter() - t0)
    value = float(done * n * n / np.sum(times) / 1e9)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded RngState media from the reference's own samplers, BASELINE construction)",
        "impl": "reference", "config": cfg,
        "step": {"sweeps_per_member": sweeps, "member_sweeps": done // max(1, args.steps)},
        "parallelism": f"host CPU, {cores} threads",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def load_traffic(config):
    """dram bytes per launch of the config's dominant (row) kernel from the committed ncu
    summary (profiles/ncu_summary.json, tools/make_profile_summary.py), if captured."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)[config]
        t = d["row"]["dram_bytes_per_launch"] + (d["row_b"]["dram_bytes_per_launch"] if "row_b" in d else 0.0)
        return t, f"{os.path.relpath(path, ROOT)} ({d['source']})"
    except Exception:
        return None, None


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_18527_b200 as bs

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1 or (args.slab and args.config in ("c2", "c3")):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    if args.config in ("c2", "c3") and (world > 1 or args.slab):
        rc = run_slab_bench(args, bs, rank, local_rank, world, barrier, max_over_ranks)
        dist.destroy_process_group()
        return rc

    from paper_2603_18527_b200.sharding import shard_members
    cfgd = bs.CONFIGS[args.config]
    total = args.batch if args.config == "c1" else cfgd["batch"]
    if args.strong:  # the config's member count split over the ranks
        first, per = shard_members(total, world, rank)
    else:  # weak scaling (batch of independent members, no collective): the N = 1 batch per rank
        first, per = rank * total, total
    cdr = args.config == "c4"
    if cdr:
        bx, by, sg, s0, f = bs.config_instances("c4", first, per)
        nd = bx.shape[1]
        row_b, col_b, sweep_b = CDR_ROW_BYTES_PER_PT, CDR_COL_BYTES_PER_PT, CDR_SWEEP_BYTES_PER_PT
    else:
        k2, f, k0, eta = bs.config_instances(args.config, first, per)
        nd = k2.shape[1]
        row_b, col_b, sweep_b = ROW_BYTES_PER_PT, COL_BYTES_PER_PT, SWEEP_BYTES_PER_PT
    dim = 3 if args.config == "c3" else 2
    if dim == 3:  # column stage = y-lines, x-lines, y-lines (32 B/pt each): 192 B/pt per sweep
        col_b, sweep_b = 3 * COL_BYTES_PER_PT, 192
    pts = nd ** dim
    cmap = {"pointwise": bs.PointwiseMap(), "scalar": bs.ScalarMap(1.0),
            "optimal_l2": bs.OptimalScalarMap("euclidean")}[args.map or cfgd["map"]]
    cfg = bs.IterationConfig(rtol=cfgd.get("rtol", 1e-6), max_iters=args.sweeps)

    if cdr:
        prob = bs.CdrNeumann(bx, by, sg, s0, device=local_rank)
    else:
        prob = bs.HelmholtzDirichlet(k2, k0, eta, device=local_rank, dim=dim)
    stream = torch.cuda.ExternalStream(prob.stream, device=local_rank)
    f_dev = torch.from_numpy(f).to(f"cuda:{local_rank}")
    u_dev = torch.empty_like(f_dev)
    import ctypes as C
    from paper_2603_18527_b200 import _native as N
    lib = N.lib()
    stride = cfg.max_iters + 1
    l2 = np.empty((per, stride))
    rt = np.empty((per, stride))
    info = (N.Trace * per)()
    mp, cc = cmap._c(), cfg._c()
    dp = C.POINTER(C.c_double)

    def step_device():
        rc = lib.bp_run_device(prob.handle, C.byref(mp), C.c_void_p(f_dev.data_ptr()), C.byref(cc),
                               None, C.c_void_p(u_dev.data_ptr()), l2.ctypes.data_as(dp),
                               rt.ctypes.data_as(dp), info)
        if rc:
            raise RuntimeError(N.last_error())
        return prob.last_run_stats()

    # Phase 1 -- the headline value: the production path (CUDA-graph replay), K steps.
    prob.set_kernel_timing(False)
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sweeps_done = 0
    launches = 0
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            st = step_device()
            sweeps_done += st["active_sweeps"]
            launches += st["kernel_launches"]
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        barrier()
        elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
        # Phase 2 -- per-kernel durations: the same steps launched without the graph, with
        # CUDA events around every launch on the library stream (bp_set_kernel_timing).
        prob.set_kernel_timing(True)
        step_device()
        row_ms = col_ms = 0.0
        timed = 0
        k0ev = torch.cuda.Event(enable_timing=True)
        k1ev = torch.cuda.Event(enable_timing=True)
        k0ev.record(stream)
        inst_sweeps = 0
        for _ in range(args.steps):
            st = step_device()
            row_ms += st["row_ms"]
            col_ms += st["col_ms"]
            timed += st["timed_sweeps"]
            inst_sweeps += st["active_sweeps"]
        k1ev.record(stream)
        k1ev.synchronize()
        inst_ms = max_over_ranks(k0ev.elapsed_time(k1ev))
        prob.set_kernel_timing(False)
    work = sum_over_ranks(float(sweeps_done * pts))
    value = work / (elapsed_ms * 1e-3) / 1e9
    value_instrumented = sum_over_ranks(float(inst_sweeps * pts)) / (inst_ms * 1e-3) / 1e9
    # per-launch kernel durations, normalised to a launch over the whole (active) batch: the
    # event time of every launch (including the early-exit launches after members converged)
    # divided by the member-sweeps done, times the members per launch
    full_launches = max(inst_sweeps, 1) / per
    row_avg = row_ms / full_launches
    col_avg = col_ms / full_launches
    pts_per_launch = per * pts
    peak, peak_src = measured_peak()
    row_gbs = row_b * pts_per_launch / (row_avg * 1e-3) / 1e9 if row_avg > 0 else 0.0
    col_gbs = col_b * pts_per_launch / (col_avg * 1e-3) / 1e9 if col_avg > 0 else 0.0
    sweep_gbs = sweep_b * pts_per_launch / ((row_avg + col_avg) * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(args.config)

    # ------------------------------------------------------------------ e2e through host buffers
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64 if cdr else torch.complex128, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    fh = pinned(f)
    if cdr:
        medium = [pinned(a) for a in (bx, by, sg)] + [s0]
    else:
        medium = [pinned(k2), k0, eta]
    prob.set_kernel_timing(False)
    # The user-facing serving call: bs.Pipeline over two handles of the step's shape
    # (bp_pipeline_*): each step = set_medium + run (H2D of the media and sources from pinned
    # host memory, the sweeps, D2H of u and the traces) on the next slot, so one step's copies
    # run under the other slot's sweeps.  --e2e-depth 1 = plain set_medium + bp_run.
    # (c4's steps are copy-bound -- its members converge in ~25 sweeps -- and gain from a third
    # slot: 23.4 -> 28.9 Gpts/s, r02i; the Helmholtz configs do not: 32.5 at depth 2 and 3)
    depth = max(1, args.e2e_depth if args.e2e_depth else (3 if cdr else 2))
    if cdr:
        extra = [bs.CdrNeumann(bx, by, sg, s0, device=local_rank) for _ in range(depth - 1)]
    else:
        extra = [bs.HelmholtzDirichlet(k2, k0, eta, device=local_rank, dim=dim) for _ in range(depth - 1)]
    slots = [prob] + extra
    uh = [pinned(np.zeros_like(f)) for _ in slots]
    pipe = bs.Pipeline(slots)
    e2e_steps = [0]

    def submit_e2e():
        j = e2e_steps[0]
        e2e_steps[0] += 1
        pipe.submit(cmap, fh, cfg, medium=medium, u_out=uh[j % depth])

    def stats_sweeps(results):
        return sum(t.iters for r in results for t in r.traces)

    for _ in range(max(1, args.warmup) * depth):
        submit_e2e()
    pipe.wait()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        submit_e2e()
    results = pipe.wait()
    e1.record(stream)
    e1.synchronize()
    barrier()
    # member-sweeps actually done (a member's trace holds iters sweeps; the device-resident
    # value counts the same quantity through last_run_stats)
    e2e_sweeps = stats_sweeps(results)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = sum_over_ranks(float(e2e_sweeps * pts)) / (e2e_ms * 1e-3) / 1e9
    pipe.close()
    for p_ in extra:
        p_.close()
    h2d = int(sum(a.nbytes for a in medium) + fh.nbytes) * world
    d2h = int(uh[0].nbytes + l2.nbytes + rt.nbytes + per * C.sizeof(N.Trace)) * world

    # ------------------------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        if cdr:
            m = min(8, per)
            v, dt, kind, sample = cpu_baseline_cdr(bx[:m], by[:m], sg[:m], s0[:m], f[:m],
                                                   args.cpu_sweeps_c4, cores)
        elif dim == 3:
            v = None  # the reference has no 3-D family
        else:
            m = min(cores, per)
            sw = args.cpu_sweeps if args.config != "c2" else max(2, args.cpu_sweeps // 50)
            v, dt, kind, sample = cpu_baseline(k2[:m], f[:m], k0[:m], eta[:m], sw, cores)
        cpu = None if v is None else {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                      "sample": sample, "seconds": round(dt, 3)}
        if cpu is not None and not cdr and dim == 2 and args.config != "c2":
            # mode (ii) next to the reference-faithful mode (i) above
            v2, dt2, sample2 = cpu_oracle_parallel(k2, f, k0, eta, 60, cores)
            cpu["oracle_parallel"] = {"value": v2, "unit": UNIT, "cores": cores, "kind": "port",
                                      "sample": sample2, "seconds": round(dt2, 3)}

    prob.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (seeded c4 media: smoothed noise b, sigma, f)" if cdr else
                     "synthetic (seeded RngState media + centre Gaussian-bump sources, BASELINE c1 construction)"),
            "config": workload_config(args.config, args.map or cfgd["map"],
                                      total if args.strong else total * world, nd, dim),
            "step": {"sweeps_per_member": args.sweeps, "members_per_gpu": per},
            "parallelism": (f"batch-shard x{world} (the {total} members split, members [{first}, "
                            f"{first + per}) on rank {rank})" if args.strong else
                            f"batch-shard x{world} ({per} independent members per GPU, "
                            f"global members [{first}, {first + per}) on rank {rank})"),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": (f"bs.Pipeline depth {depth} (bp_pipeline_*: set_medium + bp_run per step, "
                             "pinned host buffers, copies overlapped with the other slot's sweeps)"
                             if depth > 1 else "bp_problem_set_medium + bp_run with pinned host buffers")},
            "roofline": {"bound": "hbm",
                         "kernel": (f"crow_kernel<{int(np.log2(nd))},RC_A> + crow_kernel<{int(np.log2(nd))},RC_B>"
                                    if cdr else f"row_kernel<{int(np.log2(nd + 1))},R_SWEEP" +
                                    (",DIM=3>" if dim == 3 else ">")),
                         "note": ("achieved / frac: this kernel launched over the WHOLE batch, timed launch by "
                                  "launch with CUDA events in the instrumented pass; the timed region itself "
                                  "replays graphs (c1: waves of 8 single-member graphs on 8 streams, launches "
                                  "overlapping) -- its whole-sweep figure is sweep.timed_region"),
                         "achieved": row_gbs, "peak": peak, "unit": "GB/s", "frac": row_gbs / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": row_b * pts_per_launch,
                         "avg_launch_ms": row_avg,
                         "column_kernel": {"achieved": col_gbs, "frac": col_gbs / peak,
                                           "avg_launch_ms": col_avg,
                                           "algorithmic_bytes_per_launch": col_b * pts_per_launch},
                         "sweep": {"achieved": sweep_gbs, "frac": sweep_gbs / peak,
                                   "bytes_per_pt": sweep_b,
                                   "gpts_per_s_kernels_only": pts_per_launch / ((row_avg + col_avg) * 1e-3) / 1e9,
                                   # whole-sweep algorithmic bytes over the TIMED REGION itself (the
                                   # production path: graph replays, on c1 waves of 8 concurrently
                                   # replayed single-member graphs whose launches overlap -- the
                                   # per-kernel figures above are of whole-batch launches timed one
                                   # by one in the instrumented pass)
                                   "timed_region": {"achieved": value * sweep_b / world,
                                                    "frac": value * sweep_b / world / peak}}},
            "cpu_baseline": cpu,
            "gpu_launches": int(sum_over_ranks(float(launches))),
            "value_instrumented": value_instrumented,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_slab_bench(args, bs, rank, local_rank, world, barrier, max_over_ranks):
    """c2 / c3 on N GPUs: ONE 4095^2 (255^3) grid slab-decomposed over the ranks (SURVEY.md
    8(e)): per sweep a halo exchange (rows / x-planes), an all-reduce of 2 doubles and two
    all-to-alls of the transform intermediate (NCCL through torch.distributed; 3-D: over
    y-blocks, the z- and y-lines stay local).  Total work fixed ("scaling": "strong")."""
    import torch

    from paper_2603_18527_b200.slab import DistComm, SlabPart, run_slab
    cname = args.config
    k2, f, k0, eta = bs.config_instances(cname, 0, 1)
    nd = k2.shape[1]
    dim = k2.ndim - 1
    part = SlabPart(k2[0], float(k0[0]), float(eta[0]), rank, world, device=local_rank)
    comm = DistComm(fused=args.fused)
    cmap = bs.PointwiseMap()
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=args.sweeps)
    stream = torch.cuda.current_stream(local_rank)
    for _ in range(args.warmup):
        run_slab([part], comm, cmap, f[0], cfg)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    def timed(resident: bool):
        sweeps = 0
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            # value: f resident in HBM (staged by the warm-up), no result download;
            # e2e: host fields staged and the result + traces fetched inside every step
            sweeps += run_slab([part], comm, cmap, f[0], cfg, stage_fields=not resident,
                               fetch=not resident).sweeps_launched
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        barrier()
        return sweeps, max_over_ranks(ev0.elapsed_time(ev1))

    with ClockSampler(local_rank) as clocks:
        sweeps, elapsed_ms = timed(True)
    sweeps_e2e, elapsed_e2e = timed(False)
    pts = nd ** dim
    bpp = SWEEP_BYTES_PER_PT if dim == 2 else 192  # 128 (2-D), 192 (3-D)
    value = sweeps * pts / (elapsed_ms * 1e-3) / 1e9
    value_e2e = sweeps_e2e * pts / (elapsed_e2e * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    per_rank_gbs = bpp * pts / world * sweeps / (elapsed_ms * 1e-3) / 1e9
    # NVLink traffic per rank and sweep: the two transposes move the rank's
    # (P-1)/P off-rank share of its n^dim/P points, 16 B each way, plus the u halo (one row /
    # x-plane from each neighbour); the 1-element fences / 2-double all-reduce are negligible
    halo_elems = nd ** (dim - 1)
    nbr = (1 if rank in (0, world - 1) else 2) if world > 1 else 0
    nvl_bytes = (2 * 16 * (pts / world) * (world - 1) / world + 16 * halo_elems * nbr) if world > 1 else 0.0
    nvl_gbs = nvl_bytes * sweeps / (elapsed_ms * 1e-3) / 1e9
    nvl_peak = 900.0  # NVLink 5, GB/s per direction per GPU (B200 HGX, NVSwitch)
    part.close()
    if rank == 0:
        fb = int(f[0].nbytes)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (seeded RngState medium, 16 seeded point sources, BASELINE c2 construction)"
                     if dim == 2 else "synthetic (seeded RngState 3-D medium, centre bump, BASELINE c3 construction)"),
            "config": {"workload": WORKLOADS[cname] + "; map pointwise; slab-decomposed",
                       "grid": "x".join([str(nd)] * dim) + f" (n={nd + 1})", "global_batch": 1,
                       ("rows_per_gpu" if dim == 2 else "x_planes_per_gpu"): (nd + 1) // world,
                       "sweeps_per_step": args.sweeps,
                       "graph": "sweep loop captured as a CUDA graph of 16 sweeps (kernels + NCCL collectives)",
                       "parallelism": (f"x-slab x{world}: halo p2p + all-reduce + exchange fused into the kernels' "
                                       "stores over symmetric (NVLink peer) memory + 2 fences per sweep" if args.fused else
                                       f"x-slab x{world}: halo p2p + all-reduce + 2 all-to-all per sweep (NCCL)"),
                       "l2": "no flush needed: >1 GB working set >> 126 MB L2"},
            "e2e": {"value": value_e2e, "unit": UNIT, "h2d_bytes_per_step": fb, "d2h_bytes_per_step": fb,
                    "path": "run_slab from host fields (set_fields + result inside every step)"},
            "roofline": {"bound": "hbm", "kernel": "whole sweep per rank (row + column + collectives)",
                         "achieved": per_rank_gbs, "peak": peak, "unit": "GB/s",
                         "frac": per_rank_gbs / peak, "traffic": None, "peak_source": peak_src,
                         "bytes_per_pt": bpp,
                         "nvlink": {"bytes_per_sweep_per_rank": nvl_bytes, "achieved": nvl_gbs,
                                    "peak": nvl_peak, "unit": "GB/s", "frac": nvl_gbs / nvl_peak,
                                    "peak_source": "nominal NVLink 5 per-direction bandwidth (900 GB/s); "
                                                   "0 at N=1 (no off-rank traffic)"}},
            "cpu_baseline": None,
            # per sweep and rank: row + column + finalize (3-D: + two y-line launches)
            "gpu_launches": int(sweeps * (3 if dim == 2 else 5) * world),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=15)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=64, help="members of config c1 (whole job; per GPU with --weak)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank runs the N=1 batch of independent members (default: "
                         "the config's members split over the ranks, BASELINE c1 'sharded 8 per GPU at 8 GPUs')")
    ap.add_argument("--config", choices=["c0", "c1", "c2", "c3", "c4"], default="c1",
                    help="workload; the headline metric is quoted on c1 (BASELINE.json configs[1])")
    ap.add_argument("--map", choices=["pointwise", "scalar", "optimal_l2"], default=None,
                    help="correction map (default: the config's canonical map)")
    ap.add_argument("--sweeps", type=int, default=127, help="sweeps per step (max_iters)")
    ap.add_argument("--cpu-sweeps", type=int, default=300)
    ap.add_argument("--cpu-sweeps-c4", type=int, default=30)
    # sweeps per reference-arm step: enough that the run's setup (||f||, ||G f||: two
    # transform pairs) does not dominate the CPU sample (~1.3 s per step on 16 cores)
    ap.add_argument("--ref-sweeps", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-depth", type=int, default=0,
                    help="handles in the e2e bs.Pipeline (1 = set_medium + bp_run, serial)")
    ap.add_argument("--slab", action="store_true", help="c2 / c3: slab-decomposed path even at N=1")
    ap.add_argument("--fused", action="store_true",
                    help="c2 / c3 slabs: exchange fused into the kernels' stores (symmetric memory)")
    args = ap.parse_args()
    args.strong = not args.weak
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
