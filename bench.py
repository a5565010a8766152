#!/usr/bin/env python
"""Benchmark of the B200 force-evaluation hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): 32,000 particles on an
FCC lattice (20^3 cells, rho 0.8, jitter +-0.02, T*=0.9), LJ rc 2.5, ATM
nu=0.073 rc 2.5, fp64, r-RESPA with dt=0.001 and three-body factor 5.  A
"step" is one r-RESPA base step (drift, binning, survivor rows, LJ pass,
kick; the ATM pass on every 5th step) -- exactly integrators.py:148-172.

ours:       K steps replayed from CUDA graphs of one 5-step sampling period;
            inside the graph every step is preceded by an L2 flush (a 256 MiB
            write) and bracketed by external event-record nodes, so a step is
            timed on the device from its first to its last kernel; value =
            steps/s.  roofline = the ATM kernel (dominant) timed standalone
            with events, 141 FP64 flops per unique triplet
            against the FP64 FMA peak measured in this run (MEASURED_PEAKS.json
            has no FP64 figure).  e2e = the public respa_run() on host numpy
            arrays (median of three calls).
reference:  the reference's CPU path on this host's cores -- the C port of
            respamd's kernels in oracle/ (bit-exact with the reference,
            tests/test_oracle_golden.py) with all host threads, same workload.

For N > 1 (torchrun, one process per GPU) the box is cfg2's block replicated
along the rank grid (weak scaling) and run by the domain-decomposed loop
(NCCL halo exchange); each rank times its steps with events
around the steps of one trajectory, flushing L2 in between; the max over
ranks is reported.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ATM triplet interactions/s and r-RESPA MD steps/s (fp64) vs FP64 roofline"
WORKLOAD = ("cfg2: 32,000 particles, FCC 20^3 cells rho 0.8, jitter +-0.02 sigma, periodic box "
            "34.1995, T*=0.9; LJ eps=sigma=1 rc 2.5; ATM nu=0.073 rc 2.5; r-RESPA dt 0.001, "
            "three-body factor 5")
FLOPS_PER_TRIPLET = 141
FLOPS_PER_PAIR = 35


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", default="cfg2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--rc3", type=float, default=None,
                   help="three-body cutoff override (cfg3 sweep: 2.0 / 2.5 / 3.0)")
    p.add_argument("--sf", type=int, default=None,
                   help="three-body step-size factor override (cfg3 sweep: 1 / 5 / 10)")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)
        if not self.rows:  # timed region shorter than the sampler's start-up
            self.after = True
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=10).stdout
                self.rows = [[c.strip() for c in ln.split(",")] for ln in out.splitlines() if ln]
            except (OSError, subprocess.SubprocessError):
                pass

    after = False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows),
                **({"sampled": "right after the timed region (shorter than the sampler's "
                               "start-up)"} if self.after else {})}


# --------------------------------------------------------------------------
# CPU legs (the oracle port of the reference kernels)
# --------------------------------------------------------------------------
def workload_name(cfg) -> str:
    if cfg.name == "cfg2" and cfg.rc_atm == 2.5 and cfg.step_size_factor == 5:
        return WORKLOAD
    return (f"{cfg.name}: {cfg.description}; LJ rc {cfg.rc_lj}, ATM rc {cfg.rc_atm}, "
            f"three-body factor {cfg.step_size_factor} (sweep point, not the headline)")


def cpu_respa_rate(cfg, seconds: float, threads: int):
    """Steps/s of the reference loop restated in oracle/ on `threads` cores.

    Bounded sample: one calibration cycle, then a single respa_run of whole
    three-body cycles sized to take about `seconds` (its two initial passes
    are included in the timing, which slightly favours the GPU)."""
    from oracle import oracle as o

    o.set_num_threads(threads)
    s = cfg.system()
    sf = cfg.step_size_factor
    ff = o.OracleForceField(nu=0.073, cutoff=cfg.rc_lj)
    sysm = o.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    t0 = time.perf_counter()
    o.respa_run(sysm, ff, o.OracleLinkedCells(), cfg.dt, sf, sf)
    t_cycle = time.perf_counter() - t0
    steps = sf * int(min(20, max(1, round(seconds / max(t_cycle, 1e-3)))))
    sysm = o.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    t0 = time.perf_counter()
    o.respa_run(sysm, ff, o.OracleLinkedCells(), cfg.dt, sf, steps)
    elapsed = time.perf_counter() - t0
    return steps / elapsed, steps, elapsed


def reference_arm(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import oracle as o

    o.set_num_threads(threads)
    s = cfg.system()
    sysm = o.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    ff = o.OracleForceField(nu=0.073, cutoff=cfg.rc_lj)
    sf = cfg.step_size_factor
    warm = max(sf, (args.warmup + sf - 1) // sf * sf)
    steps = max(sf, (args.steps + sf - 1) // sf * sf)
    cont = o.OracleLinkedCells()
    o.respa_run(sysm, ff, cont, cfg.dt, sf, warm)
    t0 = time.perf_counter()
    o.respa_run(sysm, ff, cont, cfg.dt, sf, steps)
    elapsed = time.perf_counter() - t0
    rate = steps / elapsed
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d)",
        "config": {"workload": workload_name(cfg), "timed": "respa_run incl. its two initial passes"},
        "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} r-RESPA steps of {cfg.name} (oracle/ C port of respamd "
                                   f"kernels, OpenMP {threads} threads)"},
        "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def domain_arm(args, cfg):
    """N > 1: weak scaling with the domain-decomposed r-RESPA.

    The box is cfg2's FCC block replicated along the rank grid (32,000
    particles per GPU), decomposed over the ranks (NCCL halo exchange);
    value = ranks x steps/s (cfg2-equivalent steps per second), time = max
    over ranks of the CUDA-event time of steps W..W+K of one trajectory."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # one process per GPU over NCCL; RB_DIST_BACKEND=gloo (and
    # RB_SHARE_GPU=1: all ranks on cuda:0) exercises the same path on one GPU
    share = os.environ.get("RB_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dist.init_process_group(os.environ.get("RB_DIST_BACKEND", "nccl"))
    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200.domain import auto_dims
    from paper_2507_11172_b200.domain_run import domain_respa_run, gpu_backend_factory

    sf = cfg.step_size_factor
    dims = auto_dims(world, (world * 16, world * 16, world * 16))
    nc = tuple(cfg.params["nc"] * d for d in dims)
    s = pkg.systems.fcc_system(nc, jitter=0.02, seed=1, temperature=cfg.temperature, vseed=1)
    ff = cfg.force_field()
    K = max(sf, (int(args.steps) + sf - 1) // sf * sf)
    W = max(sf, (max(3, int(args.warmup)) + sf - 1) // sf * sf)
    L = pkg._lib.lib()
    backends = []

    def factory(dec, n_total, r_build):
        b = gpu_backend_factory(ff)(dec, n_total, r_build)
        backends.append(b)
        return b

    # one trajectory of W + K steps; each of the steps W..W+K-1 is bracketed
    # by CUDA events with an L2 flush (256 MiB write) in between, as on one
    # GPU; time = the sum of the step times (each rank's own clock, max over
    # ranks)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = pkg._lib.stream_handle()
    starts, ends, marks = [], [], {}

    def on_step(i):
        if i == W:
            torch.cuda.synchronize()
            dist.barrier()
            marks["l0"] = L.rb_launch_count()
        if W < i <= W + K:
            ends.append(torch.cuda.Event(enable_timing=True))
            ends[-1].record()
        if W <= i < W + K:
            L.rb_l2_flush(pkg._lib.ptr(flush), flush.numel(), stream)
            starts.append(torch.cuda.Event(enable_timing=True))
            starts[-1].record()
        if i == W + K:
            torch.cuda.synchronize()
            marks["l1"] = L.rb_launch_count() - K  # minus the flushes
            dist.barrier()

    run_sys = s.copy()
    with ClockSampler(local) as clocks:
        domain_respa_run(dist, run_sys, ff, pkg.RespaSchedule(cfg.dt, sf, W + K), factory,
                         dims=dims, on_step=on_step)
    step_ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    t = torch.tensor([step_ms, float(marks["l1"] - marks["l0"])], dtype=torch.float64,
                     device="cuda")
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms = float(mx[0].item())
    launches = int(sm[1].item())
    value = world * K / (ms * 1e-3)

    # e2e: the public decomposed run from host arrays (scatter, steps, gather)
    e2e_sys = s.copy()
    dist.barrier()
    t0 = time.perf_counter()
    domain_respa_run(dist, e2e_sys, ff, pkg.RespaSchedule(cfg.dt, sf, K),
                     gpu_backend_factory(ff), dims=dims)
    torch.cuda.synchronize()
    dist.barrier()
    e2e_s = time.perf_counter() - t0

    # dominant kernel: the ATM pass on this rank's local set (owned + ghosts)
    eng = backends[0].eng
    f3 = torch.empty((eng.pos.shape[0], 3), dtype=torch.float64, device="cuda")
    bk = backends[0]
    eng.reset_status(0)
    eng.atm(bk.window, bk.rc3, float(ff.nu), f3, tag=0, count_visits=True)
    torch.cuda.synchronize()
    unique = int(eng.visits.item())
    ts = []
    for _ in range(5):
        L.rb_l2_flush(pkg._lib.ptr(flush), flush.numel(), stream)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        eng.atm_kernel(bk.window, bk.rc3, float(ff.nu), f3, 0)
        eb.record()
        torch.cuda.synchronize()
        ts.append(ea.elapsed_time(eb))
    atm_ms = statistics.median(ts)
    peak = ctypes.c_double(0.0)
    L.rb_fp64_peak(2000, ctypes.byref(peak), stream)
    achieved = unique / (atm_ms * 1e-3) * FLOPS_PER_TRIPLET / 1e12
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d)",
            "config": {"workload": f"cfg2 block x {dims} = {s.n} particles, domain-decomposed",
                       "particles": s.n, "step_size_factor": sf,
                       "parallelism": f"domain decomposition {dims} "
                                      f"({dist.get_backend()} halo exchange)",
                       "value": "ranks x steps/s (cfg2-equivalent steps per second)",
                       "timed": "steps W..W+K of one decomposed trajectory, per-step CUDA "
                                "events summed, max over ranks",
                       "l2": "flushed (256 MiB write) between timed steps"},
            "roofline": {"bound": "fp64", "kernel": "ATM triplet pass on rank 0's local set",
                         "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": achieved / peak.value if peak.value else None, "traffic": None,
                         "work": f"{FLOPS_PER_TRIPLET} FP64 flops per unique triplet x {unique} "
                                 f"triplets (owned + ghost bases)",
                         "kernel_ms": atm_ms},
            "e2e": {"value": world * K / e2e_s, "unit": "steps/s",
                    "h2d_bytes_per_step": 2 * s.n * 24 / K,
                    "d2h_bytes_per_step": 4 * s.n * 24 / K,
                    "note": f"domain_respa_run({K} steps) from host arrays on every rank, wall "
                            f"clock incl. scatter, initial passes and the final gather"},
            "gpu_launches": launches,
            "gpu_launches_detail": {"note": "this library's launches during the timed steps, "
                                            "summed over ranks"},
            "clocks": clocks.summary(),
        }), flush=True)
    dist.destroy_process_group()


def ours_arm(args, cfg):
    import torch

    world, rank, local = dist_env()
    if world > 1:
        return domain_arm(args, cfg)
    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import _lib
    from paper_2507_11172_b200.integrators import DeviceRespa, RespaSchedule

    _lib.require_device()
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    sf = cfg.step_size_factor
    K, W = int(args.steps), max(3, int(args.warmup))

    s = cfg.system()
    ff = cfg.force_field()
    periods = (K + sf - 1) // sf  # whole sampling periods replayed; exactly K steps timed
    W = (W + sf - 1) // sf * sf
    total_steps = sf + W + periods * sf + 2 * sf
    run = DeviceRespa(s.copy(), ff, pkg.CudaLinkedCells(), RespaSchedule(cfg.dt, sf, total_steps),
                      sf)
    run.start()
    run.run_periods(0, 1)  # eager warm-up period: allocations, attributes
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # one CUDA graph per sampling period; inside it every step is bracketed by
    # event-record nodes and preceded by an L2 flush (outside the brackets),
    # so each step is timed on the device from its first to its last kernel
    ev = []
    for _ in range(2 * sf):
        e = ctypes.c_void_p()
        _lib.check(L.rb_event_create(ctypes.byref(e)), "rb_event_create")
        ev.append(e)

    def timed_period():
        st = _lib.stream_handle()
        for j in range(sf):
            L.rb_l2_flush(_lib.ptr(flush), flush.numel(), st)
            _lib.check(L.rb_event_record(ev[2 * j], st), "rb_event_record")
            run._step(j, j)
            _lib.check(L.rb_event_record(ev[2 * j + 1], st), "rb_event_record")

    l0 = L.rb_launch_count()
    graph = run._captured(timed_period)
    launches_per_period = L.rb_launch_count() - l0 - sf  # minus the flushes
    # kernels of the conditional rebuild body run only on rebuild steps
    body = run.eng.cond_body_launches
    launches_per_step = launches_per_period / sf - body
    for _ in range(W // sf):
        graph.replay()
    torch.cuda.synchronize()
    rebuilds0 = int(run.eng.status[3].item())
    ms = 0.0
    el = ctypes.c_float()
    with ClockSampler(local) as clocks:
        timed = 0
        for _ in range(periods):
            graph.replay()
            for j in range(sf):  # (synchronises on the period's last event)
                if timed == K:  # steps past K: replayed, not timed
                    break
                _lib.check(L.rb_event_elapsed(ev[2 * j], ev[2 * j + 1], ctypes.byref(el)),
                           "rb_event_elapsed")
                ms += el.value
                timed += 1
        torch.cuda.synchronize()
    rebuilds = int(run.eng.status[3].item()) - rebuilds0
    status = run.eng.read_status()
    if status is not None or run.eng.overflowed():
        raise RuntimeError(f"device error during the timed run: {status}")
    for e in ev:
        L.rb_event_destroy(e)
    ms_max = ms
    ms_per_step = ms_max / K
    value = world * K / (ms_max * 1e-3)
    stream = _lib.stream_handle()

    # ---- dominant kernel: the ATM pass, standalone, events on its stream
    eng, geom = run.eng, run._geom()
    eng.bin(geom, run.x)
    eng.nlist(geom, run.r_build, capacity=run.capacity, checked=True)
    eng.slots = run.slots
    f3 = torch.empty_like(run.f3)
    eng.reset_status(0)
    eng.atm(geom, run.rc3, run.nu, f3, tag=0, count_visits=True)
    torch.cuda.synchronize()
    unique = int(eng.visits.item())

    def atm_once():
        eng.atm_kernel(geom, run.rc3, run.nu, f3, tag=0)

    def atm_c01_once():
        eng.atm_c01(geom, run.rc3, run.nu, f3, tag=0, reduce=False)

    def lj_once():
        eng.lj_kernel(geom, run.rc2, 1.0, 1.0, f3, tag=0)

    def time_kernel(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            L.rb_l2_flush(_lib.ptr(flush), flush.numel(), stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts), ts

    atm_ms, _ = time_kernel(atm_once, 20)
    c01_ms, _ = time_kernel(atm_c01_once, 10)
    lj_ms, _ = time_kernel(lj_once, 20)
    pairs = int((eng.row_count[: eng.n].sum().item()))  # row entries (rc + skin)
    tflop = torch.empty(1, dtype=torch.float64)
    peak = ctypes.c_double(0.0)
    L.rb_fp64_peak(2000, ctypes.byref(peak), stream)
    peak_tf = float(peak.value)
    triplets_per_s = unique / (atm_ms * 1e-3)
    achieved_tf = triplets_per_s * FLOPS_PER_TRIPLET / 1e12
    traffic = None
    prof = os.path.join(REPO, "profiles", "atm_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    del tflop

    # ---- e2e through the public API on host arrays
    e2e_steps = (K + sf - 1) // sf * sf
    # warm-up call (module loading, allocator, graph instantiation paths),
    # then the median of three timed calls
    pkg.respa_run(cfg.system(), ff, pkg.CudaLinkedCells(),
                  pkg.RespaSchedule(cfg.dt, sf, max(W, 3) * sf))
    e2e_runs = []
    for _ in range(3):
        host = cfg.system()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pkg.respa_run(host, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(cfg.dt, sf, e2e_steps))
        torch.cuda.synchronize()
        e2e_runs.append(time.perf_counter() - t0)
        if os.environ.get("RB_E2E_DEBUG"):
            from paper_2507_11172_b200 import integrators as _it
            marks = _it.LAST_RUN[0].marks
            print("e2e call", " ".join(f"{lab}:{1e3 * (t - t0):.1f}" for lab, t in marks),
                  file=sys.stderr)
    e2e_s = statistics.median(e2e_runs)
    n = s.positions.shape[0]
    h2d = 2 * n * 24  # positions + velocities
    d2h = 4 * n * 24 + (e2e_steps // sf + 1) * 64  # x, v, f2, f3 + trace rows

    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d; no public dataset)",
        "config": {"workload": workload_name(cfg), "particles": n, "step_size_factor": sf,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "graph": "one CUDA graph per 5-step sampling period; each step bracketed "
                            "by external event-record nodes (flush outside the brackets)"},
        "roofline": {"bound": "fp64", "kernel": "ATM triplet pass (k_atm3 + k_atm3_gather)",
                     "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf if peak_tf > 0 else None,
                     "traffic": traffic,
                     "peak_source": "measured in this run: rb_fp64_peak DFMA chains on all SMs "
                                    "(MEASURED_PEAKS.json has no FP64 entry)",
                     "work": f"{FLOPS_PER_TRIPLET} FP64 flops per unique triplet x {unique} "
                             f"unique triplets per launch",
                     "kernel_ms": atm_ms, "triplets_per_s": triplets_per_s,
                     "c01_kernel_ms": c01_ms,
                     "c01_triplets_per_s": unique / (c01_ms * 1e-3),
                     "lj_kernel_ms": lj_ms, "lj_row_entries": pairs,
                     "skin": run.skin},
        "e2e": {"value": e2e_steps / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps,
                "note": f"public respa_run({e2e_steps} steps) on host numpy arrays, wall clock "
                        f"incl. upload, graph capture, download; median of 3 calls "
                        f"({', '.join(f'{1e3 * t:.1f}' for t in e2e_runs)} ms)"},
        "gpu_launches": int(round(launches_per_step * K)) + rebuilds * body + K,
        "gpu_launches_detail": {"per_step": launches_per_step, "l2_flush_per_step": 1,
                                "timing": "per-step external event-record nodes inside the "
                                          "period graph",
                                "rebuild_steps": rebuilds, "per_rebuild": body},
        "clocks": clocks.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, done, el = cpu_respa_rate(cfg, args.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": rate, "unit": "steps/s", "cores": threads, "kind": "port",
                                "sample": f"{done} r-RESPA steps of {cfg.name} in {el:.1f}s (oracle/ C "
                                          f"port of respamd kernels, OpenMP {threads} threads)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse_args()
    from paper_2507_11172_b200 import systems

    cfg = systems.CONFIGS[args.config]
    if args.rc3 is not None or args.sf is not None:  # sweep points of a config (not the headline)
        import dataclasses

        cfg = dataclasses.replace(cfg, rc_atm=cfg.rc_atm if args.rc3 is None else args.rc3,
                                  step_size_factor=cfg.step_size_factor if args.sf is None
                                  else args.sf)
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        ours_arm(args, cfg)


if __name__ == "__main__":
    main()
