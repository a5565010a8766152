#!/usr/bin/env python
"""Benchmark of the B200 force-evaluation hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg4] [--no-cpu-baseline] [--no-secondary]

Workload (BASELINE.json configs[3]): cfg4, 2,048,000
particles on an FCC lattice (80^3 cells, rho 0.8, jitter +-0.02, T*=0.9), LJ
rc 2.5, ATM nu=0.073 rc 2.5, fp64, r-RESPA dt=0.001 with three-body factor
5 -- the configuration BASELINE.json's scaling target is quoted on, run at
every N (strong scaling: the same box on 1, 2, 4, 8 GPUs).  A "step" is
one r-RESPA base step (drift, gated rebuild, LJ pass, kick; the ATM pass on
every 5th step) -- exactly integrators.py:148-172.

ours (N = 1): K steps replayed from CUDA graphs of one 5-step sampling
            period; inside the graph every step is preceded by an L2 flush
            (a 256 MiB write; cfg4's rows alone are 1.3 GB, far above L2)
            and bracketed by external event-record nodes, so a step is timed
            on the device from its first to its last kernel; value =
            steps/s.  roofline = the ATM pass (dominant) timed standalone
            with events, 141 FP64 flops per unique triplet
            against the FP64 FMA peak measured in this run (MEASURED_PEAKS
            has no FP64 figure); "hbm" = binning and the fused kick+drift
            timed standalone, algorithmic bytes against the
            measured copy peak.  e2e = the public respa_run() on host numpy
            arrays (median of three calls).  "secondary" = cfg2 (32,000
            particles, BASELINE configs[1]): the same device-timed loop, a
            100-step trajectory timed whole (rebuild steps included) and the
            e2e of a 20-step call.
ours (N > 1, torchrun): the same cfg4 box, domain-decomposed over the ranks
            (NCCL); each rank times steps W..W+K of one
            trajectory with events; max over ranks; value = K / that time.
reference:  the reference's CPU path on this host's cores -- the C port of
            respamd's kernels in oracle/ (bit-exact with the reference,
            tests/test_oracle_golden.py; faster than the stock numba package,
            BASELINE.md) with all host threads, same workload, a bounded
            number of timed steps.
cpu_baseline (ours, rank 0, N = 1): per-pass medians of the port (pair
            pass, triplet pass) at all cores and at 1 thread (a base-cell
            subset, scaled), extrapolated to steps/s, CPU model stated.
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
WORKLOADS = {
    "cfg4": ("cfg4: 2,048,000 particles, FCC 80^3 cells rho 0.8, jitter +-0.02 sigma, periodic "
             "box 136.798, T*=0.9; LJ eps=sigma=1 rc 2.5; ATM nu=0.073 rc 2.5; r-RESPA dt 0.001, "
             "three-body factor 5"),
    "cfg2": ("cfg2: 32,000 particles, FCC 20^3 cells rho 0.8, jitter +-0.02 sigma, periodic box "
             "34.1995, T*=0.9; LJ eps=sigma=1 rc 2.5; ATM nu=0.073 rc 2.5; r-RESPA dt 0.001, "
             "three-body factor 5"),
}
HBM_PEAK_GBS = 6551.7  # MEASURED_PEAKS.json (copy, read + write)
BIN_BYTES_PER_PARTICLE, BIN_BYTES_PER_CELL = 28, 4
STEP_BYTES_PER_PARTICLE = 192  # drift + kick, SURVEY.md §8d
FLOPS_PER_TRIPLET = 141
FLOPS_PER_PAIR = 35


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", default="cfg4")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the cfg2 secondary block")
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
    if cfg.name in WORKLOADS and cfg.rc_atm == 2.5 and cfg.step_size_factor == 5:
        return WORKLOADS[cfg.name]
    return (f"{cfg.name}: {cfg.description}; LJ rc {cfg.rc_lj}, ATM rc {cfg.rc_atm}, "
            f"three-body factor {cfg.step_size_factor} (sweep point, not the headline)")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_pass_medians(cfg, threads: int, reps: int = 3, stride: int = 1):
    """Median seconds of the reference's two passes as the port runs them
    (binning + C01 pass each, as LinkedCells.pair_pass / triplet_pass rebin
    on every call, containers.py:921,933) on cfg's step-0 system, and of one
    r-RESPA integration update (numpy, as integrators.py:150-165).
    stride > 1: only every stride-th base cell (base_cells), the time scaled
    back by (cells / timed cells) -- a bounded sample for slow legs."""
    from oracle import oracle as o

    o.set_num_threads(threads)
    s = cfg.system()
    sysm = o.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    ff2 = o.OracleForceField(nu=0.073, cutoff=cfg.rc_lj)
    ff3 = o.OracleForceField(nu=0.073, cutoff=cfg.rc_atm)

    def timed(cut, fn):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            grid = o.build_cell_grid(sysm, cut)
            base = None
            if stride > 1:
                base = np.arange(0, grid.num_cells, stride, dtype=np.int64)
            fn(grid, base)
            ts.append(time.perf_counter() - t0)
        scale = 1.0 if stride == 1 else grid.num_cells / len(base)
        return statistics.median(ts) * scale

    t_pair = timed(cfg.rc_lj, lambda g, b: o.c01_pair_pass(g, sysm, ff2, base_cells=b))
    t_trip = timed(cfg.rc_atm, lambda g, b: o.c01_triplet_pass(g, sysm, ff3, base_cells=b))
    x, v, f = sysm.positions.copy(), sysm.velocities.copy(), sysm.forces_2b.copy()
    t0 = time.perf_counter()
    for _ in range(reps):
        x += 0.001 * v + 0.5e-6 * f
        np.mod(x, sysm.box, out=x)
        v += 0.0005 * (f + f)
    t_int = (time.perf_counter() - t0) / reps
    return t_pair, t_trip, t_int


def cpu_baseline_leg(cfg):
    """The cpu_baseline object: the port's per-pass medians at all host
    cores and at 1 thread, extrapolated to r-RESPA steps/s (one pair pass +
    1/s triplet pass + one integration update per step)."""
    threads = os.cpu_count() or 1
    sf = cfg.step_size_factor
    t0 = time.perf_counter()
    tp, tt, ti = cpu_pass_medians(cfg, threads, reps=3)
    rate = 1.0 / (tp + tt / sf + ti)
    stride = 16 if cfg.name == "cfg4" else (4 if cfg.name in ("cfg3", "cfg5") else 1)
    tp1, tt1, ti1 = cpu_pass_medians(cfg, 1, reps=1, stride=stride)
    rate1 = 1.0 / (tp1 + tt1 / sf + ti1)
    detail = {}
    if cfg.name == "cfg4":  # per-pass medians of the cfg3 sweep points too
        import dataclasses

        from paper_2507_11172_b200 import systems

        for rc3 in (2.0, 2.5, 3.0):
            c3 = dataclasses.replace(systems.CONFIGS["cfg3"], rc_atm=rc3)
            p3, q3, _ = cpu_pass_medians(c3, threads, reps=1)
            detail[f"cfg3@{rc3}"] = {"pair_s": p3, "triplet_s": q3}
    return {
        "value": rate, "unit": "steps/s", "cores": threads, "kind": "port",
        "cpu_model": cpu_model(),
        "sample": (f"{cfg.name} step 0: medians of 3 pair passes ({tp:.3f} s) and 3 triplet passes "
                   f"({tt:.3f} s) incl. their binning, + one integration update ({ti:.3f} s), "
                   f"extrapolated to steps/s = 1 / (pair + triplet / {sf} + update); oracle/ C "
                   f"port of respamd's kernels, OpenMP {threads} threads"),
        "one_thread": {"value": rate1, "unit": "steps/s", "cores": 1,
                       "sample": f"the same passes on every {stride}-th base cell, scaled "
                                 f"(pair {tp1:.2f} s, triplet {tt1:.2f} s)"},
        "per_pass_s": {"pair": tp, "triplet": tt, "integration": ti, **detail},
        "note": "the port is bit-exact with respamd and faster than the stock numba package "
                "(BASELINE.md: cfg4 ~0.30 steps/s, cfg2 11.9 steps/s on 8 threads)",
        "leg_seconds": time.perf_counter() - t0,
    }


def reference_arm(args, cfg):
    """--impl reference: the port's own respa_run on this host's cores, same
    workload; a bounded number of timed steps (about a minute of CPU work)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import oracle as o

    o.set_num_threads(threads)
    s = cfg.system()
    ff = o.OracleForceField(nu=0.073, cutoff=cfg.rc_lj)
    sf = cfg.step_size_factor
    sysm = o.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    cont = o.OracleLinkedCells()
    t0 = time.perf_counter()
    o.respa_run(sysm, ff, cont, cfg.dt, sf, sf)  # warm-up cycle (also the calibration)
    t_cycle = time.perf_counter() - t0
    warm = sf
    budget = float(os.environ.get("RB_REFERENCE_SECONDS", "60"))
    cycles = int(max(1, min((args.steps + sf - 1) // sf, budget // max(t_cycle, 1e-3))))
    steps = cycles * sf
    t0 = time.perf_counter()
    o.respa_run(sysm, ff, cont, cfg.dt, sf, steps)
    elapsed = time.perf_counter() - t0
    rate = steps / elapsed
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d)",
        "config": {"workload": workload_name(cfg),
                   "timed": f"respa_run of {steps} steps incl. its two initial passes "
                            f"(bounded: {args.steps} requested, ~{budget:.0f} s of CPU work)"},
        "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
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
    """N > 1: strong scaling with the domain-decomposed r-RESPA (DESIGN.md
    §7): the same box as N = 1 (cfg4 by default) decomposed over the ranks
    (NCCL halo exchange); value = K / time, time = max over ranks of the
    CUDA-event time of steps W..W+K of one trajectory (whole-box steps/s)."""
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

    from paper_2507_11172_b200.grid import geometry

    sf = cfg.step_size_factor
    s = cfg.system()
    ff = cfg.force_field()
    cells = geometry(s.box, None, max(cfg.rc_lj, cfg.rc_atm) + 0.3, True).cells
    # the inhomogeneous slab (cfg5) gets cost-balanced blocks (domain.balanced_layout:
    # rank grid and cuts from the estimated work of the initial configuration)
    balance = cfg.name == "cfg5"
    dims = None if balance else auto_dims(world, tuple(int(c) for c in cells))
    K = max(sf, (int(args.steps) + sf - 1) // sf * sf)
    W = max(sf, (max(3, int(args.warmup)) + sf - 1) // sf * sf)
    L = pkg._lib.lib()
    backends = []

    decs = []

    def factory(dec, n_total, r_build):
        b = gpu_backend_factory(ff)(dec, n_total, r_build)
        backends.append(b)
        decs.append(dec)
        return b

    # one trajectory of W + K steps; steps W..W+K-1 are timed with two events
    # (the loop runs speculative multi-step windows, so a step can be repeated
    # after a rebuild: the window as a whole is what is timed); each rank's
    # working set (rows, partial-force buffer) is far above L2 at cfg4
    marks = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def on_step(i):
        if i == W:
            torch.cuda.synchronize()
            dist.barrier()
            marks["l0"] = L.rb_launch_count()
            ev0.record()
        if i == W + K:
            ev1.record()
            torch.cuda.synchronize()
            marks["l1"] = L.rb_launch_count()
            dist.barrier()

    run_sys = s.copy()
    with ClockSampler(local) as clocks:
        domain_respa_run(dist, run_sys, ff, pkg.RespaSchedule(cfg.dt, sf, W + K), factory,
                         dims=dims, on_step=on_step, balance=balance)
    step_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([step_ms, float(marks["l1"] - marks["l0"])], dtype=torch.float64,
                     device="cuda")
    mx, sm = t.clone(), t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms = float(mx[0].item())
    launches = int(sm[1].item())
    value = K / (ms * 1e-3)  # whole-box steps per second

    # e2e: the public decomposed run from host arrays (scatter, steps, gather)
    e2e_sys = s.copy()
    dist.barrier()
    t0 = time.perf_counter()
    domain_respa_run(dist, e2e_sys, ff, pkg.RespaSchedule(cfg.dt, sf, K),
                     gpu_backend_factory(ff), dims=dims, balance=balance)
    torch.cuda.synchronize()
    dist.barrier()
    e2e_s = time.perf_counter() - t0

    # dominant kernel: the ATM pass on this rank's local set (owned + ghosts)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = pkg._lib.stream_handle()
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
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d)",
            "config": {"workload": workload_name(cfg), "particles": s.n, "step_size_factor": sf,
                       "parallelism": f"domain decomposition {tuple(decs[0].dims) if decs else dims}"
                                      f"{' (cost-balanced blocks)' if balance else ''} "
                                      f"({dist.get_backend()} halo exchange)",
                       "value": "whole-box steps/s (the same box at every N)",
                       "timed": "steps W..W+K of one decomposed trajectory between two CUDA "
                                "events, max over ranks (speculative multi-step windows, "
                                "rebuild steps included)",
                       "l2": "not flushed: each rank's rows and partial-force buffer exceed L2"},
            "roofline": {"bound": "fp64", "kernel": "ATM triplet pass on rank 0's local set",
                         "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": achieved / peak.value if peak.value else None, "traffic": None,
                         "work": f"{FLOPS_PER_TRIPLET} FP64 flops per unique triplet x {unique} "
                                 f"triplets (owned + ghost bases)",
                         "kernel_ms": atm_ms},
            "e2e": {"value": K / e2e_s, "unit": "steps/s",
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


def _events(L, _lib, count):
    ev = []
    for _ in range(count):
        e = ctypes.c_void_p()
        _lib.check(L.rb_event_create(ctypes.byref(e)), "rb_event_create")
        ev.append(e)
    return ev


def device_loop(pkg, cfg, K, W, flush, clock_index):
    """K r-RESPA steps of cfg replayed from a captured sampling period, each
    step bracketed by event-record nodes (an L2 flush before each, outside
    the brackets).  Returns (dict, run)."""
    import torch

    from paper_2507_11172_b200 import _lib
    from paper_2507_11172_b200.integrators import DeviceRespa, RespaSchedule

    L = _lib.lib()
    sf = cfg.step_size_factor
    s = cfg.system()
    ff = cfg.force_field()
    periods = (K + sf - 1) // sf  # whole sampling periods replayed; exactly K steps timed
    W = (W + sf - 1) // sf * sf
    total_steps = sf + W + periods * sf + 2 * sf
    run = DeviceRespa(s, ff, pkg.CudaLinkedCells(), RespaSchedule(cfg.dt, sf, total_steps), sf)
    run.start()
    run.run_periods(0, 1)  # eager warm-up period: allocations, attributes
    ev = _events(L, _lib, 2 * sf)

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
    body = run.eng.cond_body_launches  # kernels of a conditional rebuild body (if any)
    launches_per_step = launches_per_period / sf - body
    for _ in range(W // sf):
        graph.replay()
    torch.cuda.synchronize()
    rebuilds0 = int(run.eng.status[3].item())
    ms = 0.0
    el = ctypes.c_float()
    with ClockSampler(clock_index) as clocks:
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
    return {"value": K / (ms * 1e-3), "ms_per_step": ms / K, "ms": ms,
            "launches_per_step": launches_per_step, "body": body, "rebuilds": rebuilds,
            "clocks": clocks.summary(), "n": s.n}, run


def time_kernel(torch, L, _lib, flush, fn, reps):
    stream = _lib.stream_handle()
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
    return statistics.median(ts)


def kernel_timings(run, flush):
    """The passes standalone on the run's final state (median of reps,
    L2 flushed before each, events on the launching stream)."""
    import torch

    from paper_2507_11172_b200 import _lib

    L = _lib.lib()
    eng, geom = run.eng, run._geom()
    eng.bin(geom, run.x)
    eng.nlist(geom, run.r_build, capacity=run.capacity, checked=True)
    eng.slots = run.slots
    f3 = torch.empty_like(run.f3)
    eng.reset_status(0)
    eng.atm(geom, run.rc3, run.nu, f3, tag=0, count_visits=True)
    torch.cuda.synchronize()
    unique = int(eng.visits.item())
    tk = lambda fn, reps: time_kernel(torch, L, _lib, flush, fn, reps)  # noqa: E731
    atm_ms = tk(lambda: eng.atm_kernel(geom, run.rc3, run.nu, f3, tag=0), 20)
    c01_ms = tk(lambda: eng.atm_c01(geom, run.rc3, run.nu, f3, tag=0, reduce=False), 5)
    lj_ms = tk(lambda: eng.lj_kernel(geom, run.rc2, 1.0, 1.0, f3, tag=0), 20)
    pairs = int(eng.row_count[: eng.n].sum().item())  # row entries (rc + skin)
    peak = ctypes.c_double(0.0)
    L.rb_fp64_peak(2000, ctypes.byref(peak), _lib.stream_handle())
    return {"atm_ms": atm_ms, "c01_ms": c01_ms, "lj_ms": lj_ms, "unique": unique,
            "pairs": pairs, "peak_tf": float(peak.value), "path":
            "cells" if eng.uses_cells(geom, run.rc3) else "rows"}


def hbm_timings(run, flush):
    """Binning (rb_bin) and the fused kick + drift of a sampling period
    (rb_respa_kick_drift) timed standalone; achieved GB/s on SURVEY §8d's
    algorithmic bytes (binning 28 B/particle + 4 B/cell; drift + kick 192
    B/particle) against the measured copy peak."""
    import torch

    from paper_2507_11172_b200 import _lib
    from paper_2507_11172_b200._lib import ptr

    L = _lib.lib()
    eng, geom = run.eng, run._geom()
    n, ncell = run.n, geom.num_cells
    tk = lambda fn, reps: time_kernel(torch, L, _lib, flush, fn, reps)  # noqa: E731
    bin_ms = tk(lambda: eng.bin(geom, run.x), 20)
    box = run.box.ctypes.data_as(ctypes.c_void_p)
    common = (ptr(eng.rank_of), ptr(eng.pos_r), ptr(eng.x_ref), run.skin, ptr(eng.rebuild_flag),
              ptr(eng.status))

    def kick_drift():
        _lib.check(L.rb_respa_kick_drift(n, ptr(run.x), ptr(run.v), ptr(run.f2_old),
                                         ptr(run.f2_new), ptr(run.f3), box, int(run.periodic),
                                         run.dt, run.half_dt, run.half_drift, run.half_respa, 0,
                                         0, *common, 0, eng.stream), "rb_respa_kick_drift")

    step_ms = tk(kick_drift, 20)
    eng.reset_status(0)
    bin_bytes = BIN_BYTES_PER_PARTICLE * n + BIN_BYTES_PER_CELL * ncell
    step_bytes = STEP_BYTES_PER_PARTICLE * n
    return {
        "peak_gbs": HBM_PEAK_GBS, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)",
        "binning": {"kernels": "rb_bin (count, scan, scatter, cell finish)", "ms": bin_ms,
                    "algorithmic_bytes": bin_bytes,
                    "achieved_gbs": bin_bytes / (bin_ms * 1e-3) / 1e9,
                    "frac": bin_bytes / (bin_ms * 1e-3) / 1e9 / HBM_PEAK_GBS},
        "integration": {"kernels": "rb_respa_kick_drift (kick of step i-1 + drift of step i)",
                        "ms": step_ms, "algorithmic_bytes": step_bytes,
                        "achieved_gbs": step_bytes / (step_ms * 1e-3) / 1e9,
                        "frac": step_bytes / (step_ms * 1e-3) / 1e9 / HBM_PEAK_GBS},
    }


def e2e_rate(pkg, cfg, steps):
    """The public respa_run on host numpy arrays, wall clock incl. upload,
    initial passes, the steps and the download; median of three calls after
    a warm-up call (the calls share one cached device run, as a user's
    repeated calls do)."""
    import torch

    sf = cfg.step_size_factor
    steps = (steps + sf - 1) // sf * sf
    ff = cfg.force_field()
    # two warm-up calls of the same shape: the first sizes the rows and
    # captures the period graph, the second the initial passes' graph
    for _ in range(2):
        pkg.respa_run(cfg.system(), ff, pkg.CudaLinkedCells(),
                      pkg.RespaSchedule(cfg.dt, sf, steps))
    runs = []
    for _ in range(3):
        host = cfg.system()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pkg.respa_run(host, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(cfg.dt, sf, steps))
        torch.cuda.synchronize()
        runs.append(time.perf_counter() - t0)
    e2e_s = statistics.median(runs)
    n = host.positions.shape[0]
    h2d = 2 * n * 24  # positions + velocities
    d2h = 4 * n * 24 + (steps // sf + 1) * 64  # x, v, f2, f3 + trace rows
    return {"value": steps / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": h2d / steps,
            "d2h_bytes_per_step": d2h / steps,
            "note": f"public respa_run({steps} steps) on host numpy arrays, wall clock incl. "
                    f"upload, initial passes, download; median of 3 calls "
                    f"({', '.join(f'{1e3 * t:.1f}' for t in runs)} ms)"}


def trajectory_rate(pkg, cfg, steps, flush):
    """A whole `steps`-step trajectory (BASELINE's run length) replayed from
    the captured period graph after one warm-up period, timed with two
    events around all of it: rebuild steps included, no per-step flush."""
    import torch

    from paper_2507_11172_b200.integrators import DeviceRespa, RespaSchedule

    sf = cfg.step_size_factor
    run = DeviceRespa(cfg.system(), cfg.force_field(), pkg.CudaLinkedCells(),
                      RespaSchedule(cfg.dt, sf, steps + 2 * sf), sf)
    run.start()
    run.run_periods(0, 1)
    run.capture()
    torch.cuda.synchronize()
    r0 = int(run.eng.status[3].item())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run.run_periods(1, steps // sf)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if run.eng.read_status() is not None or run.eng.overflowed():
        raise RuntimeError("device error during the trajectory")
    return {"value": steps / (ms * 1e-3), "unit": "steps/s", "steps": steps, "ms": ms,
            "rebuild_steps": int(run.eng.status[3].item()) - r0,
            "note": f"{steps}-step trajectory timed whole (rebuild steps included)"}


def atm_traffic(name):
    """DRAM bytes (read + write) per launch of the ATM kernel at a config, from
    the committed `ncu --set full` capture (profiles/atm_traffic_<cfg>.json)."""
    prof = os.path.join(REPO, "profiles", f"atm_traffic_{name}.json")
    try:
        return json.load(open(prof)).get("bytes_per_launch")
    except (OSError, ValueError):
        return None


def roofline_obj(kt, traffic):
    triplets_per_s = kt["unique"] / (kt["atm_ms"] * 1e-3)
    achieved = triplets_per_s * FLOPS_PER_TRIPLET / 1e12
    peak = kt["peak_tf"]
    return {"bound": "fp64", "kernel": f"ATM triplet pass ({kt['path']}-based, k_atm3 + gather)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak > 0 else None, "traffic": traffic,
            "peak_source": "measured in this run: rb_fp64_peak DFMA chains on all SMs "
                           "(MEASURED_PEAKS.json has no FP64 entry)",
            "work": f"{FLOPS_PER_TRIPLET} FP64 flops per unique triplet x {kt['unique']} "
                    f"unique triplets per launch",
            "kernel_ms": kt["atm_ms"], "triplets_per_s": triplets_per_s,
            "c01_kernel_ms": kt["c01_ms"], "c01_triplets_per_s": kt["unique"] / (kt["c01_ms"] * 1e-3),
            "lj_kernel_ms": kt["lj_ms"], "lj_row_entries": kt["pairs"],
            "lj_pairs_per_s": kt["pairs"] / 2 / (kt["lj_ms"] * 1e-3)}


def ours_arm(args, cfg):
    import torch

    world, rank, local = dist_env()
    if world > 1:
        return domain_arm(args, cfg)
    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200 import _lib, systems

    _lib.require_device()
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K, W = int(args.steps), max(3, int(args.warmup))
    sf = cfg.step_size_factor
    loop, run = device_loop(pkg, cfg, K, W, flush, local)
    kt = kernel_timings(run, flush)
    hbm = hbm_timings(run, flush)
    traffic = atm_traffic(cfg.name)
    del run
    e2e = e2e_rate(pkg, cfg, K)
    secondary = None
    if not args.no_secondary and cfg.name != "cfg2":
        c2 = systems.CONFIGS["cfg2"]
        loop2, run2 = device_loop(pkg, c2, min(max(K, 20), 200), W, flush, local)
        kt2 = kernel_timings(run2, flush)
        del run2
        secondary = {
            "workload": WORKLOADS["cfg2"], "value": loop2["value"], "unit": "steps/s",
            "ms_per_step": loop2["ms_per_step"], "rebuild_steps": loop2["rebuilds"],
            "trajectory_100": trajectory_rate(pkg, c2, 100, flush),
            "e2e": e2e_rate(pkg, c2, 20),
            "roofline": roofline_obj(kt2, atm_traffic("cfg2")),
            "note": "BASELINE.json configs[1] (32,000 particles) on one GPU; value as the "
                    "headline (device-timed steps); trajectory_100 = its 100-step run timed whole",
        }
    line = {
        "metric": METRIC, "value": loop["value"], "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": loop["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded FCC lattice + jitter, SURVEY.md §8d; no public dataset)",
        "config": {"workload": workload_name(cfg), "particles": loop["n"],
                   "step_size_factor": sf, "parallelism": "single GPU",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "graph": "one CUDA graph per 5-step sampling period; each step bracketed "
                            "by external event-record nodes (flush outside the brackets)"},
        "roofline": roofline_obj(kt, traffic),
        "hbm": hbm,
        "e2e": e2e,
        "gpu_launches": int(round(loop["launches_per_step"] * K)) + K,
        "gpu_launches_detail": {"per_step": loop["launches_per_step"], "l2_flush_per_step": 1,
                                "timing": "per-step external event-record nodes inside the "
                                          "period graph",
                                "rebuild_steps": loop["rebuilds"]},
        "clocks": loop["clocks"],
    }
    if secondary is not None:
        line["secondary"] = secondary
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)


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
