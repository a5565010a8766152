"""Device-resident r-RESPA loop (the reference's L3, integrators.py:96-191).

``respa_run`` keeps the reference signature and semantics
(``respa_run(system, ff, container, schedule, sample_interval=None,
hooks=()) -> RunTrace``) but runs every step on the GPU:

* the state lives in HBM as the reference's (n,3) float64 arrays; the host
  copy is written back at hook points and at the end of the run;
* per base step: drift kernel (kick3 fused in at cycle starts), binning,
  survivor rows, LJ pass, kick kernel (kick3 fused in at cycle ends, after
  the triplet pass, which is recomputed only every ``s``-th step);
* the rounding order of every update is numpy's (bit-exact trajectories
  given identical forces);
* failures (minimum separation, non-finite state) are recorded in a device
  status word with the iteration they happened in; later kernels become
  no-ops, so the state freezes exactly where ``IntegrationBlowUp`` would
  have been raised, and the host raises it with the same iteration number;
* one sampling period of steps is captured once as a CUDA graph and
  replayed; the trace (kinetic energy, container scalars) is recorded on the
  device and read back once.

The container must be a :class:`~.containers.CudaLinkedCells`; there is no
host fallback.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ptr
from .containers import CudaDirectSum, CudaLinkedCells, MinimumSeparationError, engine_for
from .engine import (SCALAR_E2, SCALAR_E3, SCALAR_W2, SCALAR_W3, CapacityError,
                     _round_up)
from .grid import geometry
from .model import ValidationError, triplet_cutoff


class IntegrationBlowUp(RuntimeError):
    """State became non-finite or near-singular (``integrators.py:29-35``)."""

    def __init__(self, iteration: int, reason: str, trace=None):
        self.iteration = iteration
        self.trace = trace if trace is not None else RunTrace()
        super().__init__(f"integration blew up at iteration {iteration}: {reason}")


@dataclass
class RespaSchedule:
    """Base step, step-size factor, iteration count (``integrators.py:38-60``)."""

    dt: float
    step_size_factor: int = 1
    num_iterations: int = 0

    def __post_init__(self):
        self.dt = float(self.dt)
        self.step_size_factor = int(self.step_size_factor)
        self.num_iterations = int(self.num_iterations)
        if not np.isfinite(self.dt) or self.dt <= 0:
            raise ValidationError(f"dt must be finite and > 0, got {self.dt}")
        if self.step_size_factor < 1:
            raise ValidationError("step_size_factor must be >= 1")
        if self.num_iterations < 0:
            raise ValidationError("num_iterations must be >= 0")
        if self.num_iterations % self.step_size_factor:
            raise ValidationError(
                f"num_iterations ({self.num_iterations}) must be a multiple of "
                f"the step_size_factor ({self.step_size_factor})"
            )


@dataclass
class RunTrace:
    """Observables at full iterations (``integrators.py:63-86``)."""

    iterations: list = field(default_factory=list)
    kinetic: list = field(default_factory=list)
    potential_2b: list = field(default_factory=list)
    potential_3b: list = field(default_factory=list)
    total: list = field(default_factory=list)
    virial_2b: list = field(default_factory=list)
    virial_3b: list = field(default_factory=list)

    def record_values(self, iteration, kinetic, e2, w2, e3, w3) -> None:
        self.iterations.append(int(iteration))
        self.kinetic.append(float(kinetic))
        self.potential_2b.append(float(e2))
        self.potential_3b.append(float(e3))
        self.total.append(float(kinetic) + float(e2) + float(e3))
        self.virial_2b.append(float(w2))
        self.virial_3b.append(float(w3))

    def record(self, iteration: int, system, container) -> None:
        kin = 0.5 * system.mass * float(np.sum(system.velocities * system.velocities))
        self.record_values(iteration, kin, container.pair_energy, container.pair_virial,
                           container.triplet_energy, container.triplet_virial)

    def __len__(self):
        return len(self.iterations)


_MSG = {
    _lib.RB_KIND_PAIR_MIN_SEPARATION: "particles closer than the minimum separation guard; "
                                      "the configuration is (nearly) singular",
    _lib.RB_KIND_TRIPLET_MIN_SEPARATION: "particles closer than the minimum separation guard; "
                                         "the configuration is (nearly) singular",
    _lib.RB_KIND_NONFINITE: "non-finite position or velocity",
}


class DeviceRespa:
    """One device-resident r-RESPA run (all buffers allocated up front).

    Periodic systems use Verlet rows built at r_list + ``skin``: the drift of
    each step flags a rebuild when some particle moved more than skin/2 since
    the last build, and the (gated) binning / row kernels then run inside the
    same step, so every pair within the cutoff is always in the rows.  Open
    systems rebuild every step (their grid follows the particles)."""

    DEFAULT_SKIN = float(os.environ.get("RB_SKIN", "0.3"))  # Verlet skin (sigma)

    def __init__(self, system, ff, container, schedule: RespaSchedule, sample_interval: int,
                 capacity: Optional[int] = None, use_graph: bool = True,
                 skin: Optional[float] = None):
        self.system = system
        self.ff = ff
        self.container = container
        self.schedule = schedule
        self.interval = int(sample_interval)
        self.n = int(system.positions.shape[0])
        self.periodic = bool(system.periodic)
        # DirectSum container: all pairs / triplets, no grid (open systems only)
        self.direct = isinstance(container, CudaDirectSum)
        if self.direct and self.periodic:
            raise ValidationError("DirectSum does not support periodic boundaries")
        # open linked-cell systems need a host-synchronised grid every step
        self.use_graph = use_graph and (self.periodic or self.direct)
        self.eng = engine_for(self.n, run=True)  # device workspace cached per particle count
        torch = self.torch = self.eng.torch
        dev, f64 = self.eng.device, torch.float64
        self.x = self.eng.pos  # positions live in the engine's buffer
        self.v = torch.zeros((self.n, 3), dtype=f64, device=dev)
        self.f2_old = torch.zeros((self.n, 3), dtype=f64, device=dev)
        self.f2_new = torch.zeros((self.n, 3), dtype=f64, device=dev)
        self.f3 = torch.zeros((self.n, 3), dtype=f64, device=dev)
        self.rc2 = float(ff.cutoff)
        self.rc3 = triplet_cutoff(ff)
        self.nu = float(ff.nu)
        self.with_3b = self.nu != 0.0
        self.r_list = max(self.rc2, self.rc3) if self.with_3b else self.rc2
        self.box = np.ascontiguousarray(system.box, dtype=np.float64)
        if self.periodic:
            want = self.DEFAULT_SKIN if skin is None else float(skin)
            # the rows' grid needs box >= 2 (r_list + skin) (containers.py:248-252)
            self.skin = max(0.0, min(want, float(np.min(self.box)) / 2.0 - self.r_list))
        else:
            self.skin = 0.0
        self.r_build = self.r_list + self.skin
        s = schedule.step_size_factor
        m = float(system.mass)
        dt = schedule.dt
        self.dt = dt
        self.half_dt = 0.5 * dt / m
        self.half_drift = 0.5 * dt * dt / m
        self.half_respa = 0.5 * dt * s / m
        nsamples = schedule.num_iterations // self.interval + 1
        self.trace_dev = torch.zeros((nsamples, 8), dtype=f64, device=dev)
        self.capacity = capacity
        self.slots = None
        self.geom = None
        self.graph = None
        # the gated rebuild of a step: one fused launch (rb_rebuild, default),
        # or (RB_REBUILD=cond) the nine kernels in a conditional graph node,
        # or (RB_REBUILD=gated) the nine gated launches
        mode = os.environ.get("RB_REBUILD", "fused")
        self.cond_rebuild = mode == "cond"
        self.fused_rebuild = mode == "fused"
        # inside a sampling period a step's kick runs in the next drift
        self.fuse_kick = os.environ.get("RB_FUSE_KICK", "1") != "0"
        # three-body steps: the pair pass on a second stream beside the
        # triplet kernels (periodic Verlet-row loop only)
        self.overlap_pair = os.environ.get("RB_OVERLAP_PAIR", "1") != "0"
        # ... started after the persistent triplet kernel, beside the gather
        # (RB_PAIR_WITH_GATHER=0: from the start, filling the triplet tail)
        self.pair_with_gather = os.environ.get("RB_PAIR_WITH_GATHER", "1") != "0"

    def cache_key(self):
        """What the captured period graph bakes in (kernel arguments and
        buffer shapes): a run of the same key can replay it."""
        ff = self.ff
        return (self.n, tuple(float(b) for b in self.box), self.periodic,
                float(self.system.mass), float(ff.epsilon), float(ff.sigma), self.nu, self.rc2,
                self.rc3, type(self.container).__name__, self.dt,
                self.schedule.step_size_factor, self.interval, self.skin, self.use_graph,
                self.capacity, self.slots)

    def rebind(self, system, container, schedule: RespaSchedule) -> bool:
        """Reuse this run (buffers, rows, captured graph) for another run of
        the same shape; False when its trace rows are too few."""
        nsamples = schedule.num_iterations // self.interval + 1
        if nsamples > self.trace_dev.shape[0]:
            return False
        self.system, self.container, self.schedule = system, container, schedule
        return True

    # -------------------------------------------------------------- pieces
    def _geom(self):
        if self.periodic:
            if self.geom is None:
                self.geom = geometry(self.box, None, self.r_build, True)
            return self.geom
        lo_hi = self.torch.aminmax(self.x, dim=0)
        pos = np.stack([lo_hi.min.cpu().numpy(), lo_hi.max.cpu().numpy()])
        if not np.all(np.isfinite(pos)):
            return None  # the drift already recorded the non-finite state
        return geometry(self.box, pos, self.r_build, False)

    def _forces(self, tag: int, with_triplet: bool, f2_out, cond: int = 0,
                scalars: bool = True) -> None:
        """The step's passes.  scalars=False: the pair pass computes forces
        only (a step inside a sampling period that is not its sample point:
        nothing reads its pair energy / virial)."""
        eng = self.eng
        if self.direct:
            eng.direct_pairs(self.ff.epsilon, self.ff.sigma, f2_out, tag=tag, reduce=False)
            if with_triplet:
                if self.with_3b:
                    eng.direct_triplets(self.nu, self.f3, tag=tag)
                    # E3, W3 come as totals: one entry of the per-rank arrays
                    eng.e3_rank.zero_()
                    eng.w3_rank.zero_()
                    eng.e3_rank[:1].copy_(eng.scalars[SCALAR_E3:SCALAR_E3 + 1])
                    eng.w3_rank[:1].copy_(eng.scalars[SCALAR_W3:SCALAR_W3 + 1])
                else:
                    self.f3.zero_()
                    eng.e3_rank.zero_()
                    eng.w3_rank.zero_()
            return
        geom = self._geom()
        if geom is None:
            # open system with non-finite positions: forces are undefined;
            # the step is already marked RB_KIND_NONFINITE (integrators.py:166-170)
            f2_out.fill_(float("nan"))
            if with_triplet:
                self.f3.fill_(float("nan"))
            return
        if self.periodic:  # Verlet rows: rebuild only when the drift flagged it
            eng.rebuild(geom, self.r_build, self.capacity, self.x, tag=tag, cond=cond,
                        fused=self.fused_rebuild)
        else:
            eng.bin(geom, self.x, tag=tag)
            eng.nlist(geom, self.r_build, capacity=self.capacity, checked=False, tag=tag)
        if with_triplet and self.with_3b and self.overlap_pair:
            # the triplet kernels first, the pair pass on a second stream
            # (a parallel graph branch): its blocks fill the SMs the triplet
            # pass releases in its tail; the gather, which alone writes the
            # triplet outputs, runs after both
            torch = self.torch
            main = torch.cuda.current_stream()
            side = self._pair_stream = getattr(self, "_pair_stream", None) or torch.cuda.Stream()
            if self.pair_with_gather:
                # the pair pass (L1-bound) beside the gather (HBM-bound):
                # both start when the persistent triplet kernel ends
                eng.atm_kernel(geom, self.rc3, self.nu, self.f3, tag=tag, part=1)
                side.wait_stream(main)
            else:
                side.wait_stream(main)
                eng.atm_kernel(geom, self.rc3, self.nu, self.f3, tag=tag, part=1)
            with torch.cuda.stream(side):
                eng.lj(geom, self.rc2, self.ff.epsilon, self.ff.sigma, f2_out, tag=tag,
                       reduce=False, scalars=scalars)
            if self.pair_with_gather:
                eng.atm_kernel(geom, self.rc3, self.nu, self.f3, tag=tag, part=2)
                main.wait_stream(side)
            else:
                main.wait_stream(side)
                eng.atm_kernel(geom, self.rc3, self.nu, self.f3, tag=tag, part=2)
            return
        eng.lj(geom, self.rc2, self.ff.epsilon, self.ff.sigma, f2_out, tag=tag, reduce=False,
               scalars=scalars)
        if with_triplet:
            if self.with_3b:
                eng.atm(geom, self.rc3, self.nu, self.f3, tag=tag, count_visits=False,
                        reduce=False)
            else:
                self.f3.zero_()
                self.eng.e3_rank.zero_()
                self.eng.w3_rank.zero_()

    def _reduce_scalars(self) -> None:
        self.eng.reduce_pair()
        self.eng.reduce_triplet()

    def _record(self) -> None:
        # sums of the five trace scalars + the trace row, one launch
        self.eng.sample(self.v, self.trace_dev, self.interval)

    def _step(self, i: int, j: Optional[int] = None) -> None:
        """Loop body of integrators.py:148-172 for iteration i (tag i+1).

        j = position of the step inside a sampling period (None: a step on
        its own).  Inside a period the kick that ends step i is folded into
        the drift of step i+1 (rb_respa_kick_drift, one pass over the
        particles, bit-identical); the period's last step kicks itself, so
        the sample point and the host see completed steps."""
        L, eng = self.eng.L, self.eng
        s = self.schedule.step_size_factor
        verlet = self.periodic
        null = ctypes.c_void_p(0)
        fuse = self.fuse_kick and j is not None and j > 0
        defer = self.fuse_kick and j is not None and j < self.interval - 1
        # under capture: the drift sets the rebuild conditional with the flag
        cond = eng.rebuild_cond() if verlet and self.cond_rebuild else 0
        box = self.box.ctypes.data_as(ctypes.c_void_p)
        common = (ptr(eng.rank_of) if verlet else null, ptr(eng.pos_r) if verlet else null,
                  ptr(eng.x_ref) if verlet else null, self.skin,
                  ptr(eng.rebuild_flag) if verlet else null, ptr(eng.status))
        if fuse:  # the kick of step i-1, then the drift opening step i
            st = L.rb_respa_kick_drift(self.n, ptr(self.x), ptr(self.v), ptr(self.f2_old),
                                       ptr(self.f2_new), ptr(self.f3), box, int(self.periodic),
                                       self.dt, self.half_dt, self.half_drift, self.half_respa,
                                       int(i % s == 0), int(i % s == 0), *common, cond,
                                       eng.stream)
            _lib.check(st, "rb_respa_kick_drift")
        else:  # the drift opens the device step (status[1] = last closed + 1)
            st = L.rb_respa_drift(self.n, ptr(self.x), ptr(self.v), ptr(self.f2_old),
                                  ptr(self.f3), box, int(self.periodic), self.dt,
                                  self.half_drift, self.half_respa, int(i % s == 0), *common,
                                  _lib.RB_TAG_FROM_DEVICE, 1, cond, eng.stream)
            _lib.check(st, "rb_respa_drift")
        end_of_cycle = (i + 1) % s == 0
        # pair scalars only where something reads them: the period's sample
        # point, and every step run on its own (the last pass of a run feeds
        # the container's scalars)
        sample = j is None or (i + 1) % self.interval == 0
        self._forces(_lib.RB_TAG_FROM_DEVICE, end_of_cycle, self.f2_new, cond, scalars=sample)
        if not defer:
            st = L.rb_respa_kick(self.n, ptr(self.v), ptr(self.f2_old), ptr(self.f2_new),
                                 ptr(self.f3), self.half_dt, self.half_respa, int(end_of_cycle),
                                 ptr(eng.status), _lib.RB_TAG_FROM_DEVICE, eng.stream)
            _lib.check(st, "rb_respa_kick")
        if (i + 1) % self.interval == 0:
            self._record()

    def _period(self, first: int) -> None:
        for j in range(self.interval):
            self._step(first + j, j)

    # ----------------------------------------------------------------- run
    def _pinned(self):
        """Page-locked host staging of the run's transfers (allocated once)."""
        if getattr(self, "_pin", None) is None:
            t, n = self.torch, self.n

            def pin(shape, dtype):
                return t.empty(shape, dtype=dtype, pin_memory=True)

            self._pin = dict(x=pin((n, 3), t.float64), v=pin((n, 3), t.float64),
                             f2=pin((n, 3), t.float64), f3=pin((n, 3), t.float64),
                             trace=pin(tuple(self.trace_dev.shape), t.float64),
                             scalars=pin((8,), t.float64), status=pin((4,), t.int64),
                             maxc=pin((1,), t.int32))
        return self._pin

    def start(self) -> None:
        """Upload, initial passes (integrators.py:133-137) and sample 0."""
        torch, eng = self.torch, self.eng
        pin = self._pinned()  # host arrays -> page-locked staging -> async copies
        _host_copy(pin["x"], self.system.positions)
        _host_copy(pin["v"], self.system.velocities)
        eng.pos[: self.n].copy_(pin["x"], non_blocking=True)
        self.v.copy_(pin["v"], non_blocking=True)
        if self.graph is not None:
            # a cached run (same shape, rows and slots sized): the initial
            # passes replay as one graph (captured on the first reuse)
            if getattr(self, "start_graph", None) is None:
                self.start_graph = self._captured(self._initial_passes)
            self.start_graph.replay()
            return
        eng.reset_status(0)
        eng.rebuild_flag.zero_()  # tag 0 == forced build for the initial passes
        if not self.direct and (self.capacity is None or self.slots is None):
            geom = self._geom()
            eng.bin(geom, self.x)
            # rows (at r_list + skin) and the triplet pass's shared-memory slots
            # (at most the neighbours within the three-body cutoff) are sized
            # from the initial configuration with margin; an overflow later is
            # detected on the device and the run is repeated larger
            if self.with_3b:
                eng.nlist(geom, self.rc3, capacity=None, checked=True)
                within = int(eng.max_count.item())
            eng.nlist(geom, self.r_build, capacity=None, checked=True)
            longest = int(eng.max_count.item())
            if self.capacity is None:
                self.capacity = min(4096, _round_up(int(longest * 1.3) + 16, 32))
            if self.slots is None:
                self.slots = self.capacity if not self.with_3b else min(
                    self.capacity, _round_up(int(within * 1.25) + 8, 32))
        eng.max_count.zero_()
        eng.slots = self.slots
        self._forces(0, True, self.f2_old)
        self._record()

    def _initial_passes(self) -> None:
        """start() after the upload, for a run whose rows and slots are sized
        (device work only: capturable)."""
        eng = self.eng
        eng.reset_status(0)
        eng.rebuild_flag.zero_()  # tag 0 == forced build for the initial passes
        eng.max_count.zero_()
        eng.slots = self.slots
        self._forces(0, True, self.f2_old)
        self._record()

    def finish_scalars(self) -> None:
        """Container scalars of the most recent passes (integrators.py:74-83)."""
        self._reduce_scalars()

    def _captured(self, body):
        """CUDA graph of `body` captured on a side stream.  (torch.cuda.graph
        would also empty the allocator cache on entry: a device-wide
        cudaFree of every cached block, hundreds of ms after a large run.)"""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        cur = torch.cuda.current_stream()
        side = self._side_stream = getattr(self, "_side_stream", None) or torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            g.capture_begin()
            try:
                body()
            finally:
                g.capture_end()
        cur.wait_stream(side)
        return g

    def capture(self) -> None:
        """Capture one sampling period as a CUDA graph (after a warm-up)."""
        self.graph = self._captured(lambda: self._period(0))

    def capture_steps(self):
        """One CUDA graph per step position inside a sampling period (the
        step kinds repeat with the period), for per-step timing."""
        return [self._captured(lambda j=j: self._step(j, j)) for j in range(self.interval)]

    def run_periods(self, first_period: int, count: int) -> None:
        for k in range(first_period, first_period + count):
            if self.graph is not None:
                self.graph.replay()
            else:
                self._period(k * self.interval)

    def collect(self, upto: int) -> dict:
        """Every result of the run to the host in one synchronisation: the
        status words, the row high-water mark, the trace rows, the state and
        the container scalars (async copies into page-locked buffers)."""
        pin, eng = self._pinned(), self.eng
        pin["status"].copy_(eng.status, non_blocking=True)
        pin["maxc"].copy_(eng.max_count, non_blocking=True)
        pin["trace"][:upto].copy_(self.trace_dev[:upto], non_blocking=True)
        pin["x"].copy_(self.x[: self.n], non_blocking=True)
        pin["v"].copy_(self.v, non_blocking=True)
        pin["f2"].copy_(self.f2_old, non_blocking=True)
        pin["f3"].copy_(self.f3, non_blocking=True)
        pin["scalars"].copy_(eng.scalars, non_blocking=True)
        self.torch.cuda.current_stream().synchronize()
        return pin

    def apply_collected(self, pin) -> None:
        """The collected state into the host system and the container."""
        sysm = self.system
        _host_copy(sysm.positions, pin["x"])
        _host_copy(sysm.velocities, pin["v"])
        _host_copy(sysm.forces_2b, pin["f2"])
        _host_copy(sysm.forces_3b, pin["f3"])
        sc = pin["scalars"].numpy()
        c = self.container
        c.pair_energy, c.pair_virial = float(sc[SCALAR_E2]), float(sc[SCALAR_W2])
        c.triplet_energy, c.triplet_virial = float(sc[SCALAR_E3]), float(sc[SCALAR_W3])

    def download(self) -> None:
        sysm = self.system
        sysm.positions[:] = self.x.cpu().numpy()
        sysm.velocities[:] = self.v.cpu().numpy()
        sysm.forces_2b[:] = self.f2_old.cpu().numpy()
        sysm.forces_3b[:] = self.f3.cpu().numpy()

    def trace_rows(self, upto: int) -> np.ndarray:
        return self.trace_dev[:upto].cpu().numpy()

    def update_container(self) -> None:
        sc = self.eng.scalar_values()
        c = self.container
        c.pair_energy, c.pair_virial = float(sc[SCALAR_E2]), float(sc[SCALAR_W2])
        c.triplet_energy, c.triplet_virial = float(sc[SCALAR_E3]), float(sc[SCALAR_W3])


def _host_copy(dst, src) -> None:
    """dst[:] = src between host arrays / page-locked tensors, with torch's
    multi-threaded copy for large arrays (numpy's is single-threaded: ~20 ms
    per 49 MB array at 2 M particles)."""
    import torch

    d = dst if isinstance(dst, torch.Tensor) else None
    s_ = src if isinstance(src, torch.Tensor) else None
    try:
        if d is None:
            d = torch.from_numpy(dst)
        if s_ is None:
            s_ = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
        if d.shape == s_.shape and d.dtype == s_.dtype:
            d.copy_(s_)
            return
    except (TypeError, ValueError, RuntimeError):
        pass
    dst[:] = src.numpy() if isinstance(src, torch.Tensor) else src


def _fill_trace(trace: RunTrace, rows: np.ndarray, mass: float) -> None:
    for row in rows:
        trace.record_values(int(round(row[0])), 0.5 * mass * row[1], row[2], row[3], row[4], row[5])


LAST_RUN = [None]  # the DeviceRespa of the most recent respa_run (diagnostics)


def respa_run(system, ff, container, schedule: RespaSchedule, sample_interval: Optional[int] = None,
              hooks=(), use_graph: bool = True, capacity: Optional[int] = None,
              skin: Optional[float] = None, device_hooks=()) -> RunTrace:
    """Integrate in place with the r-RESPA loop on the GPU (integrators.py:96-173).

    ``hooks`` are the reference's host hooks (iteration, system view,
    container) at every sample point -- they force a download per period.
    ``device_hooks`` are called as hook(iteration, positions) at the same
    points with the device positions (particle order) and must only enqueue
    device work (e.g. accumulate an RDF histogram): no synchronisation.

    A neighbour-row overflow on the device (no reference analogue) repeats
    the run from the initial state with larger rows.  Before a repeat every
    hook with a ``reset()`` method is reset, so its state reflects only the
    attempt that completes; a hook without one sees the repeated iterations
    again (the reference never repeats a run)."""
    if not isinstance(container, (CudaLinkedCells, CudaDirectSum)):
        raise TypeError("respa_run needs a CudaLinkedCells or CudaDirectSum container "
                        "(GPU only, no host fallback)")
    s = schedule.step_size_factor
    if sample_interval is None:
        sample_interval = s
    sample_interval = int(sample_interval)
    if sample_interval < 1 or sample_interval % s != 0:
        raise ValidationError(
            f"sample_interval ({sample_interval}) must be a positive multiple "
            f"of the step_size_factor ({s})"
        )
    hooks = tuple(hooks)
    # the state to repeat a run from after a row overflow: without host hooks
    # the host arrays are written only after the run succeeded (apply_collected)
    x0 = np.array(system.positions, copy=True) if hooks else None
    v0 = np.array(system.velocities, copy=True) if hooks else None
    slots = None
    for attempt in range(3):
        run = _cached_run(system, ff, container, schedule, sample_interval, capacity,
                          use_graph and not hooks, skin) if attempt == 0 else None
        if run is None:
            run = DeviceRespa(system, ff, container, schedule, sample_interval,
                              capacity=capacity, use_graph=use_graph and not hooks, skin=skin)
            run.slots = slots
        LAST_RUN[0] = run
        try:
            run.eng.busy = True
            trace = _drive(run, hooks, tuple(device_hooks))
            _keep_run(run, capacity, skin)
            return trace
        except CapacityError:
            _RUNS.pop(_run_key(run.n, sample_interval, capacity, skin), None)
            capacity = min(4096, _round_up(int(run.capacity * 1.5) + 32, 32))
            slots = capacity
            run.eng.grow_cells()
            if x0 is not None:
                system.positions[:] = x0
                system.velocities[:] = v0
            _reset_hooks(hooks + tuple(device_hooks))
        finally:
            run.eng.busy = False
    raise CapacityError("neighbour rows kept overflowing")


# The most recent graph-driven run per (n, sample interval, requested
# capacity, skin): its buffers, rows and captured period graph are reused by
# the next respa_run of the same shape (DeviceRespa.cache_key), which then
# pays upload, the initial passes, the replays and the download -- no
# allocation, capture or eager warm-up period.
_RUNS = {}


def _run_key(n, interval, capacity, skin):
    return (int(n), int(interval), capacity, skin)


def _cached_run(system, ff, container, schedule, interval, capacity, use_graph, skin):
    if not use_graph:
        return None
    run = _RUNS.get(_run_key(system.positions.shape[0], interval, capacity, skin))
    if run is None or run.graph is None or run.eng.busy:
        return None
    probe = DeviceRespa.__new__(DeviceRespa)  # the key of the new run, without allocating
    probe.ff, probe.system, probe.container, probe.schedule = ff, system, container, schedule
    probe.n, probe.periodic = system.positions.shape[0], bool(system.periodic)
    probe.box = np.ascontiguousarray(system.box, dtype=np.float64)
    probe.nu, probe.rc2, probe.rc3 = float(ff.nu), float(ff.cutoff), triplet_cutoff(ff)
    probe.dt, probe.interval = schedule.dt, int(interval)
    probe.skin, probe.use_graph = run.skin, use_graph
    probe.capacity, probe.slots = run.capacity, run.slots
    if probe.cache_key() != run.cache_key():
        return None
    if skin is not None and run.skin != min(float(skin), run.skin):
        return None
    return run if run.rebind(system, container, schedule) else None


def _keep_run(run, capacity, skin) -> None:
    if run.use_graph and run.graph is not None:
        if len(_RUNS) > 4:
            _RUNS.clear()
        _RUNS[_run_key(run.n, run.interval, capacity, skin)] = run


def _reset_hooks(hooks) -> None:
    """Tell hooks that the run starts over (capacity retry)."""
    for hook in hooks:
        reset = getattr(hook, "reset", None)
        if callable(reset):
            reset()


def _drive(run: DeviceRespa, hooks, device_hooks=()) -> RunTrace:
    sysm, n_periods = run.system, run.schedule.num_iterations // run.interval
    trace = RunTrace()
    run.marks = [("drive", time.perf_counter())]
    run.start()

    def on_device(k):  # after sample point k (iteration k * interval)
        for hook in device_hooks:
            hook(k * run.interval, run.x)

    on_device(0)
    if hooks:
        # hooks see the host system at every sample point: sync per period
        _check(run, trace, upto=1)
        view = sysm.view() if hasattr(sysm, "view") else sysm
        run.download()
        run.update_container()
        trace.record_values(*_row_values(run, 0))
        for hook in hooks:
            hook(0, view, run.container)
        for k in range(n_periods):
            run.run_periods(k, 1)
            on_device(k + 1)
            _check(run, trace, upto=k + 2)
            run.download()
            run.update_container()
            trace.record_values(*_row_values(run, k + 1))
            for hook in hooks:
                hook((k + 1) * run.interval, view, run.container)
        for i in range(n_periods * run.interval, run.schedule.num_iterations):
            run._step(i)
        run.finish_scalars()
        _check(run, trace, upto=n_periods + 1)
        run.download()
        run.update_container()
        return trace
    mark = run.marks.append
    mark(("started", time.perf_counter()))
    if n_periods > 0 and run.use_graph and run.graph is not None:
        # a cached run (same shape): its captured period graph replays from
        # the first period on
        if device_hooks:
            for k in range(n_periods):
                run.run_periods(k, 1)
                on_device(k + 1)
        else:
            run.run_periods(0, n_periods)
        mark(("replays enqueued (cached graph)", time.perf_counter()))
    elif n_periods > 0 and run.use_graph:
        run.run_periods(0, 1)  # warm-up, also the first period of the run
        on_device(1)
        mark(("eager period", time.perf_counter()))
        run.capture()
        mark(("captured", time.perf_counter()))
        # the capture recorded but did not execute; rewind nothing: replay the rest
        run.eng.set_step(run.interval)
        if device_hooks:
            for k in range(1, n_periods):
                run.run_periods(k, 1)
                on_device(k + 1)
        else:
            run.run_periods(1, n_periods - 1)
        mark(("replays enqueued", time.perf_counter()))
    else:
        for k in range(n_periods):
            run.run_periods(k, 1)
            on_device(k + 1)
    for i in range(n_periods * run.interval, run.schedule.num_iterations):
        run._step(i)  # iterations past the last sample point
    run.finish_scalars()
    upto = n_periods + 1
    pin = run.collect(upto)  # the one synchronisation of the run
    mark(("collected (synced)", time.perf_counter()))
    word = int(pin["status"][0]) & 0xFFFFFFFFFFFFFFFF
    kind = word & 0xFF if word != _lib.RB_STATUS_CLEAR else None
    if int(pin["maxc"][0]) > run.eng.capacity or kind == _lib.RB_KIND_CAPACITY:
        raise CapacityError("neighbour row overflow")
    rows = pin["trace"][:upto].numpy()
    if kind is not None:  # as _check: the trace up to the failing step, the state
        tag = word >> 8
        _fill_trace(trace, rows[rows[:, 0] < tag] if tag > 0 else rows[:0], float(sysm.mass))
        run.apply_collected(pin)
        raise IntegrationBlowUp(int(tag), _MSG.get(kind, f"device error kind {kind}"), trace)
    _fill_trace(trace, rows, float(sysm.mass))
    run.apply_collected(pin)
    mark(("downloaded", time.perf_counter()))
    return trace


def _row_values(run: DeviceRespa, k: int):
    row = run.trace_dev[k].cpu().numpy()
    return int(round(row[0])), 0.5 * float(run.system.mass) * row[1], row[2], row[3], row[4], row[5]


def _check(run: DeviceRespa, trace: RunTrace, upto: int) -> None:
    """Raise IntegrationBlowUp / CapacityError for errors recorded so far."""
    if run.eng.overflowed():
        raise CapacityError("neighbour row overflow")
    err = run.eng.read_status()
    if err is None:
        return
    tag, kind = err
    rows = run.trace_rows(upto)
    keep = rows[rows[:, 0] < tag] if tag > 0 else rows[:0]
    if not len(trace):
        _fill_trace(trace, keep, float(run.system.mass))
    run.finish_scalars()
    run.download()
    run.update_container()
    raise IntegrationBlowUp(int(tag), _MSG.get(kind, f"device error kind {kind}"), trace)


def verlet_run(system, ff, container, dt: float, num_iterations: int,
               sample_interval: Optional[int] = None, hooks=()) -> RunTrace:
    """Velocity Verlet = r-RESPA with s = 1 (``integrators.py:176-191``)."""
    schedule = RespaSchedule(dt=dt, step_size_factor=1, num_iterations=num_iterations)
    return respa_run(system, ff, container, schedule, sample_interval, hooks)


@dataclass
class EquilibrationReport:
    """Outcome of an equilibration window (integrators.py:192-201)."""

    system: object
    rescale_factors: list
    tail_temperature: float
    target_temperature: float
    converged: bool


def measured_temperature(system) -> float:
    """Equipartition estimate T = (2/3) K / N (integrators.py:204-206)."""
    return 2.0 * system.kinetic_energy() / (3.0 * system.positions.shape[0])


def equilibrate(system, ff, container, dt: float, steps: int, target_temperature: float,
                rescale_interval: int = 10) -> EquilibrationReport:
    """Velocity-rescaling Verlet towards the target temperature
    (integrators.py:209-252), device-resident: the state stays in HBM, each
    window of `rescale_interval` steps is a replayed CUDA graph, and only the
    window's kinetic energy comes back to the host (one synchronisation per
    window) for the rescale factor sqrt(T_target / T_measured)."""
    if target_temperature <= 0:
        raise ValidationError("target temperature must be > 0")
    if steps < 0:
        raise ValidationError("steps must be >= 0")
    if not isinstance(container, (CudaLinkedCells, CudaDirectSum)):
        raise TypeError("equilibrate needs a CudaLinkedCells or CudaDirectSum container")
    x0 = np.array(system.positions, copy=True)
    v0 = np.array(system.velocities, copy=True)
    capacity = None
    for attempt in range(3):  # a row overflow repeats the run larger (as respa_run)
        try:
            return _equilibrate(system, ff, container, dt, steps, target_temperature,
                                rescale_interval, capacity)
        except CapacityError as exc:
            capacity = min(4096, _round_up(int(exc.args[1] * 1.5) + 32, 32)) \
                if len(exc.args) > 1 else None
            engine_for(system.positions.shape[0]).grow_cells()
            if x0 is not None:
                system.positions[:] = x0
                system.velocities[:] = v0
    raise CapacityError("neighbour rows kept overflowing")


def _equilibrate(system, ff, container, dt, steps, target_temperature, rescale_interval,
                 capacity) -> EquilibrationReport:
    factors, temperatures = [], []
    if steps > 0:
        interval = int(rescale_interval)
        run = DeviceRespa(system, ff, container, RespaSchedule(dt, 1, steps), interval,
                          capacity=capacity)
        run.start()
        n, m = system.positions.shape[0], float(system.mass)
        eng = run.eng
        done = 0
        try:
            while done < steps:
                chunk = min(interval, steps - done)
                if chunk == interval and run.use_graph and run.graph is not None:
                    run.graph.replay()
                else:
                    for i in range(done, done + chunk):
                        run._step(i)
                    if chunk == interval and run.use_graph and run.graph is None:
                        run.capture()  # the windows repeat (s = 1): one graph serves all
                done += chunk
                _check(run, RunTrace(), upto=(done + interval - 1) // interval + 1)
                eng.sum_f64(run.v, 0, square=True, n=3 * n)
                kinetic = 0.5 * m * float(eng.scalars[0].item())
                t_now = 2.0 * kinetic / (3.0 * n)
                temperatures.append(t_now)
                if t_now > 0:
                    factor = math.sqrt(target_temperature / t_now)
                    run.v.mul_(factor)
                    factors.append(factor)
        except CapacityError as exc:  # carry the capacity that overflowed
            raise CapacityError("neighbour row overflow", run.capacity) from exc
        run.finish_scalars()
        run.download()
        run.update_container()
    return _equilibrate_report(system, factors, temperatures, steps, target_temperature)


def _equilibrate_report(system, factors, temperatures, steps,
                        target_temperature) -> EquilibrationReport:
    tail = temperatures[-max(1, len(temperatures) // 10):] if temperatures else []
    tail_t = float(np.mean(tail)) if tail else measured_temperature(system)
    converged = steps == 0 or abs(tail_t - target_temperature) <= 0.02 * target_temperature
    return EquilibrationReport(system=system, rescale_factors=factors, tail_temperature=tail_t,
                               target_temperature=target_temperature, converged=converged)


__all__ = ["EquilibrationReport", "IntegrationBlowUp", "RespaSchedule", "RunTrace", "equilibrate",
           "measured_temperature", "respa_run", "verlet_run", "MinimumSeparationError"]
