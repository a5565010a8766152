"""Domain-decomposed r-RESPA over ranks (one process per GPU).

The loop of ``respamd/integrators.py:96-173`` on each rank's owned particles,
with the exchange of ``domain.py`` around the force passes:

    kick3 / drift / wrap (owned)               -- backend
    row-rebuild vote (any rank's particle moved > skin/2; all_reduce MAX)
    rebuild:  migrate + ghosts + local rows    -- domain.py + backend
    else:     refresh ghost positions          -- domain.py
    LJ on the local set, kick, [ATM every s-th step, kick3]
    samples: per-rank partial scalars summed in rank order; device errors
             (tagged with the device step counter) checked there

The force backend is the sm_100a engine (``GpuBackend``): the owned state
lives in device buffers and each step is drift kernel (publishing the owned
positions) -> vote (the one host synchronisation) -> halo refresh (one
peer-memory pull launch, or pack / NCCL / unpack) -> LJ [-> ATM] -> kick.  The CPU
tests plug in a numpy restatement and take the torch version of the same
loop.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .domain import PAYLOAD, Decomposition, Exchanger, allsum_in_rank_order, balanced_bounds, \
    balanced_layout, build_ghosts, cell_costs, cell_occupancy, migrate, refresh_ghosts
from .grid import geometry
from .integrators import IntegrationBlowUp, RespaSchedule, RunTrace
from .model import triplet_cutoff


class GpuBackend:
    """sm_100a passes and r-RESPA updates on one rank's particles."""

    def __init__(self, n_max: int, ff, r_build: float, halo: str = "peer"):
        from . import _lib
        from .engine import ForceEngine, _round_up

        if halo not in ("peer", "nccl"):
            raise ValueError(f"halo must be 'peer' or 'nccl', got {halo!r}")
        self.halo = halo
        self.n_max = int(n_max)
        self._pub = None  # IPC-shared published positions (2 x stride x 3, by step parity)
        self._graphs, self._fresh = {}, set()  # step kind -> graph executable (this epoch: fresh)
        self._opened = []
        self._lib = _lib
        self.eng = ForceEngine(n_max)
        self.torch = self.eng.torch
        self.device = self.eng.device
        self.ff = ff
        self.rc2 = float(ff.cutoff)
        self.rc3 = triplet_cutoff(ff)
        self.r_build = float(r_build)
        self._round_up = _round_up
        self.window = None
        self.n_own = 0
        self.n_local = 0
        z = lambda: self.torch.zeros((n_max, 3), dtype=self.torch.float64, device=self.device)  # noqa: E731
        self.f_local = z()
        # device-resident owned state (particle order, owned rows first): the
        # fused drift / kick kernels update it in place between rebuilds
        self.v, self.f2, self.f2_new, self.f3 = z(), z(), z(), z()
        self._zero2 = self.torch.zeros(2, dtype=self.torch.float64, device=self.device)
        self.eng.reset_status(0)

    def set_local(self, local, n_own: int, window, rebuild: bool) -> None:
        eng, torch = self.eng, self.torch
        n = int(local.shape[0])
        if rebuild:
            eng.set_count(n)
            self.window, self.n_own, self.n_local = window, int(n_own), n
            eng.pos[:n] = local
            eng.bin(window)
            eng.nlist(window, self.r_build, capacity=eng.capacity or None, checked=True)
            # owned flags only with ghosts present (a rank owning its whole
            # local set -- world 1 -- takes the undecomposed kernels, whose
            # triplet pass recovers the energy from the slot virial)
            eng.owned_rank = (eng.parts[:n] < n_own).to(torch.uint8) if n > n_own else None
        else:
            eng.pos[:n] = local
            eng.pos_r[:n][eng.rank_of[:n].long()] = eng.pos[:n]

    def pair(self, scalars: bool = True):
        eng = self.eng
        eng.lj(self.window, self.rc2, self.ff.epsilon, self.ff.sigma, self.f_local,
               tag=self._lib.RB_TAG_FROM_DEVICE, reduce=scalars)
        return self.f_local[: self.n_own].clone(), eng.scalars[1:3].clone()

    def triplet(self, scalars: bool = True):
        eng = self.eng
        if float(self.ff.nu) == 0.0:
            return (self.torch.zeros((self.n_own, 3), dtype=self.torch.float64, device=self.device),
                    self.torch.zeros(2, dtype=self.torch.float64, device=self.device))
        eng.atm(self.window, self.rc3, float(self.ff.nu), self.f_local,
                tag=self._lib.RB_TAG_FROM_DEVICE, count_visits=False, reduce=scalars)
        return self.f_local[: self.n_own].clone(), eng.scalars[3:5].clone()

    # ---- fused per-step primitives (the loop's fast path on the GPU) ----
    # ---- peer-memory halo (rb_halo_pull) ----
    def attach_peers(self, dist) -> None:
        """Allocate this rank's published-position buffer, swap CUDA IPC
        handles with every rank and map the peers' buffers (once)."""
        L, torch = self.eng.L, self.torch
        wire = torch.device("cpu") if dist.get_backend() == "gloo" else self.device
        # one parity stride for every rank: a reader offsets into the
        # writer's buffer
        stride = torch.tensor([self.n_max], dtype=torch.int64, device=wire)
        dist.all_reduce(stride, op=dist.ReduceOp.MAX)
        self._stride = int(stride.item())
        ptr = ctypes.c_void_p()
        self._lib.check(L.rb_ipc_alloc(2 * self._stride * 24, ctypes.byref(ptr)), "rb_ipc_alloc")
        self._pub = ptr.value
        handle = np.zeros(64, dtype=np.uint8)
        self._lib.check(L.rb_ipc_handle(self._pub, handle.ctypes.data), "rb_ipc_handle")
        mine = torch.from_numpy(handle).to(wire)
        every = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
        dist.all_gather(every, mine)
        bases = []
        for r, h in enumerate(every):
            if r == dist.get_rank():
                bases.append(self._pub)
                continue
            peer = ctypes.c_void_p()
            h = np.ascontiguousarray(h.cpu().numpy())
            self._lib.check(L.rb_ipc_open(h.ctypes.data, ctypes.byref(peer)), "rb_ipc_open")
            self._opened.append(peer.value)
            bases.append(peer.value)
        self._peers = torch.tensor(np.array(bases, dtype=np.uint64).view(np.int64),
                                   dtype=torch.int64, device=self.device)

    def close(self, dist=None) -> None:
        """Unmap the peers' buffers, then (after every rank did) free ours."""
        self.torch.cuda.synchronize(self.device)
        for p in self._opened:
            self.eng.L.rb_ipc_close(p)
        self._opened = []
        if self._pub is not None:
            if dist is not None:
                dist.barrier()
            self.eng.L.rb_ipc_free(self._pub)
            self._pub = None

    @property
    def peer(self) -> bool:
        return self._pub is not None

    def bind(self, st, plan) -> None:
        """After a rebuild: the owned state moves into the device buffers and
        `st` becomes views of them (positions are eng.pos[:n_own]); the
        ghost send lists become int32 device arrays for rb_halo_pack."""
        n = self.n_own
        for name, buf in (("v", self.v), ("f2", self.f2), ("f3", self.f3)):
            buf[:n] = getattr(st, name)
            setattr(st, name, buf[:n])
        st.x = self.eng.pos[:n]
        self.v[n:self.n_local].zero_()  # rb_sample sums v^2 over the local rows
        i32 = self.torch.int32
        self._lists = [(d, tm.to(i32), tp.to(i32), n_fp, n_fm)
                       for d, tm, tp, n_fp, n_fm in plan.stages]
        if self.peer:
            ghosts = plan.origin[n:]
            self._src_rank = ghosts[:, 0].to(i32).contiguous()
            self._src_index = ghosts[:, 1].to(i32).contiguous()

    def refresh_halo(self, dec, ex) -> None:
        """Per step between rebuilds: the owners' new positions into the ghost
        rows (and their rank-order copy), stage by stage (x -> y -> z): pack
        kernel, NCCL point-to-point, unpack kernel."""
        eng, L, ptr, torch = self.eng, self.eng.L, self._lib.ptr, self.torch
        if self.peer:
            # every rank's publishing drift of this step finished before the
            # rebuild vote this rank has passed: read the ghosts in place
            n = self.n_local - self.n_own
            self._lib.check(L.rb_halo_pull(n, ptr(self._src_rank), ptr(self._src_index),
                                           ptr(self._peers), self._stride, ptr(eng.status),
                                           self.n_own, ptr(eng.pos), ptr(eng.rank_of),
                                           ptr(eng.pos_r), eng.stream), "rb_halo_pull")
            return
        at = self.n_own
        for d, tm, tp, n_fp, n_fm in self._lists:
            send = []
            for idx in (tm, tp):
                buf = torch.empty((idx.shape[0], 3), dtype=torch.float64, device=self.device)
                self._lib.check(L.rb_halo_pack(idx.shape[0], ptr(idx), ptr(eng.pos), ptr(buf),
                                               eng.stream), "rb_halo_pack")
                send.append(buf)
            from_plus, from_minus = ex.exchange_fixed(send[0], send[1], dec.neighbor(d, -1),
                                                      dec.neighbor(d, +1), n_fp, n_fm)
            for buf, cnt in ((from_plus, n_fp), (from_minus, n_fm)):
                self._lib.check(L.rb_halo_unpack(cnt, ptr(buf.contiguous()), at, ptr(eng.pos),
                                                 ptr(eng.rank_of), ptr(eng.pos_r), eng.stream),
                                "rb_halo_unpack")
                at += cnt

    def local_view(self):
        return self.eng.pos[: self.n_local]

    def drift(self, box, dt, half_drift, half_respa, kick3: bool, skin: float):
        """kick3 / drift / wrap of the owned rows, their rank-order copy and
        the skin check (rb_respa_drift, opening the device step; `moved`
        reads the vote)."""
        eng, L = self.eng, self.eng.L
        ptr = self._lib.ptr
        args = (self.n_own, ptr(eng.pos), ptr(self.v), ptr(self.f2), ptr(self.f3),
                box.ctypes.data_as(ctypes.c_void_p), 1, dt, half_drift, half_respa, int(kick3),
                ptr(eng.rank_of), ptr(eng.pos_r), ptr(eng.x_ref), skin, ptr(eng.rebuild_flag),
                ptr(eng.status), self._lib.RB_TAG_FROM_DEVICE, 1)
        if self.peer:  # also publish the drifted owned rows for the peers' pulls
            st = L.rb_respa_drift_publish(*args, self._pub, self._stride, eng.stream)
        else:
            st = L.rb_respa_drift(*args, 0, eng.stream)
        self._lib.check(st, "rb_respa_drift")

    def moved(self):
        """This rank's rebuild vote for the drifted step (0-d device tensor)."""
        return self.eng.rebuild_flag[0] == self.eng.status[1]

    # ---- device trace and captured steps ----
    def trace_setup(self, rows: int, interval: int) -> None:
        """Device trace rows [tag, sum v^2, E2, W2, E3, W3, 0, 0] of this
        rank's partial sums, written by `sample` (rb_sample)."""
        self.trace = self.torch.zeros((rows, 8), dtype=self.torch.float64, device=self.device)
        self.interval = int(interval)

    def sample(self) -> None:
        """Trace row of the current device step (owned velocities; velocity
        rows past the owned ones are kept zero by bind)."""
        self.eng.sample(self.v, self.trace, self.interval)

    def step_body(self, end_of_cycle: bool, sample: bool, pull: bool, drift_next, kick_args):
        """Step i after its drift and vote: [ghost pull] -> LJ -> [ATM] ->
        kick -> [trace row] -> [drift of step i + 1]; `drift_next` = None or
        the drift arguments.  Launch-only: capturable."""
        if pull:
            self.refresh_halo(None, None)
        self.pair_into_new(False)
        if end_of_cycle:
            self.triplet_into_f3(False)
        self.kick(*kick_args, end_of_cycle)
        if sample:
            self.sample()
        if drift_next is not None:
            self.drift(*drift_next)

    def invalidate_graphs(self) -> None:
        """A rebuild changed counts and lists: every step kind is recaptured
        at its next use (into its existing executable: rb_graph_end updates)."""
        self._fresh = set()

    def replay(self, key, body) -> None:
        """Launch the captured graph of a step kind of the current row epoch
        (captured on first use in the epoch)."""
        torch, L = self.torch, self.eng.L
        cur = torch.cuda.current_stream()
        if key not in self._fresh:
            side = self._side = getattr(self, "_side", None) or torch.cuda.Stream()
            side.wait_stream(cur)
            h = ctypes.c_void_p(side.cuda_stream)
            exe = ctypes.c_uint64(self._graphs.get(key, 0))
            with torch.cuda.stream(side):
                self._lib.check(L.rb_graph_begin(h), "rb_graph_begin")
                try:
                    body()
                finally:
                    st = L.rb_graph_end(h, ctypes.byref(exe))
                self._lib.check(st, "rb_graph_end")
            cur.wait_stream(side)
            self._graphs[key] = exe.value
            self._fresh.add(key)
        self._lib.check(L.rb_graph_launch(self._graphs[key], ctypes.c_void_p(cur.cuda_stream)),
                        "rb_graph_launch")

    def destroy_graphs(self) -> None:
        for exe in self._graphs.values():
            self.eng.L.rb_graph_destroy(exe)
        self._graphs, self._fresh = {}, set()

    def pair_into_new(self, scalars: bool):
        eng = self.eng
        eng.lj(self.window, self.rc2, self.ff.epsilon, self.ff.sigma, self.f2_new,
               tag=self._lib.RB_TAG_FROM_DEVICE, reduce=scalars)
        return eng.scalars[1:3]

    def triplet_into_f3(self, scalars: bool):
        eng = self.eng
        if float(self.ff.nu) == 0.0:
            self.f3.zero_()
            return self._zero2
        eng.atm(self.window, self.rc3, float(self.ff.nu), self.f3,
                tag=self._lib.RB_TAG_FROM_DEVICE, count_visits=False, reduce=scalars)
        return eng.scalars[3:5]

    def kick(self, half_dt, half_respa, kick3: bool) -> None:
        """v += half_dt (f2_old + f2_new), f2_old := f2_new [, v += half_respa f3]."""
        eng, L = self.eng, self.eng.L
        ptr = self._lib.ptr
        st = L.rb_respa_kick(self.n_own, ptr(self.v), ptr(self.f2), ptr(self.f2_new), ptr(self.f3),
                             half_dt, half_respa, int(kick3), ptr(eng.status),
                             self._lib.RB_TAG_FROM_DEVICE, eng.stream)
        self._lib.check(st, "rb_respa_kick")

    def check(self):
        """(iteration, reason) of the first recorded device error, or None."""
        err = self.eng.read_status()
        if err is None:
            return None
        reason = {1: "particles closer than the minimum separation guard",
                  2: "particles closer than the minimum separation guard",
                  3: "non-finite position or velocity"}.get(err[1], f"device error kind {err[1]}")
        return int(err[0]), reason


# speculative-window bookkeeping of this process (tests, probes)
WINDOW_STATS = {"runs": 0, "resumes": 0, "rebuild_s": 0.0}


@dataclass
class DomainState:
    ids: object  # (n_own,) float64 global ids
    x: object
    v: object
    f2: object
    f3: object
    x_ref: object


def _numpy_like_update(torch, a, scale, b):
    """a + scale*b with numpy's rounding (two roundings)."""
    return a + (scale * b)


def domain_respa_run(dist, system, ff, schedule: RespaSchedule, backend_factory, skin: float = 0.3,
                     sample_interval: Optional[int] = None, dims=None, device=None,
                     on_step=None, balance: bool = False):
    """Run r-RESPA decomposed over dist.get_world_size() ranks.

    Every rank passes the same full initial `system` (host arrays); on return
    every rank's `system` holds the final state (gathered by particle id) and
    the same RunTrace.  `on_step(i)` (optional) is called on the host before
    step i and once more with i = num_iterations after the last step (the
    bench records its CUDA events there).  `balance` cuts the blocks by the
    estimated work of the initial configuration (domain.balanced_layout: for
    inhomogeneous systems such as the cfg5 slab) instead of evenly."""
    import torch

    world, rank = dist.get_world_size(), dist.get_rank()
    s = schedule.step_size_factor
    interval = s if sample_interval is None else int(sample_interval)
    rc2, rc3 = float(ff.cutoff), triplet_cutoff(ff)
    r_list = max(rc2, rc3) if float(ff.nu) != 0.0 else rc2
    box = np.asarray(system.box, dtype=np.float64)
    skin = max(0.0, min(float(skin), float(box.min()) / 2.0 - r_list))
    r_build = r_list + skin
    bounds = None
    if balance:
        geom = geometry(box, None, r_build, True)
        occ = cell_occupancy(system.positions, geom)
        costs = cell_costs(system.positions, geom, 0.29 / s if float(ff.nu) != 0.0 else 0.0)
        if dims is None:
            dims, bounds = balanced_layout(costs, world, occ)
        else:
            bounds = [balanced_bounds(costs.sum(axis=tuple(a for a in range(3) if a != d)),
                                      int(dims[d])) for d in range(3)]
    dec = Decomposition(box, r_build, world, rank, dims, bounds)
    n_total = system.positions.shape[0]
    # the whole initial state once to the device; ownership and the window
    # population from device cell maps (domain.cells_of_t)
    dev0 = torch.device(device) if device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
        else torch.device("cpu"))
    pos_all = torch.as_tensor(np.ascontiguousarray(system.positions, dtype=np.float64),
                              device=dev0)
    dec.local_estimate = dec.window_count_t(pos_all)
    backend = backend_factory(dec, n_total, r_build)
    dev = backend.device if device is None else device
    ex = Exchanger(dist, dev)
    m = float(system.mass)
    dt = schedule.dt
    half_dt, half_drift, half_respa = 0.5 * dt / m, 0.5 * dt * dt / m, 0.5 * dt * s / m
    box_t = torch.as_tensor(box, device=dev)

    pos_all = pos_all.to(dev)
    mine = torch.nonzero(dec.owner_rank_t(pos_all) == rank).reshape(-1)
    vel_all = torch.as_tensor(np.ascontiguousarray(system.velocities, dtype=np.float64),
                              device=dev)
    st = DomainState(ids=mine.to(torch.float64), x=pos_all[mine].contiguous(),
                     v=vel_all[mine].contiguous(), f2=None, f3=None, x_ref=None)
    del pos_all, vel_all
    window = dec.window()
    trace = RunTrace()

    # GPU backends run the per-step updates as fused kernels on device-resident
    # state (one host synchronisation per step: the rebuild vote); other
    # backends (the numpy one of the CPU tests) take the torch restatement
    fast = hasattr(backend, "bind")
    peer = fast and world > 1 and getattr(backend, "halo", None) == "peer"
    if peer:
        backend.attach_peers(dist)

    split = any(dec.split(d) for d in range(3))

    def rebuild():
        nonlocal window
        if st.f2 is None:
            st.f2 = torch.zeros_like(st.x)
            st.f3 = torch.zeros_like(st.x)
        elif split:  # (one block: nothing can move)
            payload = torch.cat([st.ids[:, None], st.x, st.v, st.f2, st.f3], dim=1)
            payload = migrate(dec, ex, payload)
            st.ids, st.x, st.v = payload[:, 0], payload[:, 1:4], payload[:, 4:7]
            st.f2, st.f3 = payload[:, 7:10].contiguous(), payload[:, 10:13].contiguous()
            st.x, st.v = st.x.contiguous(), st.v.contiguous()
        origin = None
        if peer:
            n_own = int(st.x.shape[0])
            origin = torch.stack([torch.full((n_own,), float(rank), dtype=torch.float64,
                                             device=st.x.device),
                                  torch.arange(n_own, dtype=torch.float64, device=st.x.device)],
                                 dim=1)
        local, plan = build_ghosts(dec, ex, st.x, origin)
        backend.set_local(local, plan.n_owned, window, rebuild=True)
        if fast:
            backend.bind(st, plan)
            return backend.local_view(), plan
        st.x_ref = st.x.clone()
        return local, plan

    def refresh(plan, local):
        local[: plan.n_owned] = st.x
        refresh_ghosts(dec, ex, plan, local)
        backend.set_local(local, plan.n_owned, window, rebuild=False)

    def scalars(e2w2, e3w3):
        kin = float((st.v * st.v).sum().item())
        return allsum_in_rank_order(dist, [kin, float(e2w2[0]), float(e2w2[1]), float(e3w3[0]),
                                           float(e3w3[1])], dev)

    def record(it, e2w2, e3w3):
        tot = scalars(e2w2, e3w3)
        trace.record_values(it, 0.5 * m * tot[0], tot[1], tot[2], tot[3], tot[4])

    wire = torch.device("cpu") if dist.get_backend() == "gloo" else dev

    def any_flag(flag) -> bool:
        """Global OR of a per-rank flag (python bool or 0-d device tensor):
        one all_reduce and the step's single host synchronisation."""
        if world == 1:
            return bool(flag)
        t = torch.as_tensor(flag, dtype=torch.int64).reshape(1).to(wire)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return bool(t.item())

    # errors are checked at sample points (as the single-GPU loop does at the
    # end): the first non-finite step is kept on the device meanwhile
    first_bad = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)

    never = np.iinfo(np.int64).max

    def check(upto: int) -> None:
        """Raise IntegrationBlowUp at the first failing iteration of any rank
        (integrators.py:154-170), checked at sample points."""
        err = backend.check()
        mine = torch.stack([first_bad.to(wire)[0],
                            torch.tensor(never if err is None else err[0], dtype=torch.int64,
                                         device=wire)])
        both = mine.clone()
        dist.all_reduce(both, op=dist.ReduceOp.MIN)
        it = int(both.min().item())
        if it <= upto:
            if err is not None and err[0] == it:
                reason = err[1]
            elif int(mine[0].item()) == it:
                reason = "non-finite position or velocity"
            else:
                reason = "error on another rank"
            raise IntegrationBlowUp(it, reason, trace)

    def first_error():
        """(iteration, reason) of the earliest device error over all ranks
        (collective; iteration = never when there is none)."""
        err = backend.check()
        t = torch.tensor([never if err is None else err[0]], dtype=torch.int64, device=wire)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        it = int(t.item())
        reason = err[1] if err is not None and err[0] == it else "error on another rank"
        return it, reason

    # Speculative windows: the rebuild vote of each step is a
    # device flag reduced over the ranks (one NCCL all_reduce enqueued from
    # the host, none at world 1) that freezes the rest of the window on the
    # device (RB_KIND_REBUILD); the host synchronises once per window, then
    # rebuilds and resumes the frozen step.  The all_reduce also orders the
    # peers' publishing drifts before every rank's ghost pull.  Message
    # halos and gloo keep the per-step host vote.
    wlen = int(os.environ.get("RB_DOMAIN_WINDOW", "16"))
    # (RB_DOMAIN_WINDOW_ANY=1: also over gloo, whose all_reduce of a CUDA
    # tensor synchronises the stream -- slower, the same protocol; tests run
    # ranks sharing one GPU that way)
    windowed = (fast and wlen > 1 and skin > 0.0 and
                (world == 1 or (peer and (dist.get_backend() == "nccl" or
                                          os.environ.get("RB_DOMAIN_WINDOW_ANY") == "1"))))

    def run_windows(num, drift_args, kick_args):
        WINDOW_STATS["runs"] += 1
        L, eng, lib = backend.eng.L, backend.eng, backend._lib
        ptr = lib.ptr
        vflag = torch.zeros(1, dtype=torch.int64, device=dev)
        head = np.zeros(2, dtype=np.uint64)
        i = 0
        while i < num:
            j = min(num, i + wlen)
            for k in range(i, j):
                if k > i and on_step is not None:
                    on_step(k)
                # the vote of step k (its drift ran at the end of step k-1)
                lib.check(L.rb_vote_flag(ptr(eng.rebuild_flag), ptr(eng.status), ptr(vflag),
                                         eng.stream), "rb_vote_flag")
                if world > 1:
                    dist.all_reduce(vflag, op=dist.ReduceOp.MAX)
                lib.check(L.rb_vote_freeze(ptr(vflag), ptr(eng.status), eng.stream),
                          "rb_vote_freeze")
                sample = (k + 1) % interval == 0
                end_of_cycle = (k + 1) % s == 0
                nxt = drift_args(k + 1) if k + 1 < num else None
                backend.replay((end_of_cycle, sample, peer, nxt is not None),
                               lambda: backend.step_body(end_of_cycle, sample, peer, nxt,
                                                         kick_args))
            head[:] = eng.status[:2].cpu().numpy().view(np.uint64)  # the window's sync
            word = int(head[0])
            # one decision for every rank: an error (key 2 tag) before a
            # rebuild request (2 tag + 1) of the same step, nothing: never
            key = never if word == lib.RB_STATUS_CLEAR else \
                2 * (word >> 8) + (1 if (word & 0xFF) == lib.RB_KIND_REBUILD else 0)
            if world > 1:
                t = torch.tensor([key], dtype=torch.int64, device=wire)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                key = int(t.item())
            if key == never:
                i = j
                if i < num and on_step is not None:
                    on_step(i)
                continue
            if key % 2 == 0:
                return  # a device error: reported by the caller (first_error)
            # a rank flagged step k = tag - 1: every rank froze there; the
            # rows are rebuilt after its drift, then the step runs eagerly
            k = key // 2 - 1
            WINDOW_STATS["resumes"] += 1
            eng.status[0:1].fill_(-1)  # RB_STATUS_CLEAR
            t_rb = time.perf_counter()
            rebuild()
            WINDOW_STATS["rebuild_s"] += time.perf_counter() - t_rb
            backend.invalidate_graphs()
            nxt = drift_args(k + 1) if k + 1 < num else None
            if on_step is not None and k > i:
                on_step(k)
            backend.step_body((k + 1) % s == 0, (k + 1) % interval == 0, False, nxt, kick_args)
            i = k + 1
            if i < num and on_step is not None:
                on_step(i)

    def run_device_loop():
        """GPU backends: device-resident state, one host synchronisation per
        step (the rebuild vote).  Between rebuilds each step after its vote
        is one replayed CUDA graph: [ghost pull] -> LJ -> [ATM] -> kick ->
        [trace row] -> drift of the next step (publishing its positions);
        the graphs are captured per row epoch (pointers and counts change
        only at rebuilds).  Trace rows stay on the device until the end;
        device errors are read at rebuilds (before migrating) and at the end."""
        num = schedule.num_iterations
        rows = num // interval + 1
        backend.trace_setup(rows, interval)
        backend.pair_into_new(False)
        st.f2.copy_(backend.f2_new[: backend.n_own])
        backend.triplet_into_f3(False)
        backend.sample()
        kick_args = (half_dt, half_respa)

        def drift_args(j):
            return (box, dt, half_drift, half_respa, j % s == 0, skin)

        if on_step is not None:
            on_step(0)
        if num > 0:
            backend.drift(*drift_args(0))
        if windowed:
            run_windows(num, drift_args, kick_args)
            num_done = num
        else:
            num_done = 0
        for i in range(num_done, num):
            if i > 0 and on_step is not None:
                on_step(i)
            sample = (i + 1) % interval == 0
            end_of_cycle = (i + 1) % s == 0
            nxt = drift_args(i + 1) if i + 1 < num else None
            if any_flag(backend.moved() if skin > 0.0 else True):
                if first_error()[0] <= i + 1:
                    break  # never migrate a broken state; reported below
                rebuild()
                backend.invalidate_graphs()
                backend.step_body(end_of_cycle, sample, False, nxt, kick_args)
            else:
                if not peer:
                    backend.refresh_halo(dec, ex)  # messages: outside the graph
                backend.replay((end_of_cycle, sample, peer, nxt is not None),
                               lambda: backend.step_body(end_of_cycle, sample, peer, nxt,
                                                         kick_args))
        if on_step is not None:
            on_step(num)
        backend.destroy_graphs()
        it, reason = first_error()
        # per-rank partial rows summed in rank order (row k: iteration k * interval)
        mine = backend.trace.to(wire)
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        acc = np.zeros(tuple(mine.shape))
        for part in parts:
            acc = acc + part.cpu().numpy()
        for k in range(rows):
            if k * interval >= it:
                break
            trace.record_values(k * interval, 0.5 * m * acc[k, 1], acc[k, 2], acc[k, 3],
                                acc[k, 4], acc[k, 5])
        if it <= num:
            raise IntegrationBlowUp(it, reason, trace)

    clean = False
    try:
        local, plan = rebuild()
        if fast:
            run_device_loop()
        else:
            f2, e2w2 = backend.pair()
            f3, e3w3 = backend.triplet()
            st.f2, st.f3 = f2, f3
            check(0)
            record(0, e2w2, e3w3)
            half_skin2 = (0.5 * skin) ** 2 * (1.0 - 1e-9)
            for i in range(schedule.num_iterations):
                if on_step is not None:
                    on_step(i)
                sample = (i + 1) % interval == 0
                end_of_cycle = (i + 1) % s == 0
                if hasattr(backend, "advance"):
                    backend.advance()
                if i % s == 0:
                    st.v = _numpy_like_update(torch, st.v, half_respa, st.f3)
                st.x = st.x + ((dt * st.v) + (half_drift * st.f2))
                st.x = torch.remainder(st.x, box_t)  # numpy mod semantics for box > 0
                st.x = torch.where(st.x >= box_t, torch.zeros_like(st.x), st.x)
                if skin == 0.0 or st.x.shape[0] == 0:
                    moved = skin == 0.0
                else:
                    d = st.x - st.x_ref
                    d = d - box_t * torch.where(d > 0.5 * box_t, 1.0, torch.where(d < -0.5 * box_t, -1.0, 0.0))
                    moved = ((d * d).sum(dim=1).max() > half_skin2)
                if any_flag(moved):
                    local, plan = rebuild()
                else:
                    refresh(plan, local)
                f2_new, e2w2 = backend.pair(scalars=sample)
                st.v = st.v + (half_dt * (st.f2 + f2_new))
                st.f2 = f2_new
                if (i + 1) % s == 0:
                    st.f3, e3w3 = backend.triplet(scalars=sample)
                    st.v = _numpy_like_update(torch, st.v, half_respa, st.f3)
                finite = torch.isfinite(st.x).all() & torch.isfinite(st.v).all()
                first_bad = torch.where(finite | (first_bad <= i), first_bad,
                                        torch.full_like(first_bad, i + 1))
                if sample:
                    check(i + 1)
                    record(i + 1, e2w2, e3w3)
            if on_step is not None:
                on_step(schedule.num_iterations)
            check(schedule.num_iterations)
        clean = True
    except IntegrationBlowUp:
        clean = True
        raise
    finally:
        if peer:
            # collective only when every rank got here (blow-ups are raised
            # by the collective check, so they count as clean)
            backend.close(dist if clean else None)

    # gather the owned state of every rank into the host system (by id): one
    # tensor all_gather of the padded payloads (id -1 pads), placed by id on
    # the device, then one copy per array to the host
    payload = torch.cat([st.ids[:, None], st.x, st.v, st.f2, st.f3], dim=1)
    cnt = torch.tensor([payload.shape[0]], dtype=torch.int64, device=wire)
    dist.all_reduce(cnt, op=dist.ReduceOp.MAX)
    padded = torch.full((int(cnt.item()), payload.shape[1]), -1.0, dtype=torch.float64,
                        device=payload.device)
    padded[: payload.shape[0]] = payload
    padded = padded.to(wire)
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded)
    allp = torch.cat(parts, dim=0).to(dev)
    allp = allp[allp[:, 0] >= 0.0]
    ids = allp[:, 0].to(torch.int64)
    seen = torch.zeros(n_total, dtype=torch.int64, device=dev)
    seen.index_add_(0, ids.clamp(0, n_total - 1), torch.ones_like(ids))
    if ids.shape[0] != n_total or not bool(torch.all(seen == 1)):
        raise RuntimeError("particles lost or duplicated by the decomposition")
    out = torch.empty((n_total, payload.shape[1] - 1), dtype=torch.float64, device=dev)
    out[ids] = allp[:, 1:]
    out = out.cpu()
    from .integrators import _host_copy

    _host_copy(system.positions, out[:, 0:3].contiguous())
    _host_copy(system.velocities, out[:, 3:6].contiguous())
    _host_copy(system.forces_2b, out[:, 6:9].contiguous())
    _host_copy(system.forces_3b, out[:, 9:12].contiguous())
    return trace


def gpu_backend_factory(ff, headroom: float = 1.6, halo: Optional[str] = None):
    """Backend factory for domain_respa_run on the local CUDA device.

    `halo`: "peer" (default; env RB_HALO) refreshes ghosts from the owners'
    published positions over CUDA IPC peer memory, "nccl" with pack /
    point-to-point / unpack.  Buffers are sized from the rank's initial
    window population (`dec.local_estimate`, set by domain_respa_run)."""
    import os

    mode = halo or os.environ.get("RB_HALO", "peer")

    def make(dec: Decomposition, n_total: int, r_build: float):
        est = getattr(dec, "local_estimate", None)
        if est is None:
            est = n_total / dec.world * _ghost_factor(dec, r_build)
        n_max = int(headroom * est) + 1024
        return GpuBackend(min(n_max, n_total * 2 + 1024), ff, r_build, halo=mode)

    return make


def _ghost_factor(dec: Decomposition, r_build: float) -> float:
    cells = np.asarray(dec.geom.cells, dtype=np.float64)
    f = 1.0
    for d in range(3):
        if dec.split(d):
            blk = cells[d] / dec.dims[d]
            f *= (blk + 2.0) / blk
    return f


__all__ = ["GpuBackend", "domain_respa_run", "gpu_backend_factory", "PAYLOAD"]
