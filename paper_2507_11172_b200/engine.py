"""Device workspace and pass sequencing for the sm_100a kernels.

``ForceEngine`` owns the device buffers of one particle count (torch CUDA
tensors used as plain memory) and issues the C-ABI passes on the current
torch stream:

    bin (counting sort, containers.py:175-209)
      -> nlist + mirror (rank-sorted survivor rows, :437-474)
      -> lj   (pair pass, :282-370)           -> deterministic sums
      -> atm  (Newton-3 triplet pass, :373-535) -> deterministic sums

Every buffer lives in HBM for the whole run; nothing is reallocated per
step.  State stays in the reference's (n,3) AoS particle order; the binning
gathers a rank-ordered copy ``pos_r`` that the force kernels read, and they
write forces straight back into particle order.

Inside a device-resident run the rows are Verlet rows built at rc + skin: the
rebuild kernels are launched every step but gated on ``rebuild_flag`` (set
by the drift kernel of that step when a particle moved more than skin/2).
"""

from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ptr
from .grid import Geometry, rb_grid

SCALAR_SUMSQ, SCALAR_E2, SCALAR_W2, SCALAR_E3, SCALAR_W3 = 0, 1, 2, 3, 4
_NULL = ctypes.c_void_p(0)


def _round_up(x: int, m: int) -> int:
    return int((x + m - 1) // m * m)


class CapacityError(RuntimeError):
    """A neighbour row outgrew its capacity inside a device-resident run."""


class ForceEngine:
    """Device buffers + pass launches for `n` particles."""

    def __init__(self, n: int, device: Optional[int] = None):
        torch = _lib.require_device()
        self.torch = torch
        self.L = _lib.lib()
        self.n = int(n)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        dev, f64, i32, i64 = self.device, torch.float64, torch.int32, torch.int64
        n = max(self.n, 1)
        self.pos = torch.zeros((n, 3), dtype=f64, device=dev)
        self.pos_r = torch.zeros((n, 3), dtype=f64, device=dev)  # rank order
        self.x_ref = torch.zeros((n, 3), dtype=f64, device=dev)  # positions at the last build
        self.parts = torch.zeros(n, dtype=i32, device=dev)  # rank -> particle
        self.rank_of = torch.zeros(n, dtype=i32, device=dev)  # particle -> rank
        self.cell_of_rank = torch.zeros(n, dtype=i32, device=dev)
        self.e2_rank = torch.zeros(n, dtype=f64, device=dev)
        self.w2_rank = torch.zeros(n, dtype=f64, device=dev)
        self.e3_rank = torch.zeros(n, dtype=f64, device=dev)
        self.w3_rank = torch.zeros(n, dtype=f64, device=dev)
        self.v_rank = torch.zeros(n, dtype=i32, device=dev)
        self.row_count = torch.zeros(n, dtype=i32, device=dev)
        self.max_count = torch.zeros(1, dtype=i32, device=dev)
        # status[0]: error word (all ones = clear); status[1]: current device
        # step; status[2]: last closed step (the kick); status[3]: rebuild
        # steps flagged by drifts (include/respa_b200.h)
        self.status = torch.tensor([-1, 0, 0, 0], dtype=i64, device=dev)
        self.rebuild_flag = torch.zeros(1, dtype=i64, device=dev)
        self.scalars = torch.zeros(8, dtype=f64, device=dev)
        self.visits = torch.zeros(1, dtype=i64, device=dev)
        self.red_scratch = torch.empty(
            max(1, int(self.L.rb_reduce_scratch_bytes(n * 3)) // 8), dtype=f64, device=dev)
        self.sample_scratch = torch.zeros(  # zero-filled once (rb_sample contract)
            (int(self.L.rb_sample_scratch_bytes(n)) + 7) // 8, dtype=f64, device=dev)
        self.cell_start = None
        self.bin_scratch = None
        self.rebuild_scratch = None
        self.rows = None
        self.mirror = None
        self.dir_scratch = None  # mirror directory of the staged rows (uint16 [n][32])
        self.atm_scratch = None
        self.capacity = 0
        self.slots = 0  # shared-memory slots of the triplet pass (longest row)
        self.owned_rank = None  # uint8 per rank in decomposed runs
        self._geom_key = None
        self._grid = None
        self._stream_override = None  # capture of a conditional body
        self.cond_body_launches = 0  # kernels in the last conditional rebuild body
        self.direct_scratch = None
        self.busy = False  # held by a device-resident run (containers.engine_for)
        # cell-based triplet pass (rb_atm_pass_cells): scratch, staged
        # neighbourhood capacity (measured, with margin) and its margin
        self.cells_scratch = None
        self.nb_cap = 0
        self.nb_margin = 1.1
        self._cells_ok = {}
        self._cells_slots = 0
        self.slots_margin = 1.0
        self._nb_max = torch.zeros(1, dtype=i32, device=dev)

    # ------------------------------------------------------------------ misc
    @property
    def stream(self):
        if self._stream_override is not None:
            return self._stream_override
        return _lib.stream_handle()

    def rebuild_cond(self) -> int:
        """Conditional handle for the rebuild of the step being captured
        (0 when the stream is not capturing)."""
        h = ctypes.c_uint64(0)
        st = self.L.rb_rebuild_cond_create(self.stream, ctypes.byref(h))
        if st == _lib.RB_NOT_CAPTURING:
            return 0
        _lib.check(st, "rb_rebuild_cond_create")
        return int(h.value)

    def rebuild(self, geom: Geometry, r_list: float, capacity: int, pos=None, tag: int = 0,
                cond: int = 0, fused: bool = False) -> None:
        """Gated rebuild (binning, rows, mirror) of the device loop.

        `fused`: one rb_rebuild launch (the same phases behind grid barriers;
        exits at once when the step did not flag a rebuild).  With a
        conditional handle (captured step, set by the drift) the nine gated
        launches go into the body of an IF node, so steps that do not rebuild
        skip them; otherwise they are launched directly."""
        if fused:
            pos = self.pos if pos is None else pos
            self._ensure_cells(geom.num_cells)
            self._ensure_rows(capacity)
            need = int(self.L.rb_rebuild_scratch_bytes(self.n, geom.num_cells))
            if self.rebuild_scratch is None or self.rebuild_scratch.numel() < need:
                # zero-filled once: the grid-barrier words at its head
                self.rebuild_scratch = self.torch.zeros(need, dtype=self.torch.uint8,
                                                        device=self.device)
            g = self.grid_struct(geom)
            st = self.L.rb_rebuild(ctypes.byref(g), self.n, ptr(pos), ptr(self.cell_start),
                                   ptr(self.parts), ptr(self.cell_of_rank), ptr(self.pos_r),
                                   ptr(self.rank_of), ptr(self.x_ref), float(r_list),
                                   int(self.capacity), ptr(self.rows), ptr(self.row_count),
                                   ptr(self.max_count), ptr(self.mirror), self._gate(True),
                                   ptr(self.status), int(tag), ptr(self.rebuild_scratch),
                                   self.rebuild_scratch.numel(), self.stream)
            _lib.check(st, "rb_rebuild")
            return
        if cond:
            body = ctypes.c_void_p()
            _lib.check(self.L.rb_rebuild_cond_begin(cond, self.stream, ctypes.byref(body)),
                       "rb_rebuild_cond_begin")
            parent = self.stream
            self._stream_override = body
            l0 = self.L.rb_launch_count()
            try:
                self.bin(geom, pos, gated=True, tag=tag)
                self.nlist(geom, r_list, capacity=capacity, checked=False, gated=True, tag=tag)
            finally:
                self._stream_override = None
                self.cond_body_launches = self.L.rb_launch_count() - l0
                _lib.check(self.L.rb_rebuild_cond_end(parent), "rb_rebuild_cond_end")
            return
        self.bin(geom, pos, gated=True, tag=tag)
        self.nlist(geom, r_list, capacity=capacity, checked=False, gated=True, tag=tag)

    def grid_struct(self, geom):
        if geom != self._geom_key:
            self._grid = geom.to_rb_grid() if hasattr(geom, "to_rb_grid") else rb_grid(geom)
            self._geom_key = geom
        return self._grid

    def set_count(self, n: int) -> None:
        """Use the first `n` particles of the buffers (decomposed runs,
        where the local count changes at every row rebuild)."""
        if n > self.pos.shape[0]:
            raise ValueError(f"{n} local particles exceed the engine's {self.pos.shape[0]}")
        self.n = int(n)

    def reset_status(self, step: int = 0) -> None:
        self.status[0:1].fill_(-1)  # (fill kernels: capturable)
        self.status[3:].zero_()
        self.set_step(step)

    def set_step(self, step: int) -> None:
        """Device step counter: step `step` current and closed (the next
        step-opening drift numbers its step step + 1)."""
        self.status[1:3].fill_(int(step))

    def read_status(self):
        """(tag, kind) of the first recorded device error, or None (syncs)."""
        word = int(self.status[0].item()) & 0xFFFFFFFFFFFFFFFF
        if word == _lib.RB_STATUS_CLEAR:
            return None
        return word >> 8, word & 0xFF

    def upload_positions(self, positions: np.ndarray) -> None:
        src = np.ascontiguousarray(positions, dtype=np.float64)
        self.pos.copy_(self.torch.from_numpy(src), non_blocking=False)

    def _gate(self, gated: bool):
        return ptr(self.rebuild_flag) if gated else _NULL

    def _owned(self):
        # rank-indexed owned flags of a decomposed (domain) run; NULL otherwise
        return ptr(self.owned_rank) if self.owned_rank is not None else _NULL

    # --------------------------------------------------------------- binning
    def _ensure_cells(self, ncell: int) -> None:
        torch = self.torch
        if self.cell_start is None or self.cell_start.numel() < ncell + 1:
            self.cell_start = torch.zeros(ncell + 1, dtype=torch.int32, device=self.device)
        need = int(self.L.rb_bin_scratch_bytes(self.n, ncell))
        if self.bin_scratch is None or self.bin_scratch.numel() < need:
            self.bin_scratch = torch.empty(need, dtype=torch.uint8, device=self.device)

    def bin(self, geom: Geometry, pos=None, gated: bool = False, tag: int = 0) -> None:
        pos = self.pos if pos is None else pos
        self._ensure_cells(geom.num_cells)
        g = self.grid_struct(geom)
        st = self.L.rb_bin(ctypes.byref(g), self.n, ptr(pos), ptr(self.cell_start), ptr(self.parts),
                           ptr(self.cell_of_rank), ptr(self.pos_r), ptr(self.rank_of),
                           ptr(self.x_ref), self._gate(gated), ptr(self.status), int(tag),
                           ptr(self.bin_scratch), self.bin_scratch.numel(), self.stream)
        _lib.check(st, "rb_bin")

    # ------------------------------------------------------- neighbour rows
    def estimate_capacity(self, geom: Geometry, r_list: float) -> int:
        """Row capacity from the densest cell of the current binning (syncs)."""
        counts = self.cell_start[1:geom.num_cells + 1] - self.cell_start[:geom.num_cells]
        max_occ = int(counts.max().item()) if geom.num_cells else 1
        vol = float(np.prod(geom.cell_size))
        dens = max(max_occ / vol, self.n / float(np.prod(geom.box)))
        est = dens * 4.0 / 3.0 * math.pi * r_list ** 3
        cap = max(32, _round_up(int(1.3 * est) + 32, 32))
        return int(min(4096, cap, max(32, _round_up(self.n, 32))))

    def _ensure_rows(self, capacity: int) -> None:
        # sized for the whole particle buffer, not the current count: a
        # decomposed run changes n at every rebuild (set_count)
        if self.rows is None or self.capacity != capacity:
            torch = self.torch
            n_buf = max(int(self.pos.shape[0]), 1)
            self.rows = torch.zeros(n_buf * capacity, dtype=torch.int32, device=self.device)
            self.mirror = torch.zeros(n_buf * capacity, dtype=torch.int32, device=self.device)
            need = int(self.L.rb_atm_scratch_bytes(n_buf, capacity))
            # zero-filled once: the overflow count at its tail (rb_atm_pass contract)
            self.atm_scratch = torch.zeros((need + 7) // 8, dtype=torch.float64, device=self.device)
            self.capacity = capacity

    def nlist(self, geom: Geometry, r_list: float, capacity: Optional[int] = None,
              checked: bool = True, gated: bool = False, tag: int = 0) -> None:
        """Build rank-sorted rows within r_list and their mirror indices.

        ``checked`` syncs and grows the capacity until no row overflows
        (container path); the device loop passes ``checked=False`` (and
        ``gated=True``) and inspects ``max_count`` at its sync points."""
        if capacity is None:
            capacity = self.capacity or self.estimate_capacity(geom, r_list)
        while True:
            self._ensure_rows(capacity)
            if checked:
                self.max_count.zero_()
            g = self.grid_struct(geom)
            need = int(self.L.rb_nlist_mirror_scratch_bytes(max(int(self.pos.shape[0]), 1)))
            if self.dir_scratch is None or self.dir_scratch.numel() < need:
                self.dir_scratch = self.torch.empty(need, dtype=self.torch.uint8,
                                                    device=self.device)
            st = self.L.rb_nlist_rows_mirror(
                ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.cell_start),
                ptr(self.cell_of_rank), float(r_list), int(self.capacity), ptr(self.rows),
                ptr(self.row_count), ptr(self.max_count), ptr(self.mirror), ptr(self.dir_scratch),
                self.dir_scratch.numel(), self._gate(gated), ptr(self.status), int(tag),
                self.stream)
            _lib.check(st, "rb_nlist_rows_mirror")
            if not checked:
                return
            worst = int(self.max_count.item())
            if worst <= self.capacity:
                self.slots = min(self.capacity, max(32, _round_up(worst, 32)))
                return
            if worst > 4096:
                raise CapacityError(f"a neighbour row holds {worst} entries (> 4096)")
            capacity = min(4096, _round_up(int(worst * 1.25) + 32, 32))

    def overflowed(self) -> bool:
        if int(self.max_count.item()) > self.capacity:
            return True
        err = self.read_status()
        return err is not None and err[1] == _lib.RB_KIND_CAPACITY

    # -------------------------------------------------------------- passes
    def lj(self, geom: Geometry, rc: float, epsilon: float, sigma: float, forces,
           tag: int = 0, reduce: bool = True, scalars: bool = True) -> None:
        self.lj_kernel(geom, rc, epsilon, sigma, forces, tag, scalars=scalars)
        if reduce:
            self.reduce_pair()

    def reduce_pair(self) -> None:
        self.sum_f64(self.e2_rank, SCALAR_E2)
        self.sum_f64(self.w2_rank, SCALAR_W2)

    def lj_kernel(self, geom: Geometry, rc: float, epsilon: float, sigma: float, forces,
                  tag: int = 0, scalars: bool = True) -> None:
        """The rb_lj_pass launch alone; scalars=False: forces only (the
        per-rank energy and virial are left as they are)."""
        g = self.grid_struct(geom)
        e2 = ptr(self.e2_rank) if scalars else _NULL
        w2 = ptr(self.w2_rank) if scalars else _NULL
        st = self.L.rb_lj_pass(ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.parts),
                               ptr(self.rows), ptr(self.row_count), int(self.capacity), float(rc),
                               float(epsilon), float(sigma), ptr(forces), e2, w2, self._owned(),
                               ptr(self.status), int(tag), self.stream)
        _lib.check(st, "rb_lj_pass")

    def atm(self, geom: Geometry, rc: float, nu: float, forces, tag: int = 0,
            count_visits: bool = True, reduce: bool = True) -> None:
        """Newton-3 triplet pass; ``self.visits`` <- unique triplet count."""
        self.atm_kernel(geom, rc, nu, forces, tag)
        if reduce:
            self.reduce_triplet()
        if count_visits:
            self._count()

    def reduce_triplet(self) -> None:
        self.sum_f64(self.e3_rank, SCALAR_E3)
        self.sum_f64(self.w3_rank, SCALAR_W3)

    CELLS_MODE = os.environ.get("RB_ATM_CELLS", "0")  # "1": cell-based where supported

    def uses_cells(self, geom: Geometry, rc: float) -> bool:
        """Whether the triplet pass of this geometry runs cell-based
        (rb_atm_pass_cells) rather than on the neighbour rows."""
        if self.CELLS_MODE == "0":
            return False
        key = (geom, float(rc))
        ok = self._cells_ok.get(key)
        if ok is None:
            g = self.grid_struct(geom)
            ok = bool(self.L.rb_atm_cells_supported(ctypes.byref(g), float(rc)))
            self._cells_ok[key] = ok
        return ok

    def cells_slots(self) -> int:
        """Slots of the cell-based pass: |S+(i)| is the forward half of the
        neighbours within the cutoff, (2/3) pi rc^3 rho on average; sized
        from the densest cell with margin (measured at nb_cap time)."""
        return int(self._cells_slots or min(256, max(32, _round_up(int(self.slots or 64), 32))))

    def _size_cells_slots(self, geom: Geometry, rc: float) -> None:
        counts = self.cell_start[1:geom.num_cells + 1] - self.cell_start[:geom.num_cells]
        max_occ = int(counts.max().item()) if geom.num_cells else 1
        dens = max(max_occ / float(np.prod(geom.cell_size)), self.n / float(np.prod(geom.box)))
        est = 2.0 / 3.0 * math.pi * rc ** 3 * dens
        self._cells_slots = int(min(256, max(32, _round_up(int(est * 1.45 * self.slots_margin)
                                                             + 8, 32))))

    def measure_nb_cap(self, geom: Geometry) -> int:
        """Staged-neighbourhood capacity from the current binning (syncs)."""
        g = self.grid_struct(geom)
        _lib.check(self.L.rb_atm_cells_nb_max(ctypes.byref(g), ptr(self.cell_start),
                                              ptr(self._nb_max), self.stream),
                   "rb_atm_cells_nb_max")
        worst = int(self._nb_max.item())
        self.nb_cap = _round_up(int(worst * self.nb_margin) + 16, 32)
        return self.nb_cap

    def grow_cells(self) -> None:
        """After a capacity error: larger margins at the next measurement."""
        self.nb_margin *= 1.5
        self.slots_margin *= 1.5
        self.nb_cap = 0

    def _atm_cells(self, geom: Geometry, rc: float, nu: float, forces, tag: int,
                   part: int) -> bool:
        torch = self.torch
        n_buf = max(int(self.pos.shape[0]), 1)
        need = int(self.L.rb_atm_cells_scratch_bytes(n_buf))
        if self.cells_scratch is None or self.cells_scratch.numel() * 8 < need:
            # zero-filled once: the cell counter at its head (rb_atm_pass_cells)
            self.cells_scratch = torch.zeros((need + 7) // 8, dtype=torch.float64,
                                             device=self.device)
        if self.nb_cap == 0:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("the cell-based triplet pass was first used under graph "
                                   "capture (run it once eagerly to size it)")
            self.measure_nb_cap(geom)
            self._size_cells_slots(geom, rc)
        slots = self.cells_slots()
        if int(self.L.rb_atm_cells_smem_bytes(int(self.nb_cap), slots)) > 227 * 1024:
            return False  # too dense for one CTA's shared memory: the row-based pass
        g = self.grid_struct(geom)
        st = self.L.rb_atm_pass_cells(ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.parts),
                                      ptr(self.cell_start), ptr(self.cell_of_rank),
                                      int(self.nb_cap), slots, float(rc), float(nu),
                                      ptr(forces), ptr(self.e3_rank), ptr(self.w3_rank),
                                      ptr(self.v_rank), self._owned(), ptr(self.cells_scratch),
                                      self.cells_scratch.numel() * 8, ptr(self.status),
                                      int(tag), int(part), self.stream)
        _lib.check(st, "rb_atm_pass_cells")
        return True

    def atm_kernel(self, geom: Geometry, rc: float, nu: float, forces, tag: int = 0,
                   part: int = 0) -> None:
        """The triplet pass launches alone (bench timing): cell-based when the
        geometry allows it (uses_cells), else on the rows.  part 1: the
        triplet kernels only (results in the scratch), part 2: the gather
        that writes forces and the per-rank scalars; 0: both."""
        if self.uses_cells(geom, rc) and self._atm_cells(geom, rc, nu, forces, tag, part):
            return
        g = self.grid_struct(geom)
        st = self.L.rb_atm_pass_part(ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.parts),
                                     ptr(self.rows), ptr(self.row_count), ptr(self.mirror),
                                     int(self.capacity), int(self.slots or self.capacity),
                                     float(rc), float(nu), ptr(forces), ptr(self.e3_rank),
                                     ptr(self.w3_rank), ptr(self.v_rank), self._owned(),
                                     ptr(self.atm_scratch), self.atm_scratch.numel() * 8,
                                     ptr(self.status), int(tag), int(part), self.stream)
        _lib.check(st, "rb_atm_pass_part")

    def atm_c01(self, geom: Geometry, rc: float, nu: float, forces, tag: int = 0,
                reduce: bool = True) -> None:
        """C01 (owner-computes) triplet pass; ``self.visits`` <- accepted visits."""
        g = self.grid_struct(geom)
        st = self.L.rb_atm_pass_c01(ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.parts),
                                    ptr(self.rows), ptr(self.row_count), int(self.capacity),
                                    float(rc), float(nu), ptr(forces), ptr(self.e3_rank),
                                    ptr(self.w3_rank), ptr(self.v_rank), ptr(self.status),
                                    int(tag), self.stream)
        _lib.check(st, "rb_atm_pass_c01")
        if not reduce:
            return
        self.reduce_triplet()
        self._count()

    # ------------------------------------------------------------ DirectSum
    def direct_pairs(self, epsilon: float, sigma: float, forces, tag: int = 0,
                     reduce: bool = True, rng=None) -> None:
        """All pairs of the particle-order positions (no cutoff, no image);
        per-particle halves in e2_rank/w2_rank, summed into scalars[E2],
        scalars[W2] when `reduce`.  `rng` = (lo, hi): the particles of one
        rank of a distributed DirectSum (other rows untouched)."""
        lo, hi = (0, self.n) if rng is None else (int(rng[0]), int(rng[1]))
        st = self.L.rb_direct_pairs_range(self.n, ptr(self.pos), lo, hi, float(epsilon),
                                          float(sigma), ptr(forces), ptr(self.e2_rank),
                                          ptr(self.w2_rank), ptr(self.status), int(tag),
                                          self.stream)
        _lib.check(st, "rb_direct_pairs_range")
        if reduce:
            self.reduce_pair()

    def direct_triplets(self, nu: float, forces, tag: int = 0, rng=None) -> None:
        """All triplets (Newton-3); scalars[E3], scalars[W3] <- energy, virial.
        `rng` = (lo, hi): only the triplets whose lowest member is in it."""
        need = int(self.L.rb_direct_scratch_bytes(self.n))
        if self.direct_scratch is None or self.direct_scratch.numel() * 8 < need:
            self.direct_scratch = self.torch.empty((need + 7) // 8, dtype=self.torch.float64,
                                                   device=self.device)
        ew = ctypes.c_void_p(self.scalars.data_ptr() + 8 * SCALAR_E3)
        lo, hi = (0, self.n) if rng is None else (int(rng[0]), int(rng[1]))
        st = self.L.rb_direct_triplets_range(self.n, ptr(self.pos), lo, hi, float(nu),
                                             ptr(forces), ew, ptr(self.direct_scratch),
                                             self.direct_scratch.numel() * 8, ptr(self.status),
                                             int(tag), self.stream)
        _lib.check(st, "rb_direct_triplets_range")

    def _count(self) -> None:
        st = self.L.rb_reduce_sum_i32(self.n, ptr(self.v_rank), ptr(self.visits),
                                      ptr(self.red_scratch), self.stream)
        _lib.check(st, "rb_reduce_sum_i32")

    def visit_rows(self, geom: Geometry, rc: float) -> np.ndarray:
        """Sorted (i, j, k) rows of every accepted visit (after :meth:`atm_c01`)."""
        torch = self.torch
        counts = self.v_rank[: self.n].to(torch.int64)
        offsets = torch.cumsum(counts, 0) - counts
        total = int(counts.sum().item())
        out = torch.empty(max(total, 1) * 3, dtype=torch.int32, device=self.device)
        g = self.grid_struct(geom)
        st = self.L.rb_atm_visit_rows(ctypes.byref(g), self.n, ptr(self.pos_r), ptr(self.parts),
                                      ptr(self.rows), ptr(self.row_count), int(self.capacity),
                                      float(rc), ptr(offsets), ptr(out), self.stream)
        _lib.check(st, "rb_atm_visit_rows")
        return out[: 3 * total].view(total, 3).cpu().numpy().astype(np.int64)

    # ----------------------------------------------------------- reductions
    def sum_f64(self, x, slot: int, square: bool = False, n: Optional[int] = None) -> None:
        fn = self.L.rb_reduce_sumsq_f64 if square else self.L.rb_reduce_sum_f64
        count = self.n if n is None else n
        out = ctypes.c_void_p(self.scalars.data_ptr() + 8 * slot)
        st = fn(count, ptr(x), out, ptr(self.red_scratch), self.stream)
        _lib.check(st, "rb_reduce")

    def sample(self, vel, trace=None, interval: int = 1) -> None:
        """scalars[0..4] <- (sum v^2, E2, W2, E3, W3) and, with `trace`, the
        trace row of the current device step, in one launch."""
        sc = self.scalars.data_ptr()
        st = self.L.rb_sample(self.n, ptr(vel), ptr(self.e2_rank), ptr(self.w2_rank),
                              ptr(self.e3_rank), ptr(self.w3_rank), ctypes.c_void_p(sc),
                              ptr(self.status), int(interval),
                              ptr(trace) if trace is not None else _NULL,
                              ptr(self.sample_scratch), self.sample_scratch.numel() * 8,
                              self.stream)
        _lib.check(st, "rb_sample")

    def scalar_values(self):
        return self.scalars.cpu().numpy()
