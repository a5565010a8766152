"""Run-time contracts of the device loop that have no reference analogue:
the neighbour-row overflow retry and the device workspace shared between a
running respa_run and container passes."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2507_11172_b200 as p
    from paper_2507_11172_b200 import _lib

    _lib.require_device()
    return p


def _fcc(pkg, nc=6):
    return pkg.systems.fcc_system(nc, jitter=0.02, seed=3, temperature=0.9, vseed=4)


def test_capacity_retry_resets_hooks(pkg):
    """Rows too small for the system: the run repeats larger, and a hook with
    reset() ends up with exactly one attempt's samples."""
    from paper_2507_11172_b200 import integrators

    class Hook:
        def __init__(self):
            self.iterations, self.resets = [], 0

        def __call__(self, iteration, positions):
            self.iterations.append(iteration)

        def reset(self):
            self.iterations, self.resets = [], self.resets + 1

    s = _fcc(pkg)
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    hook = Hook()
    pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 20), capacity=32,
                  device_hooks=(hook,))
    assert integrators.LAST_RUN[0].capacity > 32  # the run was repeated larger
    assert hook.resets >= 1
    assert hook.iterations == [0, 5, 10, 15, 20]
    ref = _fcc(pkg)
    pkg.respa_run(ref, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 20))
    np.testing.assert_array_equal(s.positions, ref.positions)


def test_container_pass_inside_hook_leaves_run_untouched(pkg):
    """A host hook that runs container passes on the same particle count
    gets its own workspace: the trajectory is bit-identical."""
    ff = pkg.ForceField(nu=0.073, cutoff=2.5)
    seen = []

    def hook(iteration, view, container):
        probe = pkg.CudaLinkedCells()
        sys2 = view.copy()
        probe.pair_pass(sys2, ff)
        probe.triplet_pass(sys2, ff)
        seen.append(probe.triplet_energy)

    a = _fcc(pkg)
    pkg.respa_run(a, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 30), hooks=(hook,))
    b = _fcc(pkg)
    pkg.respa_run(b, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.001, 5, 30))
    assert len(seen) == 7
    np.testing.assert_array_equal(a.positions, b.positions)
    np.testing.assert_array_equal(a.velocities, b.velocities)


def test_equilibrate_retries_after_row_overflow(pkg, monkeypatch):
    from paper_2507_11172_b200 import integrators
    from paper_2507_11172_b200.engine import CapacityError

    real = integrators._equilibrate
    calls = []

    def flaky(*args):
        calls.append(1)
        if len(calls) == 1:
            raise CapacityError("neighbour row overflow", 64)
        return real(*args)

    monkeypatch.setattr(integrators, "_equilibrate", flaky)
    s = _fcc(pkg, 4)
    x0 = s.positions.copy()
    rep = integrators.equilibrate(s, pkg.ForceField(nu=0.073, cutoff=2.5), pkg.CudaLinkedCells(),
                                  0.001, 20, 0.9)
    assert len(calls) == 2 and len(rep.rescale_factors) == 2
    ref = pkg.systems.fcc_system(4, jitter=0.02, seed=3, temperature=0.9, vseed=4)
    np.testing.assert_array_equal(ref.positions, x0)


@pytest.mark.parametrize("mode", ["rows", "cells"])
def test_runs_are_bitwise_reproducible(pkg, monkeypatch, mode):
    """Shared-memory ordering (warp sub-steps, per-warp target accumulators,
    persistent work counters) must not leak into the results: two runs of
    the same trajectory are bit-identical (a race would show up here; the
    pool has no compute-sanitizer)."""
    from paper_2507_11172_b200.engine import ForceEngine

    monkeypatch.setattr(ForceEngine, "CELLS_MODE", "1" if mode == "cells" else "0")
    ff = pkg.ForceField(nu=0.073, cutoff=2.5, cutoff_3b=3.0)
    out = []
    for _ in range(2):
        s = pkg.systems.fcc_system(7, jitter=0.03, seed=11, temperature=1.2, vseed=12)
        tr = pkg.respa_run(s, ff, pkg.CudaLinkedCells(), pkg.RespaSchedule(0.002, 5, 50))
        out.append((s, tr))
    (a, ta), (b, tb) = out
    assert np.array_equal(a.positions, b.positions)
    assert np.array_equal(a.velocities, b.velocities)
    assert np.array_equal(a.forces_3b, b.forces_3b)
    assert ta.total == tb.total and ta.potential_3b == tb.potential_3b
