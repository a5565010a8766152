"""Observables on the device.

The radial distribution function is the one O(N^2) observable of the
reference (``respamd/observables.py:143-214``); here its pair-distance
histogram runs in ``rb_distance_histogram`` (bit-exact integer counts, the
reference's arithmetic) and the normalisation repeats the reference's numpy
expression.  The per-sample scalars (kinetic energy, virials, pressure) are
already device reductions of the r-RESPA loop (``RunTrace``); the small host
helpers here restate the reference's formulas for the experiment runner.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import _lib
from .model import ValidationError


def distance_histogram(positions, box, r_max: float, bins: int, counts=None):
    """Ordered minimum-image pair counts per bin (observables.py:143-177).

    `positions` is a host (n, 3) array or a device tensor; `counts` an int64
    device tensor of `bins` entries to accumulate into (allocated when None).
    Returns the device counts."""
    import torch

    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    pos = torch.as_tensor(np.ascontiguousarray(positions, dtype=np.float64)
                          if isinstance(positions, np.ndarray) else positions,
                          dtype=torch.float64, device=dev).contiguous()
    if counts is None:
        counts = torch.zeros(int(bins), dtype=torch.int64, device=dev)
    box3 = np.ascontiguousarray(box, dtype=np.float64)
    r_max = float(r_max)
    # the reference's own expressions (observables.py:145-146)
    inv_width = bins / r_max
    r2_max = r_max * r_max
    st = L.rb_distance_histogram(int(pos.shape[0]), _lib.ptr(pos), box3.ctypes.data,
                                 r2_max, inv_width, int(bins), _lib.ptr(counts),
                                 _lib.stream_handle())
    _lib.check(st, "rb_distance_histogram")
    return counts


def rdf(samples: Sequence, r_max: Optional[float] = None, bins: int = 200) -> np.ndarray:
    """Radial distribution function over periodic snapshots
    (observables.py:180-214): rows (r_center, g)."""
    if not samples:
        raise ValidationError("need at least one snapshot")
    first = samples[0]
    if not first.periodic:
        raise ValidationError("rdf requires periodic systems")
    box = np.asarray(first.box, dtype=np.float64)
    half_box = float(box.min()) / 2.0
    if r_max is None:
        r_max = half_box
    if r_max > half_box + 1e-12:
        raise ValidationError(f"r_max ({r_max}) must be <= half the smallest box edge ({half_box})")
    if bins < 1:
        raise ValidationError("bins must be >= 1")
    n = first.positions.shape[0]
    counts = None
    for system in samples:
        counts = distance_histogram(system.positions, system.box, float(r_max), bins, counts)
    return rdf_from_counts(counts.cpu().numpy(), n, float(np.prod(box)), float(r_max), bins,
                           len(samples))


def rdf_from_counts(counts: np.ndarray, n: int, volume: float, r_max: float, bins: int,
                    frames: int) -> np.ndarray:
    """g(r) = hist / (N rho V_shell n_frames), rho = N / V (observables.py:205-214)."""
    edges = np.linspace(0.0, r_max, bins + 1)
    shell_volumes = 4.0 / 3.0 * np.pi * (edges[1:] ** 3 - edges[:-1] ** 3)
    rho = n / volume
    g = counts / (n * rho * shell_volumes * frames)
    centers = 0.5 * (edges[:-1] + edges[1:])
    return np.column_stack([centers, g])


def rvite(total_energy: np.ndarray, mean_kinetic: float) -> float:
    """Relative variation in true energy (observables.py:90-102):
    sum |e - mean(e)| / (K J)."""
    e = np.asarray(total_energy, dtype=np.float64)
    if e.size < 1:
        raise ValidationError("energy series must not be empty")
    if mean_kinetic <= 0 or not np.isfinite(mean_kinetic):
        raise ValidationError(f"mean kinetic energy must be > 0, got {mean_kinetic}")
    return float(np.sum(np.abs(e - e.mean())) / (mean_kinetic * len(e)))


def pressure_virial(temperature: float, n: int, volume: float, pair_virial: float,
                    triplet_virial: float) -> float:
    """Virial pressure P = N T / V + (W2 + W3) / (3 V) (observables.py:217-225)."""
    return n * temperature / volume + (pair_virial + triplet_virial) / (3.0 * volume)


__all__ = ["distance_histogram", "pressure_virial", "rdf", "rdf_from_counts", "rvite"]
