"""Seeded synthetic particle systems standing in for BASELINE.json's configs.

The reference publishes no dataset; BASELINE.json's five configs are
recipes.  These builders generate them deterministically:

* lattice sites in unit-cell-major then basis order,
  ``meshgrid(arange(nc) x 3, indexing="ij")``;
* jitter ``default_rng(seed).uniform(-J, J, (N, 3))`` added to the sites,
  then wrapped with numpy ``mod`` (``respamd/model.py:274-280``);
* velocities from :func:`model.init_velocities` (the reference's
  Maxwell-Boltzmann recipe, ``respamd/model.py:255-271``).

The reduced-units FCC lattice constant at rho = 0.8 is (4/0.8)^(1/3).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .model import ForceField, ParticleSystem, init_velocities, wrap_positions

FCC_DENSITY = 0.8
FCC_A = (4.0 / FCC_DENSITY) ** (1.0 / 3.0)
FCC_BASIS = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
NU = 0.073


def _cell_grid(nc) -> np.ndarray:
    nx, ny, nz = (nc, nc, nc) if np.isscalar(nc) else nc
    g = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    return np.stack(g, axis=-1).reshape(-1, 3).astype(np.float64)


def _jitter_and_wrap(sites, box, jitter, seed) -> np.ndarray:
    rng = np.random.default_rng(seed)
    pos = sites + rng.uniform(-jitter, jitter, size=sites.shape)
    wrap_positions(pos, box)
    return pos


def fcc_system(nc, jitter: float = 0.02, seed: int = 1, temperature: float = 0.0,
               vseed: int = 1) -> ParticleSystem:
    """FCC block of nc^3 (or nx x ny x nz) unit cells at rho = 0.8, periodic."""
    cells = _cell_grid(nc)
    sites = ((cells[:, None, :] + FCC_BASIS[None, :, :]) * FCC_A).reshape(-1, 3)
    box = (np.full(3, nc * FCC_A) if np.isscalar(nc) else np.asarray(nc, dtype=np.float64) * FCC_A)
    system = ParticleSystem.empty(sites.shape[0], box, periodic=True)
    system.positions[:] = _jitter_and_wrap(sites, box, jitter, seed)
    init_velocities(system, temperature, vseed)
    return system


def sc_system(n_side: int = 10, spacing: float = 1.1, jitter: float = 0.05, seed: int = 1,
              temperature: float = 0.0, vseed: int = 1) -> ParticleSystem:
    """Simple-cubic n_side^3 lattice (BASELINE config 1)."""
    sites = _cell_grid(n_side) * spacing
    box = np.full(3, n_side * spacing)
    system = ParticleSystem.empty(sites.shape[0], box, periodic=True)
    system.positions[:] = _jitter_and_wrap(sites, box, jitter, seed)
    init_velocities(system, temperature, vseed)
    return system


def slab_system(n_total: int = 500_000, nc: int = 39, vapour_min_sep: float = 0.9, seed: int = 1,
                temperature: float = 0.8, vseed: int = 1, jitter: float = 0.02) -> ParticleSystem:
    """Liquid slab in a 1 x 1 x 4 elongated periodic box (BASELINE config 5).

    An nc x nc x 2nc FCC block (rho 0.8) fills the middle half of z; the
    remaining particles are uniform vapour in the outer halves placed by
    seeded rejection with a minimum separation (cell-accelerated).  With
    nc=39 the block holds 474,552 particles and the remaining 25,448 are
    vapour (rho_v ~ 0.043 instead of 0.02, SURVEY.md §8d recommendation).
    """
    L = nc * FCC_A
    box = np.array([L, L, 4.0 * L])
    cells = _cell_grid((nc, nc, 2 * nc))
    sites = ((cells[:, None, :] + FCC_BASIS[None, :, :]) * FCC_A).reshape(-1, 3)
    sites[:, 2] += L
    rng = np.random.default_rng(seed)
    liquid = sites + rng.uniform(-jitter, jitter, size=sites.shape)
    n_vap = n_total - liquid.shape[0]
    if n_vap < 0:
        raise ValueError("n_total smaller than the liquid block")
    # cell-accelerated rejection sampling of the vapour
    h = vapour_min_sep
    grid_n = np.maximum(1, np.floor(box / h).astype(np.int64))
    occupied: dict = {}
    for p in liquid:
        key = tuple(np.minimum((p % box) // (box / grid_n), grid_n - 1).astype(np.int64))
        occupied.setdefault(key, []).append(p % box)
    vapour = []
    sep2 = vapour_min_sep ** 2
    while len(vapour) < n_vap:
        cand = rng.uniform(0.0, 1.0, size=3) * box
        if L <= cand[2] < 3.0 * L:
            continue
        key = np.minimum(cand // (box / grid_n), grid_n - 1).astype(np.int64)
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    nb = tuple((key + (dx, dy, dz)) % grid_n)
                    for q in occupied.get(nb, ()):
                        d = cand - q
                        d -= box * np.floor(d / box + 0.5)
                        if d @ d < sep2:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            vapour.append(cand)
            occupied.setdefault(tuple(key), []).append(cand)
    pos = np.concatenate([liquid, np.array(vapour).reshape(-1, 3)], axis=0)
    wrap_positions(pos, box)
    system = ParticleSystem.empty(pos.shape[0], box, periodic=True)
    system.positions[:] = pos
    init_velocities(system, temperature, vseed)
    return system


@dataclass
class BenchConfig:
    """One BASELINE.json configuration: system recipe plus run schedule."""

    name: str
    description: str
    builder: str
    params: dict
    temperature: float
    rc_lj: float
    rc_atm: float
    dt: float
    steps: int
    step_size_factor: int

    def system(self) -> ParticleSystem:
        fn = {"fcc": fcc_system, "sc": sc_system, "slab": slab_system}[self.builder]
        return fn(temperature=self.temperature, **self.params)

    def force_field(self, rc_atm: Optional[float] = None) -> ForceField:
        rc3 = self.rc_atm if rc_atm is None else rc_atm
        return ForceField(epsilon=1.0, sigma=1.0, nu=NU, cutoff=self.rc_lj,
                          cutoff_3b=None if rc3 == self.rc_lj else rc3)


CONFIGS = {
    "cfg1": BenchConfig("cfg1", "SC 10^3 spacing 1.1, jitter 0.05, box 11, T 0.7", "sc",
                        dict(n_side=10, spacing=1.1, jitter=0.05, seed=1, vseed=1), 0.7,
                        2.5, 2.5, 0.001, 10, 1),
    "cfg2": BenchConfig("cfg2", "FCC 20^3 (32,000), rho 0.8, jitter 0.02, T 0.9", "fcc",
                        dict(nc=20, jitter=0.02, seed=1, vseed=1), 0.9, 2.5, 2.5, 0.001, 100, 5),
    "cfg3": BenchConfig("cfg3", "FCC 40^3 (256,000), rho 0.8, jitter 0.02, T 0.9", "fcc",
                        dict(nc=40, jitter=0.02, seed=1, vseed=1), 0.9, 2.5, 2.5, 0.001, 200, 5),
    "cfg4": BenchConfig("cfg4", "FCC 80^3 (2,048,000), rho 0.8, jitter 0.02, T 0.9", "fcc",
                        dict(nc=80, jitter=0.02, seed=1, vseed=1), 0.9, 2.5, 2.5, 0.001, 100, 5),
    "cfg5": BenchConfig("cfg5", "liquid slab 500,000 in L x L x 4L, T 0.8", "slab",
                        dict(n_total=500_000, nc=39, seed=1, vseed=1), 0.8, 2.5, 2.5, 0.001, 200,
                        10),
}
