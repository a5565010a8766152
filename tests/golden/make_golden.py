"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (the reference tree is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
records its outputs on seeded inputs:

* potentials.npz      -- lj_kernel / atm_kernel on random arguments
                          (respamd/potentials.py:55-114)
* small_<name>.npz    -- full arrays for small systems: binning
                          (containers.py:175-209), stencil tables (:100-172),
                          C01 pair/triplet passes (:750-822), visit counts
                          (:825-849), brute force (reference.py:111-122)
* large_<cfg>.npz     -- BASELINE configs 1-4 at step 0: a sha256 of the
                          generated positions (pins the generator), the four
                          scalars, the visit count and forces of a fixed
                          particle subset
* respa_<name>.npz    -- respa_run trajectories (integrators.py:96-173)
* rdf.npz             -- rdf / _distance_histogram (observables.py:143-214)
* lattice.npz         -- build_lattice_system (model.py:212-252)
* direct.npz          -- DirectSum pairs/triplets (containers.py:852-908) on
                          non-periodic systems (the reference test's four
                          particles and random n = 70 / 150 / 300)

Inputs are produced by this repo's generators (paper_2507_11172_b200.systems
and tests/helpers.random_positions); the reference only supplies outputs.
"""

from __future__ import annotations

import glob
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
REF_SRC = os.environ.get("RESPAMD_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from respamd import containers as rc  # noqa: E402
from respamd import integrators as ri  # noqa: E402
from respamd import model as rm  # noqa: E402
from respamd import potentials as rp  # noqa: E402
from respamd import reference as rr  # noqa: E402

from helpers import TEST_SEED, random_positions  # noqa: E402
from paper_2507_11172_b200 import systems  # noqa: E402

SUBSET = np.array(sorted(set([0, 1, 2, 3, 17, 101, 999] + list(range(500, 532)))), np.int64)


def ref_system(pos, box, periodic, vel=None):
    s = rm.ParticleSystem.empty(len(pos), box, periodic=periodic)
    s.positions[:] = pos
    if vel is not None:
        s.velocities[:] = vel
    return s


def gen_potentials():
    rng = np.random.default_rng(7)
    r2 = rng.uniform(0.7, 6.25, 2000)
    lj = np.array([rp.lj_kernel(x, 1.0, 1.0) for x in r2])
    abc = []
    while len(abc) < 2000:
        pts = rng.uniform(-2.0, 2.0, size=(3, 3))
        d = [pts[0] - pts[1], pts[0] - pts[2], pts[1] - pts[2]]
        sq = [float(v @ v) for v in d]
        if min(sq) > 0.64 and max(sq) < 6.25:
            abc.append(sq)
    abc = np.array(abc)
    atm = np.array([rp.atm_kernel(a, b, c, 0.7) for a, b, c in abc])
    np.savez_compressed(os.path.join(HERE, "potentials.npz"), r2=r2, lj=lj, abc=abc, atm=atm, nu=0.7)


SMALL = [
    # name, edge, n, periodic, seed offset
    ("e6_n120", 6.0, 120, True, 1),
    ("e7.5_n160", 7.5, 160, True, 2),
    ("e10_n200", 10.0, 200, True, 3),  # size == cutoff exactly (332 patterns)
    ("e9_n150", 9.0, 150, True, 4),
    ("e5.2_n60", 5.2, 60, True, 5),  # 2 cells per dimension
    ("e8_n180", 8.0, 180, True, 6),  # 3 cells per dimension
    ("free_e6_n70", 6.0, 70, False, 7),
    ("free_e7_n90", 7.0, 90, False, 8),
]


def gen_small():
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=0.7, cutoff=2.5)
    for name, edge, n, periodic, off in SMALL:
        rng = np.random.default_rng(TEST_SEED + off)
        pos = random_positions(rng, n, (edge,) * 3, periodic)
        sysm = ref_system(pos, (edge,) * 3, periodic)
        grid = rc.build_cell_grid(sysm, ff.cutoff)
        f2, e2, w2 = rc.c01_pair_pass(grid, sysm, ff)
        f3, e3, w3 = rc.c01_triplet_pass(grid, sysm, ff)
        visits = rc.collect_triplet_visits(grid, sysm)
        bf2, be2, bw2 = rr.brute_force_pairs(sysm, ff, cutoff=ff.cutoff)
        bf3, be3, bw3, count = rr.brute_force_triplets(sysm, ff, cutoff=ff.cutoff)
        uniq = np.unique(visits, axis=0)
        np.savez_compressed(
            os.path.join(HERE, f"small_{name}.npz"),
            positions=pos, box=np.full(3, edge), periodic=periodic, nu=ff.nu, cutoff=ff.cutoff,
            cells=grid.cells_per_dim, cell_size=grid.cell_size, origin=grid.origin,
            reach=grid.interaction_reach, cell_start=grid.cell_start,
            cell_particles=grid.cell_particles, pair_cells=grid.pair_cells,
            triplet_patterns=grid.triplet_patterns, triplet_same_cell=grid.triplet_same_cell,
            f2=f2, e2=e2, w2=w2, f3=f3, e3=e3, w3=w3, visits=len(visits),
            unique_triplets=uniq, bf2=bf2, be2=be2, bw2=bw2, bf3=bf3, be3=be3, bw3=bw3,
            brute_count=count,
        )
        print(f"small_{name}: cells {grid.cells_per_dim} patterns {len(grid.triplet_patterns)} "
              f"visits {len(visits)} brute {count}")


def pos_sha(pos):
    return hashlib.sha256(np.ascontiguousarray(pos, dtype=np.float64).tobytes()).hexdigest()


def gen_large():
    rows = [("cfg1", "cfg1", 2.5), ("cfg2", "cfg2", 2.5), ("cfg3_rc2.0", "cfg3", 2.0),
            ("cfg3_rc2.5", "cfg3", 2.5), ("cfg3_rc3.0", "cfg3", 3.0), ("cfg4", "cfg4", 2.5),
            ("cfg5", "cfg5", 2.5)]
    only = os.environ.get("GOLDEN_LARGE")  # e.g. GOLDEN_LARGE=cfg5 regenerates one row
    for name, cfg_name, rc3 in rows:
        if only and name not in only.split(","):
            continue
        cfg = systems.CONFIGS[cfg_name]
        s = cfg.system()
        sysm = ref_system(s.positions, s.box, True)
        ff2 = rm.ForceField(epsilon=1.0, sigma=1.0, nu=systems.NU, cutoff=cfg.rc_lj)
        ff3 = rm.ForceField(epsilon=1.0, sigma=1.0, nu=systems.NU, cutoff=rc3)
        t0 = time.perf_counter()
        g2 = rc.build_cell_grid(sysm, ff2.cutoff)
        f2, e2, w2 = rc.c01_pair_pass(g2, sysm, ff2)
        g3 = rc.build_cell_grid(sysm, ff3.cutoff)
        f3, e3, w3 = rc.c01_triplet_pass(g3, sysm, ff3)
        vis_rows = rc.collect_triplet_visits(g3, sysm) if s.n <= 300_000 else None
        visits = -1 if vis_rows is None else len(vis_rows)
        np.savez_compressed(
            os.path.join(HERE, f"large_{name}.npz"),
            sha=pos_sha(s.positions), n=s.n, box=s.box, rc2=cfg.rc_lj, rc3=rc3, nu=systems.NU,
            e2=e2, w2=w2, e3=e3, w3=w3, visits=visits, subset=SUBSET[SUBSET < s.n],
            f2=f2[SUBSET[SUBSET < s.n]], f3=f3[SUBSET[SUBSET < s.n]],
            f2_absmax=np.max(np.abs(f2)), f3_absmax=np.max(np.abs(f3)),
            f2_sum=np.sum(f2, axis=0), f3_sum=np.sum(f3, axis=0),
            cell_particles_head=g3.cell_particles[:4096], cells=g3.cells_per_dim,
        )
        print(f"large_{name}: N={s.n} E2={e2!r} E3={e3!r} visits={visits} "
              f"({time.perf_counter() - t0:.1f}s)")


def fill_large_visits():
    """The large fixtures of n > 300k carry no reference visit count (the
    reference's collect_triplet_visits is too slow there): fill it from the
    oracle's C01 enumeration, which is bit-pinned against the reference on
    every smaller fixture (tests/test_oracle_golden.py).  Marks the source."""
    from oracle import oracle as orc

    orc.build()
    orc.set_num_threads(os.cpu_count() or 1)
    for path in sorted(glob.glob(os.path.join(HERE, "large_*.npz"))):
        d = dict(np.load(path, allow_pickle=False))
        if int(d["visits"]) >= 0:
            continue
        cfg_name = os.path.basename(path)[len("large_"):].split(".npz")[0].split("_")[0]
        s = systems.CONFIGS[cfg_name].system()
        assert pos_sha(s.positions) == str(d["sha"])
        os_ = orc.OracleSystem.from_positions(s.positions, s.box, True)
        grid = orc.build_cell_grid(os_, float(d["rc3"]))
        d["visits"] = np.int64(orc.triplet_visit_count(grid, os_))
        d["visits_source"] = np.array("oracle")
        np.savez_compressed(path, **d)
        print(f"{os.path.basename(path)}: visits {int(d['visits'])} (oracle)")


class SplitCutoffLC:
    """Duck-typed reference container with its own ATM cutoff."""

    name = "linked_cells"

    def __init__(self, rc3):
        self.rc3 = rc3
        self.inner = rc.LinkedCells()

    def pair_pass(self, system, ff):
        self.inner.pair_pass(system, ff)

    def triplet_pass(self, system, ff):
        ff3 = rm.ForceField(epsilon=ff.epsilon, sigma=ff.sigma, nu=ff.nu, cutoff=self.rc3)
        self.inner.triplet_pass(system, ff3)

    def __getattr__(self, item):
        return getattr(self.inner, item)


def _trace_arrays(trace):
    return dict(
        t_iterations=np.array(trace.iterations), t_kinetic=np.array(trace.kinetic),
        t_p2=np.array(trace.potential_2b), t_p3=np.array(trace.potential_3b),
        t_total=np.array(trace.total), t_w2=np.array(trace.virial_2b),
        t_w3=np.array(trace.virial_3b),
    )


def gen_respa():
    # cfg1: the BASELINE parity config (10 steps, s = 1)
    cfg = systems.CONFIGS["cfg1"]
    s = cfg.system()
    sysm = ref_system(s.positions, s.box, True, s.velocities)
    x0, v0 = sysm.positions.copy(), sysm.velocities.copy()
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=systems.NU, cutoff=2.5)
    trace = ri.respa_run(sysm, ff, rc.LinkedCells(), ri.RespaSchedule(0.001, 1, 10))
    np.savez_compressed(os.path.join(HERE, "respa_cfg1.npz"), x0=x0, v0=v0, box=s.box, dt=0.001,
                        s=1, steps=10, nu=systems.NU, cutoff=2.5, x=sysm.positions,
                        v=sysm.velocities, f2=sysm.forces_2b, f3=sysm.forces_3b,
                        **_trace_arrays(trace))
    print("respa_cfg1 total:", trace.total[0], trace.total[-1])

    # small periodic system, s = 3, sampled every 3
    rng = np.random.default_rng(TEST_SEED + 11)
    pos = random_positions(rng, 60, (6.5,) * 3, True)
    sysm = ref_system(pos, (6.5,) * 3, True)
    rm.init_velocities(sysm, 1.2, seed=3)
    x0, v0 = sysm.positions.copy(), sysm.velocities.copy()
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=0.7, cutoff=2.5)
    trace = ri.respa_run(sysm, ff, rc.LinkedCells(), ri.RespaSchedule(0.002, 3, 300))
    np.savez_compressed(os.path.join(HERE, "respa_small_s3.npz"), x0=x0, v0=v0, box=np.full(3, 6.5),
                        dt=0.002, s=3, steps=300, nu=0.7, cutoff=2.5, x=sysm.positions,
                        v=sysm.velocities, f2=sysm.forces_2b, f3=sysm.forces_3b,
                        **_trace_arrays(trace))

    # cfg2: 100 steps, s = 5 (subset of the final state + full trace)
    cfg = systems.CONFIGS["cfg2"]
    s = cfg.system()
    sysm = ref_system(s.positions, s.box, True, s.velocities)
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=systems.NU, cutoff=2.5)
    t0 = time.perf_counter()
    trace = ri.respa_run(sysm, ff, rc.LinkedCells(), ri.RespaSchedule(0.001, 5, 100))
    np.savez_compressed(os.path.join(HERE, "respa_cfg2.npz"), sha=pos_sha(s.positions),
                        vsha=pos_sha(s.velocities), box=s.box, dt=0.001, s=5, steps=100,
                        nu=systems.NU, cutoff=2.5, subset=SUBSET, x=sysm.positions[SUBSET],
                        v=sysm.velocities[SUBSET], **_trace_arrays(trace))
    print(f"respa_cfg2 {time.perf_counter() - t0:.1f}s total {trace.total[0]} -> {trace.total[-1]}")

    # cfg3-like split cutoff (rc_ATM 3.0) on a small FCC block, s = 2
    s = systems.fcc_system(6, jitter=0.02, seed=3, temperature=0.9, vseed=4)
    sysm = ref_system(s.positions, s.box, True, s.velocities)
    x0, v0 = sysm.positions.copy(), sysm.velocities.copy()
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=systems.NU, cutoff=2.5)
    trace = ri.respa_run(sysm, ff, SplitCutoffLC(3.0), ri.RespaSchedule(0.001, 2, 20))
    np.savez_compressed(os.path.join(HERE, "respa_split_rc3.npz"), x0=x0, v0=v0, box=s.box,
                        dt=0.001, s=2, steps=20, nu=systems.NU, cutoff=2.5, cutoff_3b=3.0,
                        x=sysm.positions, v=sysm.velocities, f2=sysm.forces_2b,
                        f3=sysm.forces_3b, **_trace_arrays(trace))


DIRECT = [  # name, edge, n, rng offset (non-periodic random systems)
    ("e7_n70", 7.0, 70, 31),
    ("e9_n150", 9.0, 150, 32),
    ("e12_n300", 12.0, 300, 33),
]


def gen_direct():
    """DirectSum (containers.py:852-908) on non-periodic systems: the
    four-particle system of test_containers.py:189-207 and random ones."""
    ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=0.7, cutoff=2.5)
    cases = [("four", np.array([[0.0, 0.0, 0.0], [1.2, 0.0, 0.0], [0.0, 1.3, 0.0],
                                [0.0, 0.0, 1.4]]), 50.0)]
    for name, edge, n, off in DIRECT:
        rng = np.random.default_rng(TEST_SEED + off)
        cases.append((name, random_positions(rng, n, (edge,) * 3, False), edge))
    out = {}
    for name, pos, edge in cases:
        sysm = ref_system(pos, (edge,) * 3, False)
        f2, e2, w2 = rc.direct_sum_pairs(sysm, ff)
        f3, e3, w3 = rc.direct_sum_triplets(sysm, ff)
        for k, v in dict(pos=pos, box=np.full(3, edge), f2=f2, e2=e2, w2=w2, f3=f3, e3=e3,
                         w3=w3).items():
            out[f"{name}__{k}"] = v
        print(f"direct {name}: n {len(pos)} e2 {e2} e3 {e3}")
    np.savez_compressed(os.path.join(HERE, "direct.npz"), names=np.array([c[0] for c in cases]),
                        nu=ff.nu, **out)


def gen_rdf():
    """Radial distribution function (observables.py:143-214): the raw ordered
    pair counts and the g(r) curve."""
    from respamd import observables as ro

    out = {}
    s1 = systems.CONFIGS["cfg1"].system()
    rng = np.random.default_rng(TEST_SEED + 41)
    pos = random_positions(rng, 300, (8.0,) * 3, True)
    cases = [("cfg1", [s1.positions], s1.box, None, 200),
             ("rand300", [pos, np.mod(pos + 0.37, 8.0)], np.full(3, 8.0), 3.0, 50)]
    for name, frames, box, r_max, bins in cases:
        snaps = [ref_system(f, box, True) for f in frames]
        curve = ro.rdf(snaps, r_max=r_max, bins=bins)
        rm_ = float(box.min()) / 2.0 if r_max is None else r_max
        counts = sum(ro._distance_histogram(f, np.asarray(box, dtype=np.float64), rm_, bins)
                     for f in frames)
        for k, v in dict(box=np.asarray(box), r_max=rm_, bins=bins, curve=curve,
                         counts=counts).items():
            out[f"{name}__{k}"] = v
        for i, f in enumerate(frames):
            out[f"{name}__frame{i}"] = f
        out[f"{name}__frames"] = len(frames)
        print(f"rdf {name}: frames {len(frames)} pairs {int(counts.sum())}")
    np.savez_compressed(os.path.join(HERE, "rdf.npz"), names=np.array([c[0] for c in cases]),
                        **out)


LATTICES = [(1000, (11.0, 11.0, 11.0)), (37, (5.0, 6.0, 7.0)), (500, (10.0, 10.0, 40.0)),
            (8, (3.0, 3.0, 3.0))]


def gen_lattice():
    """build_lattice_system (model.py:212-252) for a few counts and boxes."""
    out = {}
    for k, (n, box) in enumerate(LATTICES):
        cfg = rm.ScenarioConfig(particle_count=n, box=np.array(box), dt=0.001, iterations=10,
                                container="linked_cells", periodic=True)
        out[f"n{k}"] = n
        out[f"box{k}"] = np.array(box)
        out[f"pos{k}"] = rm.build_lattice_system(cfg).positions
    np.savez_compressed(os.path.join(HERE, "lattice.npz"), cases=len(LATTICES), **out)
    print(f"lattice: {len(LATTICES)} cases")


if __name__ == "__main__":
    what = sys.argv[1:] or ["potentials", "small", "large", "large_visits", "respa", "direct",
                            "rdf", "lattice"]
    for w in what:
        (fill_large_visits if w == "large_visits" else globals()[f"gen_{w}"])()
