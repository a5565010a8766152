"""Experiment runner, device equilibration and CLI on the GPU path
(SURVEY §8 f2): the reference's run/sweep/compare surface
(experiment.py:119-257, integrators.py:209-252, cli.py) with CSV outputs
that are byte-identical across reruns and values that follow the oracle."""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCENARIO = """\
# small periodic sweep for the runner
[system]
particles=216
box=7.2 7.2 7.2
periodic=true
container=linked_cells
temperature=0.8
equilibration={eq}
seed=11

[integration]
dt=0.002
iterations=20
step_size_factor=1

[force_field]
nu=0.3
cutoff=2.5

[sampling]
sample_every=2
rdf_sample_every=10
rdf_bins=24

[sweep]
nu_sweep=0.0,0.3
step_size_factors=1,2
"""


@pytest.fixture(scope="module")
def pkg():
    import paper_2507_11172_b200 as p
    from paper_2507_11172_b200 import _lib

    _lib.require_device()
    return p


def _write(tmp_path, eq=0):
    p = tmp_path / "sweep.scenario"
    p.write_text(SCENARIO.format(eq=eq))
    return p


def _files(root):
    out = {}
    for dirpath, _, names in os.walk(root):
        for n in names:
            path = os.path.join(dirpath, n)
            out[os.path.relpath(path, root)] = open(path, "rb").read()
    return out


def test_sweep_outputs_and_rerun_identical(pkg, tmp_path):
    from paper_2507_11172_b200.experiment import run_experiment
    from paper_2507_11172_b200.scenarios import parse_scenario

    plan = parse_scenario(_write(tmp_path, eq=20))
    r1 = run_experiment(plan, tmp_path / "a")
    r2 = run_experiment(parse_scenario(_write(tmp_path, eq=20)), tmp_path / "b")
    assert [p.status for p in r1.points] == ["ok"] * 4
    fa, fb = _files(tmp_path / "a"), _files(tmp_path / "b")
    assert set(fa) == set(fb)
    summary = fa.pop("summary.csv").decode().splitlines()
    fb.pop("summary.csv")
    assert summary[0] == ("nu,step_size_factor,status,rvite,rvite_warning,mean_energy,"
                          "mean_pressure,wall_seconds,speedup")
    assert len(summary) == 5 and all(",cutoff," in row for row in summary[1:])
    assert fa == fb  # energies, pressure, rdf: byte-identical reruns
    assert "nu0.3_s2/rdf.csv" in fa and "nu0.0_s1/energies.csv" in fa
    rows = fa["nu0.3_s2/energies.csv"].decode().splitlines()
    assert rows[0] == "iteration,kinetic,potential_2b,potential_3b,total"
    assert [int(r.split(",")[0]) for r in rows[1:]] == list(range(0, 21, 2))


def test_grid_point_follows_oracle(pkg, oracle, tmp_path):
    """No equilibration: energies.csv and the RDF follow the oracle loop."""
    from paper_2507_11172_b200.experiment import run_grid_point
    from paper_2507_11172_b200.model import build_lattice_system, init_velocities
    from paper_2507_11172_b200.scenarios import parse_scenario

    cfg = parse_scenario(_write(tmp_path, eq=0)).config.with_overrides(step_size_factor=2)
    res = run_grid_point(cfg, tmp_path / "pt")
    assert res.status == "ok"
    sysm = build_lattice_system(cfg)
    init_velocities(sysm, cfg.temperature, cfg.seed)
    osys = oracle.OracleSystem.from_positions(sysm.positions, sysm.box, True, sysm.velocities)
    off = oracle.OracleForceField(nu=0.3, cutoff=2.5)
    frames, totals = [osys.positions.copy()], []
    for k in range(2):  # 0 -> 10 -> 20: the RDF sample points
        tr = oracle.respa_run(osys, off, oracle.OracleLinkedCells(), cfg.dt, 2, 10, 2)
        totals += tr.total[(1 if k else 0):]
        frames.append(osys.positions.copy())
    got = np.loadtxt(tmp_path / "pt" / "energies.csv", delimiter=",", skiprows=1)
    assert np.max(np.abs(got[:, 4] - np.array(totals)) / np.abs(np.array(totals))) <= 1e-10
    r_max = float(cfg.box.min()) / 2.0
    counts = sum(oracle.distance_histogram(f, cfg.box, r_max, 24) for f in frames)
    # g per ordered pair count (observables.py:205-214), 3 frames (0, 10, 20)
    unit = 1.0 / (216 * (216 / float(np.prod(cfg.box))) * 4.0 / 3.0 * np.pi
                  * np.diff(np.linspace(0.0, r_max, 25) ** 3) * 3)
    g = np.loadtxt(tmp_path / "pt" / "rdf.csv", delimiter=",", skiprows=1)
    # trajectories agree to 1e-10: at most one pair may sit on a bin edge
    assert np.all(np.abs(g[:, 1] - counts * unit) <= 2.0 * unit + 1e-12)


def test_equilibrate_matches_oracle_rescaling(pkg, oracle):
    from paper_2507_11172_b200.integrators import equilibrate

    s = pkg.systems.fcc_system(4, jitter=0.05, seed=3, temperature=1.5, vseed=4)
    ff = pkg.ForceField(nu=0.2, cutoff=2.5)
    o = oracle.OracleSystem.from_positions(s.positions, s.box, True, s.velocities)
    rep = equilibrate(s, ff, pkg.CudaLinkedCells(), 0.002, 25, 0.7, rescale_interval=10)
    factors = []
    off = oracle.OracleForceField(nu=0.2, cutoff=2.5)
    done = 0
    while done < 25:  # integrators.py:237-246 on the oracle loop
        chunk = min(10, 25 - done)
        oracle.respa_run(o, off, oracle.OracleLinkedCells(), 0.002, 1, chunk, chunk)
        done += chunk
        t_now = 2.0 * (0.5 * float(np.sum(o.velocities * o.velocities))) / (3.0 * len(o.positions))
        f = math.sqrt(0.7 / t_now)
        o.velocities *= f
        factors.append(f)
    assert np.allclose(rep.rescale_factors, factors, rtol=1e-12, atol=0)
    assert np.max(np.abs(s.velocities - o.velocities)) <= 1e-10
    assert np.max(np.abs(s.positions - o.positions)) <= 1e-10
    assert rep.target_temperature == 0.7 and len(rep.rescale_factors) == 3


def test_cli_run_and_check(pkg, tmp_path):
    from paper_2507_11172_b200.cli import main

    scen = _write(tmp_path, eq=0)
    assert main(["--output", str(tmp_path / "o"), "run", str(scen)]) == 0
    assert (tmp_path / "o" / "summary.csv").exists()
    assert (tmp_path / "o" / "nu0.3_s1" / "pressure.csv").exists()
    assert main(["check"]) == 0
    bad = tmp_path / "bad.scenario"
    bad.write_text(SCENARIO.format(eq=0).replace("seed=11", "seed=11\nbogus=1"))
    assert main(["--output", str(tmp_path / "x"), "run", str(bad)]) == 1
