"""CPU-side checks of the product: the C-ABI library and the host logic.

No kernel is launched here (there is no GPU in the build container): the
library must load, export every symbol include/respa_b200.h declares, and
the host restatements (grid geometry, stencil tables, scenario format) must
equal the reference's outputs recorded in tests/golden.
"""

import ctypes
import glob
import os
import re

import numpy as np
import pytest

from helpers import GOLDEN, REPO, load_golden

SMALL = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "small_*.npz")))


def header_symbols():
    text = open(os.path.join(REPO, "include", "respa_b200.h")).read()
    return sorted(set(re.findall(r"RB_API\s+[\w\s\*]+?\b(rb_\w+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2507_11172_b200 import _lib, build

    path = build.build()
    lib = ctypes.CDLL(path)
    names = header_symbols()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding declares exactly the header's symbols
    assert sorted(_lib.SIGNATURES) == names


def test_binding_argument_counts_match_header():
    """Every ctypes prototype has as many arguments as the header declares."""
    from paper_2507_11172_b200 import _lib

    text = open(os.path.join(REPO, "include", "respa_b200.h")).read()
    for m in re.finditer(r"RB_API\s+[\w\s\*]+?\b(rb_\w+)\s*\(([^;]*?)\);", text, re.S):
        args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        assert len(_lib.SIGNATURES[m.group(1)][1]) == len(args), m.group(1)


def test_library_metadata_calls_without_gpu():
    from paper_2507_11172_b200 import _lib

    L = _lib.lib()
    assert L.rb_abi_version() == 1
    assert L.rb_status_string(_lib.RB_ERR_CAPACITY).decode().startswith("neighbour")
    assert L.rb_bin_scratch_bytes(1000, 64) > 0


def test_sass_is_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess

    from paper_2507_11172_b200 import build

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", SMALL)
def test_geometry_and_stencils_match_reference(name):
    from paper_2507_11172_b200 import grid

    g = load_golden(name)
    pos = g["positions"]
    geom = grid.geometry(g["box"], pos, float(g["cutoff"]), bool(g["periodic"]))
    assert geom.cells == tuple(int(c) for c in g["cells"])
    assert np.array_equal(np.array(geom.cell_size), g["cell_size"])
    assert np.array_equal(np.array(geom.origin), g["origin"])
    pair, patterns, same = grid.stencil(geom)
    assert np.array_equal(pair, g["pair_cells"])
    assert np.array_equal(patterns, g["triplet_patterns"])
    assert np.array_equal(same, g["triplet_same_cell"])


def test_periodic_box_too_small_rejected():
    from paper_2507_11172_b200 import ValidationError, grid

    with pytest.raises(ValidationError):
        grid.geometry((3.0, 3.0, 3.0), None, 2.5, True)


def test_known_geometries():
    """Reference test_containers.py:36-45 geometry facts."""
    from paper_2507_11172_b200 import grid

    g10 = grid.geometry((10.0,) * 3, None, 2.5, True)
    assert g10.cells == (4, 4, 4) and g10.reach == (1, 1, 1)
    assert np.allclose(g10.cell_size, 2.5)
    assert grid.geometry((20.0,) * 3, None, 2.5, True).cells == (8, 8, 8)
    # BASELINE geometries: 27 neighbour cells, 185 patterns
    from paper_2507_11172_b200 import systems

    for nc in (20, 40, 80):
        geom = grid.geometry(np.full(3, nc * systems.FCC_A), None, 2.5, True)
        pair, patterns, same = grid.stencil(geom)
        assert pair.shape[0] == 27 and patterns.shape[0] == 185 and int(same.sum()) == 27


def test_rb_grid_struct_layout():
    from paper_2507_11172_b200 import _lib, grid

    geom = grid.geometry((11.0,) * 3, None, 2.5, True)
    g = grid.rb_grid(geom)
    assert ctypes.sizeof(_lib.RbGrid) == _lib.lib().rb_grid_bytes()
    assert tuple(g.cells) == (4, 4, 4) and g.n_offsets == 27 and g.periodic == 1
    assert g.inv_cell[0] == 1.0 / (11.0 / 4)


def test_model_mirrors_reference_validation():
    from paper_2507_11172_b200 import ForceField, ParticleSystem, ScenarioConfig, ValidationError

    with pytest.raises(ValidationError):
        ForceField(nu=-1.0)
    with pytest.raises(ValidationError):
        ForceField(cutoff=0.0)
    with pytest.raises(ValidationError):
        ScenarioConfig(particle_count=10, box=(5, 5, 5), dt=0.001, iterations=7,
                       step_size_factor=2)
    s = ParticleSystem.empty(4, (5.0, 5.0, 5.0), periodic=True)
    v = s.view()
    with pytest.raises(ValueError):
        v.positions[0, 0] = 1.0
    with pytest.raises(ValidationError):
        ParticleSystem(np.full((2, 3), 6.0), np.zeros((2, 3)), np.zeros((2, 3)), np.zeros((2, 3)),
                       1.0, (5.0, 5.0, 5.0), True)


def test_init_velocities_matches_reference_recipe():
    from paper_2507_11172_b200 import ParticleSystem, init_velocities

    s = ParticleSystem.empty(1000, (11.0,) * 3, periodic=True)
    init_velocities(s, 0.7, 1)
    g = load_golden("respa_cfg1.npz")
    assert np.array_equal(s.velocities, g["v0"])
    assert np.max(np.abs(s.velocities.sum(axis=0))) < 1e-12


def test_wrap_positions_numpy_semantics():
    from paper_2507_11172_b200 import wrap_positions

    box = np.array([5.0, 5.0, 5.0])
    x = np.array([[-1e-17, 5.0, 12.5], [-0.0, -5.0, 4.999999999999999]])
    wrap_positions(x, box)
    assert np.all(x >= 0) and np.all(x < box)
    assert x[0, 0] == 0.0 and x[0, 1] == 0.0 and x[0, 2] == 2.5


SCENARIO = """\
# a small periodic sweep in the reference format
[system]
particles=64
box=6 6 6
periodic=true
container=cuda_linked_cells
temperature=0.9
seed=3

[integration]
dt=0.002
iterations=12
step_size_factor=1

[force_field]
nu=0.3
cutoff=2.5
cutoff_3b=2.8

[sweep]
step_size_factors=1,2,3
"""


def test_scenario_format(tmp_path):
    from paper_2507_11172_b200 import ScenarioParseError, parse_scenario

    p = tmp_path / "a.scenario"
    p.write_text(SCENARIO)
    plan = parse_scenario(p)
    assert plan.config.particle_count == 64 and plan.config.periodic
    assert plan.config.force_field.cutoff_3b == 2.8
    assert plan.grid() == [(0.3, 1), (0.3, 2), (0.3, 3)]
    bad = tmp_path / "b.scenario"
    bad.write_text(SCENARIO.replace("seed=3", "seed=3\nbogus=1"))
    with pytest.raises(ScenarioParseError) as err:
        parse_scenario(bad)
    assert err.value.line_no == 9
    dup = tmp_path / "c.scenario"
    dup.write_text(SCENARIO + "nu=0.4\n")
    with pytest.raises(ScenarioParseError):
        parse_scenario(dup)


def test_direct_sum_rejects_periodic_systems():
    """test_containers.py:215-220: raised before any device work."""
    import paper_2507_11172_b200 as pkg

    s = pkg.ParticleSystem.empty(3, (8.0, 8.0, 8.0), periodic=True)
    s.positions[:] = [[0.5, 0.5, 0.5], [2.0, 0.5, 0.5], [0.5, 2.0, 0.5]]
    ff = pkg.ForceField()
    with pytest.raises(pkg.ValidationError):
        pkg.direct_sum_pairs(s, ff)
    with pytest.raises(pkg.ValidationError):
        pkg.direct_sum_triplets(s, ff)
    assert pkg.make_container("direct_sum").name == "cuda_direct_sum"


def test_lattice_system_matches_reference():
    """build_lattice_system restates model.py:212-252 (fixture made by it)."""
    from helpers import load_golden

    import paper_2507_11172_b200 as pkg
    from paper_2507_11172_b200.model import build_lattice_system

    g = load_golden("lattice.npz")
    for k in range(int(g["cases"])):
        cfg = pkg.ScenarioConfig(particle_count=int(g[f"n{k}"]), box=g[f"box{k}"], dt=0.001,
                                 iterations=10, container="cuda_linked_cells", periodic=True)
        assert np.array_equal(build_lattice_system(cfg).positions, g[f"pos{k}"])


def test_distributed_direct_sum_partition():
    """Base ranges cover [0, n) in order with equal triplet counts (to one
    base); particle ranges are equal."""
    from paper_2507_11172_b200.direct_dist import base_ranges, particle_ranges

    for n, parts in ((1000, 8), (4096, 3), (7, 4), (2, 2)):
        for ranges in (base_ranges(n, parts), particle_ranges(n, parts)):
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        if n >= 1000:
            m = np.arange(n - 1, -1, -1, dtype=np.float64)
            work = m * (m - 1) / 2.0
            shares = [work[a:b].sum() for a, b in base_ranges(n, parts)]
            assert max(shares) - min(shares) <= work.max() + 1e-9 * work.sum()


REF_SCENARIOS = "/root/reference/pkg/scenarios"
REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SCENARIOS), reason="reference tree not present")
def test_reference_bundled_scenarios_parse_identically():
    """All five scenario files bundled with the reference (pkg/scenarios)
    parse, and give the same plan as respamd's own parser (scenarios.py:150-214):
    every configuration field, the sweeps and the (nu, s) grid."""
    import dataclasses
    import glob
    import subprocess
    import sys

    from paper_2507_11172_b200 import parse_scenario

    files = sorted(glob.glob(os.path.join(REF_SCENARIOS, "*.scenario")))
    assert len(files) == 5
    code = r"""
import dataclasses, json, sys
from respamd.scenarios import parse_scenario
out = {}
for f in sys.argv[1:]:
    p = parse_scenario(f)
    c = dataclasses.asdict(p.config)
    out[f] = {"config": json.loads(json.dumps(c, default=lambda o: list(o))),
              "nu": p.nu_values, "s": p.step_size_factors, "grid": p.grid()}
print(json.dumps(out))
"""
    env = dict(os.environ, PYTHONPATH=REF_SRC, NUMBA_CACHE_DIR="/tmp/numba_cache_respamd")
    res = subprocess.run([sys.executable, "-c", code, *files], capture_output=True, text=True,
                         env=env, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    import json

    ref = json.loads(res.stdout.splitlines()[-1])
    for f in files:
        plan = parse_scenario(f)
        mine = json.loads(json.dumps(dataclasses.asdict(plan.config), default=lambda o: list(o)))
        theirs = ref[f]["config"]
        def same(a, b, where):  # every field the reference has, same value (ours may add
            if isinstance(b, dict):  # e.g. force_field.cutoff_3b, None = as the reference)
                for k, v in b.items():
                    same(a.get(k), v, where + "." + k)
            else:
                assert a == b, (os.path.basename(f), where, a, b)

        same(mine, theirs, "config")
        assert plan.nu_values == ref[f]["nu"] and plan.step_size_factors == ref[f]["s"]
        assert [list(g) for g in plan.grid()] == ref[f]["grid"]
