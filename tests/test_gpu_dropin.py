"""Drop-in proof: respamd's OWN container and integrator tests (its
pkg/tests/test_containers.py and test_integrators.py, installed beside the
unmodified reference in baseline/_ref by tools/install_reference.sh) run
with this package swapped in (tests/refswap.py):

* container mode -- respamd.containers.LinkedCells / DirectSum and the
  functional passes are the GPU versions, driven by the reference's own
  respa_run / verlet_run / equilibrate pass by pass;
* integrator mode -- respa_run / verlet_run / equilibrate are the
  device-resident loop too.

Plus respamd.integrators.respa_run itself with CudaLinkedCells against the
reference's CPU LinkedCells on the same system.  Skips when the reference
is not installed (it is not committed; numba comes with the image).
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "respamd_tests")


def _need_reference():
    if not os.path.isdir(os.path.join(REF, "respamd")) or not os.path.isdir(REF_TESTS):
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    try:
        import numba  # noqa: F401
    except ImportError:
        pytest.skip("numba (the reference's JIT) is not in this image")


def _env(mode):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO, os.path.join(REPO, "tests"),
                                         env.get("PYTHONPATH", "")])
    env["RB_SWAP"] = mode
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_respamd")
    return env


@pytest.mark.parametrize("mode", ["container", "integrator"])
def test_reference_test_suite_with_gpu_package(mode):
    _need_reference()
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refswap", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, os.path.join(REF_TESTS, "test_containers.py"),
           os.path.join(REF_TESTS, "test_integrators.py")]
    res = subprocess.run(cmd, env=_env(mode), cwd=REF_TESTS, capture_output=True, text=True,
                         timeout=1800)
    tail = "\n".join((res.stdout + res.stderr).splitlines()[-40:])
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and "failed" not in res.stdout.splitlines()[-1], tail


def test_reference_respa_run_drives_gpu_container():
    """respamd.integrators.respa_run (the reference's own loop) with
    CudaLinkedCells equals it with the reference's LinkedCells."""
    _need_reference()
    code = r"""
import numpy as np
from respamd import containers as rc, integrators as ri, model as rm
import paper_2507_11172_b200 as pkg

def system():
    s = pkg.systems.fcc_system(5, jitter=0.03, seed=41, temperature=1.0, vseed=42)
    r = rm.ParticleSystem.empty(s.n, s.box, periodic=True)
    r.positions[:] = s.positions
    r.velocities[:] = s.velocities
    return r

ff = rm.ForceField(epsilon=1.0, sigma=1.0, nu=0.2, cutoff=2.5)
a, b = system(), system()
ta = ri.respa_run(a, ff, pkg.CudaLinkedCells(), ri.RespaSchedule(0.002, 3, 30))
tb = ri.respa_run(b, ff, rc.LinkedCells(), ri.RespaSchedule(0.002, 3, 30))
dx = np.max(np.abs(a.positions - b.positions))
de = max(abs(x - y) / max(1.0, abs(y)) for x, y in zip(ta.total, tb.total))
print("DX", dx, "DE", de)
assert dx <= 1e-10 and de <= 1e-10
"""
    res = subprocess.run([sys.executable, "-c", code], env=_env("none"), capture_output=True,
                         text=True, timeout=1800)
    assert res.returncode == 0, (res.stdout + res.stderr)[-3000:]
