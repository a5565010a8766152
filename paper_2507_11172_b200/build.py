"""In-tree build of the sm_100a shared library (the C-ABI of include/respa_b200.h).

    python -m paper_2507_11172_b200.build [--force] [--verbose]

Compiles every ``csrc/*.cu`` with nvcc for ``sm_100a`` only into
``paper_2507_11172_b200/librespa_b200.so`` (static cudart, so the library
loads without a GPU and carries no runtime-version coupling to torch).
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_NAME = "librespa_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--cudart", "static", "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def _deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
        os.path.join(REPO, "include", "respa_b200.h"), os.path.abspath(__file__)]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: the sm_100a library cannot be built")
    return path


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: str = None) -> str:
    target = out or LIB_PATH
    if not force and out is None and up_to_date():
        return LIB_PATH
    tmp = target + ".tmp"
    cmd = [nvcc(), *ARCH_FLAGS, *NVCC_FLAGS, "-I", os.path.join(REPO, "include")]
    cmd += os.environ.get("RB_NVCC_EXTRA", "").split()  # tuning experiments only
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += ["-o", tmp, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
