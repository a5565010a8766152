"""Shared test helpers (input generation only; no checking logic)."""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
TEST_SEED = 20240811  # the reference suite's rng seed (pkg/tests/conftest.py:42-44)


def random_positions(rng, n, box, periodic, min_sep=0.85):
    """Rejection-sampled positions with a minimum separation.

    Same draw sequence as the reference fixture make_random_system
    (pkg/tests/conftest.py:7-21), so a given rng state gives the same system.
    """
    box = np.asarray(box, dtype=np.float64)
    pos = np.zeros((n, 3))
    placed = 0
    guard2 = min_sep * min_sep
    while placed < n:
        cand = rng.uniform(0.0, box, size=3)
        d = pos[:placed] - cand
        if periodic:
            d -= box * np.floor(d / box + 0.5)
        if placed == 0 or np.min(np.sum(d * d, axis=1)) > guard2:
            pos[placed] = cand
            placed += 1
    return pos


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def normwise(got, ref):
    """max_i |dF_i| / max_i |F_i|."""
    got = np.asarray(got).reshape(-1, 3)
    ref = np.asarray(ref).reshape(-1, 3)
    scale = float(np.max(np.linalg.norm(ref, axis=1))) if ref.size else 0.0
    err = float(np.max(np.linalg.norm(got - ref, axis=1))) if ref.size else 0.0
    return err / scale if scale > 0 else err
