"""Device RDF: rb_distance_histogram against the reference's
own counts and curves (tests/golden/rdf.npz, made by
respamd.observables.rdf / _distance_histogram) and the bit-pinned oracle.
Counts are integers: bit-exact; g(r) repeats the reference's numpy
normalisation: equal to the last bit."""

import numpy as np
import pytest

from helpers import TEST_SEED, load_golden, random_positions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2507_11172_b200 as p
    from paper_2507_11172_b200 import _lib

    _lib.require_device()
    return p


def test_rdf_matches_reference(pkg):
    from paper_2507_11172_b200 import observables as ob

    g = load_golden("rdf.npz")
    for name in [str(n) for n in g["names"]]:
        box = g[f"{name}__box"]
        frames = []
        for i in range(int(g[f"{name}__frames"])):
            s = pkg.ParticleSystem.empty(len(g[f"{name}__frame{i}"]), box, periodic=True)
            s.positions[:] = g[f"{name}__frame{i}"]
            frames.append(s)
        r_max, bins = float(g[f"{name}__r_max"]), int(g[f"{name}__bins"])
        counts = None
        for s in frames:
            counts = ob.distance_histogram(s.positions, box, r_max, bins, counts)
        assert np.array_equal(counts.cpu().numpy(), g[f"{name}__counts"])
        curve = ob.rdf(frames, r_max=None if name == "cfg1" else r_max, bins=bins)
        assert np.array_equal(curve, g[f"{name}__curve"])


def test_distance_histogram_cfg2_against_oracle(pkg, oracle):
    from paper_2507_11172_b200 import observables as ob

    s = pkg.systems.CONFIGS["cfg2"].system()
    r_max = float(s.box.min()) / 2.0
    got = ob.distance_histogram(s.positions, s.box, r_max, 300).cpu().numpy()
    assert np.array_equal(got, oracle.distance_histogram(s.positions, s.box, r_max, 300))


def test_rdf_validation(pkg):
    from paper_2507_11172_b200 import observables as ob

    rng = np.random.default_rng(TEST_SEED)
    s = pkg.ParticleSystem.empty(50, (6.0, 6.0, 6.0), periodic=True)
    s.positions[:] = random_positions(rng, 50, (6.0,) * 3, True)
    with pytest.raises(pkg.ValidationError):
        ob.rdf([])
    with pytest.raises(pkg.ValidationError):
        ob.rdf([s], r_max=3.5)
    o = pkg.ParticleSystem.empty(50, (6.0, 6.0, 6.0), periodic=False)
    with pytest.raises(pkg.ValidationError):
        ob.rdf([o])
