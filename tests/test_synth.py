"""The seeded input generator (synth/): known answers, shard invariance, recipe structure."""
import math

import numpy as np

import synth


def test_philox_known_answers():
    """Philox4x32-10 known-answer vectors (Salmon et al. SC'11, Random123 kat_vectors)."""
    assert synth.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert synth.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E,
                                                                0xA20BC7C6, 0x6D5451FD]
    assert synth.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                        [0xA4093822, 0x299F31D0]) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                      0x24126EA1]


def test_transcendentals_accuracy():
    lib = synth._load_cpu()
    for x in np.geomspace(1e-7, 1.0, 97):
        assert abs(lib.synth_log(float(x)) - math.log(x)) < 1e-13 * max(1, abs(math.log(x)))
    for u in np.arange(0, 1, 1 / 4096):
        assert abs(lib.synth_cos2pi(float(u)) - math.cos(2 * math.pi * u)) < 1e-13


def test_normal_moments():
    z = np.array([synth.normal(0, 3, i) for i in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1) < 0.02


def test_shard_invariance_and_determinism():
    cfg = synth.C3.scaled(97, 301, 7, 7)
    full = synth.x_full(cfg)
    parts = [synth.x_rows(cfg, b, min(25, cfg.m - b)) for b in range(0, cfg.m, 25)]
    assert np.array_equal(np.vstack(parts), full)
    assert np.array_equal(synth.x_full(cfg), full)


def test_recipe_structure():
    x1 = synth.x_full(synth.C1)
    assert x1.shape == (200, 100) and x1.min() > 0
    x4 = synth.x_full(synth.C4)
    nz = x4[x4 > 0]
    assert abs(nz.size / x4.size - 0.045) < 0.002
    frac = np.array([(nz == c).mean() for c in range(1, 6)])
    assert np.allclose(frac, [0.06, 0.11, 0.26, 0.35, 0.22], atol=0.01)
    x2 = synth.x_full(synth.C2)
    assert x2.min() >= 0 and x2.max() <= 1 and 0.1 < x2.mean() < 0.5
    x3 = synth.x_full(synth.C3)
    assert x3.min() > 0
