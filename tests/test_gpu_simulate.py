"""Far-field renderer on the GPU (mirrors pkg/tests/test_simulate.py)."""

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from conftest import random_spots

pytestmark = pytest.mark.gpu


def probe_oracle(pupil, phase, pts):
    tab = oracle.tables(pupil, pts[:, 0], pts[:, 1], pts[:, 2])
    f = oracle.forward(pupil, tab, phase)
    return (f.real ** 2 + f.imag ** 2) / pupil.sum_amplitude ** 2


def test_peak_at_commanded_spot(pupils):
    p = pupils["p64u0"]
    spot = (2e-5, -1e-5, 0.0)
    holo, _ = hs.rs(p, hs.SpotSet.from_points([spot]), seed=0)
    img = hs.render_plane(p, holo, window=8e-5, resolution=41)
    iy, ix = np.unravel_index(np.argmax(img.intensity), img.intensity.shape)
    xs = np.linspace(-4e-5, 4e-5, 41)
    assert abs(xs[ix] - spot[0]) <= 2.1e-6 and abs(xs[iy] - spot[1]) <= 2.1e-6


def test_defocus_drops_peak(pupils):
    p = pupils["p64u0"]
    holo, _ = hs.rs(p, hs.SpotSet.from_points([(1e-5, 0.0, 0.0)]), seed=0)
    sharp = hs.render_plane(p, holo, window=6e-5, resolution=31, z=0.0)
    blurred = hs.render_plane(p, holo, window=6e-5, resolution=31, z=2e-3)
    assert blurred.intensity.max() < 0.5 * sharp.intensity.max()


def test_matches_probe_oracle(pupils, rng):
    p = pupils["p16g2"]
    phase = hs.wrap_phase(rng.uniform(-3, 3, p.active_count))
    img = hs.render_plane(p, hs.Hologram(phase, p), window=1e-4, resolution=16, z=3e-5)
    xs = np.linspace(-5e-5, 5e-5, 16)
    pts = np.array([[x, y, 3e-5] for y in xs for x in xs])
    want = probe_oracle(p, phase, pts).reshape(16, 16)
    assert np.all(np.abs(img.intensity - want) <= 1e-4 * want + 1e-9 * want.max())


def test_large_render_chunks_match_oracle(pupils, rng):
    """> 1024 probes: several probe chunks through the 32-lane variant."""
    p = pupils["p48g2"]
    phase = hs.wrap_phase(rng.uniform(-3, 3, p.active_count))
    img = hs.render_plane(p, hs.Hologram(phase, p), window=2e-4, resolution=(50, 30), z=-1e-5)
    assert img.intensity.shape == (30, 50) and img.width == 50 and img.height == 30
    xs, ys = np.linspace(-1e-4, 1e-4, 50), np.linspace(-1e-4, 1e-4, 30)
    pts = np.array([[x, y, -1e-5] for y in ys for x in xs])
    want = probe_oracle(p, phase, pts).reshape(30, 50)
    assert np.all(np.abs(img.intensity - want) <= 1e-4 * want + 1e-9 * want.max())


def test_probe_at_spot_equals_metric(pupils, rng):
    p = pupils["p64u0"]
    spots = random_spots(rng, 3)
    holo, _ = hs.wgs(p, spots, iterations=4, seed=1)
    inten = hs.spot_intensities(p, holo, spots)
    probed = hs.probe_intensities(p, holo, spots.points())
    assert np.array_equal(inten, probed)


def test_probe_on_spot_bitwise_any_count_fp64(pupils, rng):
    """fp64 passes: the per-spot sums do not depend on the spot count, so a
    probe batch of a different size reproduces spot_intensities bit for bit."""
    p = pupils["p64u0"]
    spots = random_spots(rng, 3)
    with hs.precision("fp64"):
        holo, _ = hs.wgs(p, spots, iterations=4, seed=1)
        inten = hs.spot_intensities(p, holo, spots)
        extra = np.concatenate([spots.points(), rng.uniform(-5e-5, 5e-5, (40, 3))])
        probed = hs.probe_intensities(p, holo, extra)
    assert np.array_equal(inten, probed[:3])


def test_two_photon_is_square(pupils, rng):
    p = pupils["p64u0"]
    holo, _ = hs.rs(p, random_spots(rng, 2), seed=0)
    lin = hs.render_plane(p, holo, window=5e-5, resolution=11)
    tp = hs.render_plane(p, holo, window=5e-5, resolution=11, exposure="two_photon")
    assert np.array_equal(tp.intensity, lin.intensity * lin.intensity)
