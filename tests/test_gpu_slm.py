"""SLM rasters on the device vs the reference's PhaseLut / image layout."""

import math

import numpy as np
import pytest

import paper_2003_05293_b200 as hs
from conftest import random_spots

pytestmark = pytest.mark.gpu


def host_raster(pupil, phase, lut):
    gray = np.asarray(lut.gray(phase), dtype=np.uint8)
    return pupil.image_from_storage(gray, fill=np.uint8(0))


def test_fused_raster_matches_host_lut(pupils):
    p = pupils["p256u0"]
    sets = [hs.named_spots("grid36"), hs.random_foci(36, 3, xy=5e-5, z=2e-5)]
    cfg = hs.SolverConfig("cswgs", iterations=8, compression=0.25, seed=0)
    results, rasters = hs.solve_rasters(p, sets, cfg)
    lut = hs.PhaseLut.default()
    for (holo, _), img in zip(results, rasters):
        assert np.array_equal(img, host_raster(p, holo.phase, lut))
        assert np.array_equal(hs.slm_raster(p, holo), img)
        assert np.all(img[~p.aperture] == 0)
        back = lut.phase(p.storage_from_image(img))
        assert np.max(np.abs(hs.wrap_phase(back - holo.phase))) <= math.pi / 256


def test_rowrun_raster_large_n(pupils, rng):
    """N > 128 uses the row-run final pass; its fused raster must agree too."""
    p = pupils["p64u0"]
    s = random_spots(rng, 150)
    (res,), rasters = hs.solve_rasters(p, [s], hs.SolverConfig("wgs", iterations=3, seed=1))
    assert np.array_equal(rasters[0], host_raster(p, res[0].phase, hs.PhaseLut.default()))


def test_custom_lut_raster(pupils, rng):
    p = pupils["p64u0"]
    holo, _ = hs.wgs(p, random_spots(rng, 3), iterations=3, seed=2)
    table = np.linspace(-math.pi, math.pi, 256, endpoint=False)[::-1]
    lut = hs.PhaseLut(table)
    assert np.array_equal(hs.slm_raster(p, holo, lut), host_raster(p, holo.phase, lut))
