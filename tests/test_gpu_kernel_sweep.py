"""Kernel-variant sweep on the GPU against the CPU oracle.

The solver instantiates its pass kernels per spot count: the full-range
GEMM-tile kernel per SPT = ceil(n / 8) (1..16) and the slab window kernel
per NS = ceil(n / 16) (1..8).  Every variant is exercised here on small
pupils with CS-WGS (window passes + full passes) and compared with the
oracle (oracle/oracle.py, the bit-exact restatement of the reference
kernels) at the north-star tolerances, plus the multi-slab / multi-chunk
paths on a large pupil with a batch (slab re-staging inside a CTA).
"""

import math

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fp32_kernels():
    """These pupils hold few pixels per spot, where precision "auto" picks the
    fp64 passes; the sweep is about the fp32 kernel instantiations."""
    with hs.precision("fp32"):
        yield

EU_ATOL = 1e-3        # e, u absolute (north star)
INTEN_RTOL = 1e-4     # per-spot |E_n|^2 relative (north star)


def _check(pupil, spots, algorithm, iterations, compression, seed):
    holo, trace = hs.solve(pupil, spots, hs.SolverConfig(algorithm, iterations=iterations,
                                                         compression=compression, seed=seed))
    rep = hs.quality_report(pupil, holo, spots)
    r = oracle.solve(pupil, spots.x, spots.y, spots.z, spots.amplitude, algorithm, iterations,
                     compression, seed)
    e, u, inten, _ = oracle.quality(pupil, r["tables"], r["phase"], spots.amplitude)
    assert trace.operation_count == r["ops"]
    assert abs(rep.efficiency - e) <= EU_ATOL
    assert abs(rep.uniformity - u) <= EU_ATOL
    big = inten > 1e-6 * inten.max()   # relative check on spots that carry power
    assert np.all(np.abs(rep.intensities[big] - inten[big]) <= INTEN_RTOL * inten[big]), \
        float(np.max(np.abs(rep.intensities[big] - inten[big]) / inten[big]))
    mags = np.array([rec.magnitudes for rec in trace.records])
    want = np.array(r["mags"])
    assert np.all(np.abs(mags - want) <= 1e-4 * np.maximum(want, 1e-12 * want.max()))
    return holo


@pytest.mark.parametrize("n", [1, 5, 8, 9, 16, 17, 31, 40, 57, 64, 72, 88, 100, 111, 119, 128])
def test_spot_count_variants(n):
    """Every tile (SPT) and slab (NS) instantiation against the oracle."""
    p = hs.build_pupil(72, seed=3, waist=3e-4)
    s = hs.random_foci(n, 500 + n, xy=6e-5, z=3e-5)
    _check(p, s, "cswgs", 6, 0.25, seed=n)


@pytest.mark.parametrize("side,n", [(37, 40), (50, 48), (101, 64), (101, 120), (75, 33)])
def test_odd_sides(side, n):
    """Sides with side % 4 != 0: the scalar column paths and the clamped /
    zero-padded tail columns of the tcgen05 and slab kernels."""
    p = hs.build_pupil(side, seed=side, waist=side * 4e-6)
    s = hs.random_foci(n, 700 + side, xy=5e-5, z=2e-5)
    _check(p, s, "cswgs", 5, 0.5, seed=side)
    _check(p, s, "wgs", 3, 1.0, seed=side)


def test_multi_slab_window_lists():
    """np = 128 at side 256: the window lists span two column slabs."""
    p = hs.build_pupil(256, seed=1, waist=2e-3)
    s = hs.random_foci(128, 77, xy=8e-5, z=4e-5)
    _check(p, s, "cswgs", 5, 1 / 8, seed=2)


def test_batched_multi_slab_restaging_is_batch_invariant():
    """1152^2, N = 100, B = 16: CTAs stream several chunks and re-stage their
    gx slab when a chunk lies in the next slab, and the solve graph runs the
    two halves of the batch as parallel branches; results equal solo solves
    bit for bit and the oracle within tolerance."""
    p = hs.build_pupil(1152)
    sets = [hs.random_foci(100, 900 + k) for k in range(16)]
    cfg = hs.SolverConfig("cswgs", iterations=5, compression=1 / 16, seed=0)
    batch = hs.solve_batch(p, sets, cfg, seeds=list(range(16)))
    for k in (0, 7, 8, 15):
        solo, _ = hs.solve(p, sets[k], hs.SolverConfig("cswgs", 5, 1 / 16, seed=k))
        assert np.array_equal(batch[k][0].phase, solo.phase)
    holo = batch[7][0]
    rep = hs.quality_report(p, holo, sets[7])
    r = oracle.solve(p, sets[7].x, sets[7].y, sets[7].z, sets[7].amplitude, "cswgs", 5, 1 / 16, 7)
    e, u, _, _ = oracle.quality(p, r["tables"], r["phase"], sets[7].amplitude)
    assert abs(rep.efficiency - e) <= EU_ATOL and abs(rep.uniformity - u) <= EU_ATOL
    assert math.isfinite(rep.efficiency)
