"""Precision modes of the pixel passes against the reference and the oracle.

* fp64 (csrc/hs_f64.cuh): every pixel product in fp64 like the reference's
  numba kernels, so it agrees with the reference's golden solves to ~1e-10
  (the only differences are summation order and libm last bits);
* auto (the product default): fp64 where a solve projects over fewer than
  512 pixels per spot.  These are the ill-conditioned cases where the fp32
  passes drift past the north-star tolerance over the iterations: 600
  random-amplitude spots on a 256^2 pupil, CS-WGS at n = 200 with c = 1/4
  (tools/accuracy_probe.py measured 5.3e-4 and 3.7e-4 in fp32);
* config 4 (BASELINE.json configs[3]): WGS, 1152^2, N = 1000, I = 30 against
  the reference's own run (tests/golden/make_cfg4.py), at the north-star
  tolerances -- 1042 pixels per spot, so the fp32 kernels run it.
"""

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from conftest import load_solve
from test_gpu_parity import EU_ATOL, INTEN_RTOL, SOLVES, masked_phase_check, spots_of

pytestmark = pytest.mark.gpu

TIGHT = 1e-9   # fp64 path vs the reference (relative / absolute / rad)


@pytest.mark.parametrize("name", SOLVES)
def test_fp64_matches_reference_tightly(golden, pupils, name):
    meta = golden["solves"][name]
    d = load_solve(name)
    p = pupils[meta["pupil"]]
    s = spots_of(d)
    cfg = hs.SolverConfig(meta["algorithm"], iterations=meta["iterations"],
                          compression=meta["compression"], seed=meta["seed"])
    with hs.precision("fp64"):
        holo, trace = hs.solve(p, s, cfg)
        rep = hs.quality_report(p, holo, s)
    assert hs._lib.plan_for(p).last_precision() == "fp64"
    assert trace.operation_count == meta["ops"]
    assert abs(rep.efficiency - meta["e"]) <= TIGHT and abs(rep.uniformity - meta["u"]) <= TIGHT
    want = d["intensities"]
    assert np.all(np.abs(rep.intensities - want) <= TIGHT * want), \
        float(np.max(np.abs(rep.intensities - want) / want))
    if trace.records:
        mags = np.array([r.magnitudes for r in trace.records])
        w = np.array([r.weights for r in trace.records])
        assert np.all(np.abs(mags - d["mags"]) <= TIGHT * d["mags"])
        assert np.all(np.abs(w - d["weights"]) <= TIGHT * d["weights"])
    # phases on the golden subsample: identical up to last-bit differences,
    # except where |S_p| is ill-conditioned
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, meta["algorithm"], meta["iterations"],
                     meta["compression"], meta["seed"])
    idx = d["phase_idx"]
    tab = r["tables"]
    _, mag = oracle.superpose(p, tab, r["amps"], r["thetas"], want_mag=True)
    ok = mag[idx] >= 1e-6 * float(np.sum(r["amps"]))
    dphi = np.abs(np.mod(holo.phase[idx] - d["phase"] + np.pi, 2 * np.pi) - np.pi)
    assert np.all(dphi[ok] <= TIGHT), float(np.max(dphi[ok]))


def _rand_spots(n, seed, xy=1e-4, z=5e-5, unit=False):
    rng = np.random.default_rng(seed)
    amp = np.ones(n) if unit else rng.uniform(0.5, 1.5, n)
    return hs.SpotSet(x=rng.uniform(-xy, xy, n), y=rng.uniform(-xy, xy, n),
                      z=rng.uniform(-z, z, n), amplitude=amp)


# (algorithm, n, iterations, compression): the cases tools/accuracy_probe.py
# measured past 1e-4 in fp32 (first two), and their neighbours
ILL = [("wgs", 600, 3, 1.0), ("cswgs", 200, 4, 0.25), ("wgs", 200, 3, 1.0),
       ("cswgs", 120, 4, 0.25)]


@pytest.mark.parametrize("alg,n,iters,c", ILL)
def test_auto_precision_ill_conditioned(pupils, alg, n, iters, c):
    p = pupils["p256u0"]
    s = _rand_spots(n, 1000 + n)
    holo, trace = hs.solve(p, s, hs.SolverConfig(alg, iterations=iters, compression=c, seed=7))
    assert hs._lib.plan_for(p).last_precision() == "fp64"
    rep = hs.quality_report(p, holo, s)
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, alg, iters, c, 7)
    e, u, inten, _ = oracle.quality(p, r["tables"], r["phase"], s.amplitude)
    mags = np.array([x.magnitudes for x in trace.records])
    w = np.array([x.weights for x in trace.records])
    assert np.all(np.abs(mags - r["mags"]) <= INTEN_RTOL * r["mags"])
    assert np.all(np.abs(w - r["weights"]) <= INTEN_RTOL * r["weights"])
    assert np.all(np.abs(rep.intensities - inten) <= INTEN_RTOL * inten), \
        float(np.max(np.abs(rep.intensities - inten) / inten))
    assert abs(rep.efficiency - e) <= EU_ATOL and abs(rep.uniformity - u) <= EU_ATOL
    masked_phase_check(p, s, holo.phase, r["amps"], r["thetas"], tab=r["tables"])


def test_spot_count_above_fp32_kernels(pupils):
    """n = 1500 > 1024: fp64 passes (any spot count up to hs_max_spots)."""
    p = pupils["p512g0"]
    s = _rand_spots(1500, 31, xy=1.5e-4)
    holo, trace = hs.wgs(p, s, iterations=3, seed=2)
    assert hs._lib.plan_for(p).last_precision() == "fp64"
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, "wgs", 3, 1.0, 2)
    mags = np.array([x.magnitudes for x in trace.records])
    assert np.all(np.abs(mags - r["mags"]) <= 1e-9 * r["mags"])
    with pytest.raises(hs.InvalidParameterError):
        with hs.precision("fp32"):
            hs.wgs(p, s, iterations=2, seed=2)


def test_fp64_bitwise_repeatable_and_batch_invariant(pupils):
    p = pupils["p256u0"]
    sets = [_rand_spots(40, 300 + k) for k in range(3)]
    cfg = hs.SolverConfig("cswgs", iterations=6, compression=1 / 8, seed=0)
    with hs.precision("fp64"):
        solo = [hs.solve(p, s, hs.SolverConfig("cswgs", 6, 1 / 8, seed=k))[0].phase
                for k, s in enumerate(sets)]
        again = hs.solve(p, sets[0], hs.SolverConfig("cswgs", 6, 1 / 8, seed=0))[0].phase
        batch = hs.solve_batch(p, sets, cfg, seeds=[0, 1, 2])
    assert np.array_equal(solo[0], again)
    for k in range(3):
        assert np.array_equal(batch[k][0].phase, solo[k])


def test_precision_modes_validated():
    with pytest.raises(hs.InvalidParameterError):
        hs.set_precision("fp16")
    assert hs.get_precision() == "auto"
    with hs.precision("fp32"):
        assert hs.get_precision() == "fp32"
    assert hs.get_precision() == "auto"


def test_config4_matches_reference(pupils):
    """BASELINE configs[3] on the 1152^2 stand-in: WGS, N = 1000 random foci
    (spot seed 4, xy +-150 um, z +-50 um), I = 30, against the reference run
    (tests/golden/solve_cfg4_wgs1000.npz) at the north-star tolerances."""
    d = load_solve("cfg4_wgs1000")
    p = pupils["p1152g0"]
    s = spots_of(d)
    holo, trace = hs.wgs(p, s, iterations=30, seed=0)
    assert hs._lib.plan_for(p).last_precision() == "fp32"
    rep = hs.quality_report(p, holo, s)
    mags = np.array([x.magnitudes for x in trace.records])
    w = np.array([x.weights for x in trace.records])
    assert np.all(np.abs(mags - d["mags"]) <= INTEN_RTOL * d["mags"]), \
        float(np.max(np.abs(mags - d["mags"]) / d["mags"]))
    assert np.all(np.abs(w - d["weights"]) <= INTEN_RTOL * d["weights"])
    assert np.all(np.abs(rep.intensities - d["intensities"]) <= INTEN_RTOL * d["intensities"])
    assert abs(rep.efficiency - float(d["e"])) <= EU_ATOL
    assert abs(rep.uniformity - float(d["u"])) <= EU_ATOL
    # the fused estimate of the last pass
    assert abs(trace.quality.efficiency - float(d["e"])) <= EU_ATOL
    # final phase on the golden subsample, masked by the reference's |S_p|
    idx = d["phase_idx"]
    ok = d["s_mag"] >= 1e-3 * float(np.sum(d["amps"]))
    dphi = np.abs(np.mod(holo.phase[idx] - d["phase"] + np.pi, 2 * np.pi) - np.pi)
    assert np.all(dphi[ok] <= 1e-3), float(np.max(dphi[ok]))
    assert float(np.sum(dphi * d["s_mag"]) / np.sum(d["s_mag"])) <= 1e-5
