"""GPU parity: the sm_100a path against the reference's golden vectors and
the CPU oracle on identical seeded inputs.

Tolerances (north star, BASELINE.json): per-spot |E_n|^2 within 1e-4
relative, wrapped phase within 1e-3 rad on pixels whose coherent sum is
not ill-conditioned (|S_p| >= 1e-3 * sum_n a_n), e and u
within 1e-3 absolute.  Determinism is checked bitwise.
"""

import math

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from conftest import load_solve, random_spots, wrap_diff

pytestmark = pytest.mark.gpu

PHASE_TOL = 1e-3
INTEN_RTOL = 1e-4
EU_ATOL = 1e-3
MASK_FRAC = 1e-3


def spots_of(d):
    return hs.SpotSet(x=d["x"], y=d["y"], z=d["z"], amplitude=d["a0"])


def masked_phase_check(pupil, spots, got, amps, thetas, idx=None, tab=None):
    """Compare wrapped phases on well-conditioned pixels; returns stats."""
    tab = tab or oracle.tables(pupil, spots.x, spots.y, spots.z)
    want, mag = oracle.superpose(pupil, tab, amps, thetas, want_mag=True)
    if idx is not None:
        want, mag = want[idx], mag[idx]
    ok = mag >= MASK_FRAC * float(np.sum(amps))
    d = wrap_diff(got, want)
    assert np.all(d[ok] <= PHASE_TOL), float(np.max(d[ok]))
    wmean = float(np.sum(d * mag) / np.sum(mag))
    assert wmean <= 1e-5, wmean
    assert ok.mean() >= 0.99, float(ok.mean())   # the mask drops < 1% of pixels
    return float(np.max(d[ok])), float(ok.mean())


# ----------------------------------------------------------------- kernels
def test_superpose_matches_golden(golden, golden_kernels, pupils):
    for case, pkey in golden["kernels"].items():
        g = lambda k: golden_kernels[f"{case}.{k}"]  # noqa: E731
        p = pupils[pkey]
        s = hs.SpotSet(x=g("x"), y=g("y"), z=g("z"), amplitude=np.ones(g("x").shape[0]))
        co = hs.SpotCoefficients(g("amp"), g("theta"))
        got = hs.superpose(p, s, co)
        tab = oracle.tables(p, s.x, s.y, s.z)
        want, mag = oracle.superpose(p, tab, co.amplitude, co.theta, want_mag=True)
        assert np.array_equal(want, g("superpose"))  # oracle pinned to the reference
        ok = mag >= MASK_FRAC * float(np.sum(co.amplitude))
        assert np.all(wrap_diff(got, want)[ok] <= PHASE_TOL)
        lo, hi = int(g("lo")), int(g("hi"))
        got_r = hs.superpose(p, s, co, (lo, hi))
        assert np.all(wrap_diff(got_r, g("superpose_range"))[ok[lo:hi]] <= PHASE_TOL)
        assert np.all((got >= -math.pi) & (got < math.pi))


def test_forward_matches_golden(golden, golden_kernels, pupils):
    for case, pkey in golden["kernels"].items():
        g = lambda k: golden_kernels[f"{case}.{k}"]  # noqa: E731
        p = pupils[pkey]
        s = hs.SpotSet(x=g("x"), y=g("y"), z=g("z"), amplitude=np.ones(g("x").shape[0]))
        holo = hs.Hologram(g("phase"), p)
        scale = p.sum_amplitude
        f = hs.forward_project(p, holo, s)
        assert np.all(np.abs(f - g("fields")) <= 1e-5 * np.abs(g("fields")) + 1e-6 * scale)
        lo, hi = int(g("lo")), int(g("hi"))
        fr = hs.forward_project(p, holo, s, (lo, hi), chunk=37)
        assert np.all(np.abs(fr - g("fields_range")) <= 1e-5 * np.abs(g("fields_range"))
                      + 1e-6 * scale)
        inten = hs.spot_intensities(p, holo, s)
        want = g("intensities")
        assert np.all(np.abs(inten - want) <= INTEN_RTOL * want + 1e-10)


def test_conjugate_spot_sums_all_power(pupils):
    p = pupils["p64u0"]
    spot = (2e-5, -1e-5, 5e-5)
    s = hs.SpotSet.from_points([spot])
    phase = hs.wrap_phase(hs.spot_phase(p, spot, (p.xs, p.ys)))
    field = hs.forward_project(p, hs.Hologram(phase, p), s)[0]
    m = p.active_count
    assert abs(field - m) <= 1e-6 * m
    rep = hs.quality_report(p, hs.Hologram(phase, p), s)
    assert abs(rep.efficiency - 1.0) <= 1e-5 and rep.uniformity == 1.0


def test_origin_spot_is_plain_sum(pupils, rng):
    p = pupils["p16g2"]
    phase = hs.wrap_phase(rng.uniform(-3, 3, p.active_count))
    s = hs.SpotSet.from_points([[0.0, 0.0, 0.0]])
    got = hs.forward_project(p, hs.Hologram(phase, p), s)[0]
    want = np.sum(p.amplitude * np.exp(-1j * phase))
    assert abs(got - want) <= 1e-6 * abs(want)


def test_superpose_conventions(pupils, rng):
    p = pupils["p8u1"]
    s = hs.SpotSet.from_points([[0.0, 0.0, 0.0]])
    frag = hs.superpose(p, s, hs.SpotCoefficients([1.0], [0.3]))
    assert np.all(np.abs(frag - 0.3) < 1e-6)
    s2 = hs.SpotSet.from_points([[1e-5, 0, 0], [0, 1e-5, 0]])
    frag = hs.superpose(p, s2, hs.SpotCoefficients([0.0, 0.0], [0.1, 2.0]))
    assert np.all(frag == 0.0)                   # arg(0) = 0
    frag = hs.superpose(p, s, hs.SpotCoefficients([1.0], [math.pi]))
    assert np.all(wrap_diff(frag, -math.pi) < 1e-6) and np.all(frag < math.pi)
    s3 = random_spots(rng, 3)
    th = np.round(rng.uniform(0, 6.2, 3) * 2**20) / 2**20
    amp = rng.uniform(0.3, 1.5, 3)
    a = hs.superpose(pupils["p16g2"], s3, hs.SpotCoefficients(amp, th))
    b = hs.superpose(pupils["p16g2"], s3, hs.SpotCoefficients(amp, th + 2 * math.pi))
    assert np.array_equal(a, b)                  # exact theta wrap


def test_validation_before_compute(pupils):
    p = pupils["p8u1"]
    s = hs.SpotSet.from_points([[0.0, 0.0, 0.0]])
    with pytest.raises(hs.InvalidParameterError):
        hs.superpose(p, s, hs.SpotCoefficients(np.ones(2), np.zeros(2)))
    with pytest.raises(hs.InvalidParameterError):
        hs.superpose(p, s, hs.SpotCoefficients([1.0], [0.0]), (0, p.active_count + 1))
    holo = hs.Hologram(np.zeros(p.active_count), p)
    with pytest.raises(hs.InvalidParameterError):
        hs.forward_project(p, holo, s, chunk=0)
    other = hs.build_pupil(8, illumination="uniform", seed=5)
    with pytest.raises(hs.GeometryMismatchError):
        hs.forward_project(other, holo, s)
    assert np.array_equal(hs.forward_project(p, holo, s, (3, 3)), np.zeros(1))
    assert hs.superpose(p, s, hs.SpotCoefficients([1.0], [0.0]), (2, 2)).shape == (0,)


# ------------------------------------------------------------------ solvers
SOLVES = ["wgs_p64", "cswgs_p48", "rs_p64", "cswgs_p64_i2", "cswgs_p64_c1", "wgs_grid36_256",
          "cswgs_grid36_256", "cfg1", "cfg2_rs", "cfg3_grid100", "cfg3_random"]


@pytest.mark.parametrize("name", SOLVES)
def test_solver_matches_reference(golden, pupils, name):
    meta = golden["solves"][name]
    d = load_solve(name)
    p = pupils[meta["pupil"]]
    s = spots_of(d)
    cfg = hs.SolverConfig(meta["algorithm"], iterations=meta["iterations"],
                          compression=meta["compression"], seed=meta["seed"])
    holo, trace = hs.solve(p, s, cfg)
    rep = hs.quality_report(p, holo, s)
    assert trace.operation_count == meta["ops"]
    assert [r.subset_size for r in trace.records] == list(d["sizes"])
    assert abs(rep.efficiency - meta["e"]) <= EU_ATOL
    assert abs(rep.uniformity - meta["u"]) <= EU_ATOL
    want = d["intensities"]
    assert np.all(np.abs(rep.intensities - want) <= INTEN_RTOL * want), \
        float(np.max(np.abs(rep.intensities - want) / want))
    if trace.records:
        mags = np.array([r.magnitudes for r in trace.records])
        assert np.all(np.abs(mags - d["mags"]) <= 1e-4 * d["mags"])
        w = np.array([r.weights for r in trace.records])
        assert np.all(np.abs(w - d["weights"]) <= 1e-4 * d["weights"])
    # final phase on the golden subsample, masked by the oracle's |S_p|
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, meta["algorithm"], meta["iterations"],
                     meta["compression"], meta["seed"])
    idx = d["phase_idx"]
    assert np.array_equal(r["phase"][idx], d["phase"])
    masked_phase_check(p, s, holo.phase[idx], r["amps"], r["thetas"], idx, r["tables"])
    # the solver's fused estimate (last pass, no re-projection) agrees
    fused = trace.quality
    assert abs(fused.efficiency - rep.efficiency) <= 1e-5
    assert abs(fused.uniformity - rep.uniformity) <= 1e-4
    assert abs(fused.efficiency - meta["e"]) <= EU_ATOL and abs(fused.uniformity - meta["u"]) <= EU_ATOL


def test_quality_gate_grid100(golden, pupils):
    """Paper headline case: 1152^2, N=100 grid, c=1/16, I=20 -> e, u > 0.9."""
    p = pupils["p1152g0"]
    s = hs.named_spots("grid100")
    holo, _ = hs.cswgs(p, s, iterations=20, compression=1 / 16, seed=0)
    rep = hs.quality_report(p, holo, s)
    assert rep.efficiency > 0.9 and rep.uniformity > 0.9


def test_compression_golden_table(golden, pupils):
    """Reference demo table (demos/output/compression_runs.csv rows 2-41)."""
    p = pupils["p256u0"]
    frames = [hs.SpotSet(x=f["x"], y=f["y"], z=f["z"], amplitude=f["a0"])
              for f in golden["grid36_frames"]]
    worst = {}
    for row in golden["compression_runs"]:
        s = frames[row["seed"]]
        cfg = hs.SolverConfig(row["algorithm"], iterations=row["iterations"],
                              compression=row["c"], seed=row["seed"])
        holo, trace = hs.solve(p, s, cfg)
        assert trace.operation_count == row["ops"]
        rep = hs.quality_report(p, holo, s)
        err = max(abs(rep.efficiency - row["e"]), abs(rep.uniformity - row["u"]))
        worst[row["iterations"]] = max(worst.get(row["iterations"], 0.0), err)
        assert err <= EU_ATOL, (row, rep.efficiency, rep.uniformity)
    print("worst |de|,|du| by iteration count:", worst)


# -------------------------------------------------------------- determinism
def test_bitwise_repeatable_and_batch_invariant(pupils):
    p = pupils["p512g0"]
    sets = [hs.random_foci(10, 100 + k) for k in range(3)]
    cfg = hs.SolverConfig("cswgs", iterations=10, compression=1 / 8, seed=0)
    solo = [hs.solve(p, s, hs.SolverConfig("cswgs", 10, 1 / 8, seed=k))[0].phase
            for k, s in enumerate(sets)]
    again = hs.solve(p, sets[0], hs.SolverConfig("cswgs", 10, 1 / 8, seed=0))[0].phase
    assert np.array_equal(solo[0], again)
    batch = hs.solve_batch(p, sets, cfg, seeds=[0, 1, 2])
    for k in range(3):
        assert np.array_equal(batch[k][0].phase, solo[k])


def test_wgs_equals_cswgs_c1(pupils, rng):
    p = pupils["p64u0"]
    s = random_spots(rng, 4)
    a, ta = hs.wgs(p, s, iterations=6, seed=3)
    b, tb = hs.cswgs(p, s, iterations=6, compression=1.0, seed=3)
    assert np.array_equal(a.phase, b.phase)
    assert ta.operation_count == tb.operation_count


def test_trace_weight_identity(pupils, rng):
    """sum_n (w_j/w_{j-1}) |E_n| = N mean|E| (reference test_solvers.py)."""
    p = pupils["p64u0"]
    s = random_spots(rng, 4)
    _, trace = hs.wgs(p, s, iterations=8, seed=9)
    prev = np.ones(s.count)
    for rec in trace.records:
        lhs = float(np.sum(rec.weights / prev * rec.magnitudes))
        rhs = s.count * float(np.mean(rec.magnitudes))
        assert abs(lhs - rhs) <= 1e-12 * abs(rhs)
        prev = rec.weights


def test_underdetermined_warning_and_errors(pupils, rng):
    p = pupils["p64u0"]
    s = random_spots(rng, 40)
    with pytest.warns(RuntimeWarning, match="underdetermined"):
        hs.cswgs(p, s, iterations=4, compression=1e-3, seed=0)
    with pytest.raises(hs.InvalidParameterError):
        hs.cswgs(p, s, iterations=1, compression=0.5)
    with pytest.raises(hs.InvalidParameterError):
        hs.wgs(p, s, iterations=0)


def test_large_spot_count_path(pupils, rng):
    """N > 512 uses the 32-lane x 32-spot fp32 variant; compare with the oracle.
    (5 pixels per spot: precision "auto" would run fp64, so fp32 is forced.)"""
    p = pupils["p64u0"]
    s = hs.SpotSet(x=rng.uniform(-1e-4, 1e-4, 600), y=rng.uniform(-1e-4, 1e-4, 600),
                   z=rng.uniform(-5e-5, 5e-5, 600), amplitude=np.ones(600))
    with hs.precision("fp32"):
        holo, trace = hs.wgs(p, s, iterations=3, seed=1)
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, "wgs", 3, seed=1)
    mags = np.array([rec.magnitudes for rec in trace.records])
    assert np.all(np.abs(mags - r["mags"]) <= 1e-4 * r["mags"])
    masked_phase_check(p, s, holo.phase, r["amps"], r["thetas"], tab=r["tables"])


def test_pipelined_host_api_matches_batch(pupils):
    """hs_solve_host_async: back-to-back calls with double-buffered outputs
    return the same phases / e / u as solve_batch."""
    import ctypes
    import math
    from paper_2003_05293_b200 import _lib
    p = pupils["p512g0"]
    lib = _lib.load()
    plan = _lib.Plan(p)
    cfg = hs.SolverConfig("cswgs", iterations=6, compression=1 / 8, seed=0)
    sub = math.ceil(p.active_count / 8)
    calls, keep = [], []

    def pinned(arr):
        ptr = lib.hs_host_alloc(arr.nbytes)
        view = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)),
                                     shape=arr.shape)
        view[...] = arr
        keep.append(ptr)
        return ptr, view

    for k in range(3):
        sets = [hs.random_foci(10, 50 + 2 * k + b) for b in range(2)]
        th = np.stack([np.random.default_rng(10 * k + b).random(10) * 2 * math.pi
                       for b in range(2)])
        bufs = [pinned(np.stack([getattr(s, f) for s in sets])) for f in ("x", "y", "z", "amplitude")]
        thb = pinned(th)
        ph = pinned(np.zeros((2, p.active_count)))
        e = pinned(np.zeros(2))
        u = pinned(np.zeros(2))
        _lib.check(lib.hs_solve_host_async(plan.handle, _lib.ALG_CSWGS, 6, sub, 2, 10,
                                           *[b[0] for b in bufs], thb[0], ph[0], e[0], u[0]))
        calls.append((sets, [10 * k, 10 * k + 1], ph[1], e[1], u[1]))
    plan.sync()
    for sets, seeds, ph, e, u in calls:
        want = hs.solve_batch(p, sets, cfg, seeds=seeds)
        for b in range(2):
            assert np.array_equal(ph[b], want[b][0].phase)
            assert e[b] == want[b][1].quality.efficiency and u[b] == want[b][1].quality.uniformity
    for ptr in keep:
        lib.hs_host_free(ptr)


def test_unlit_pupil_semantics():
    """sum_amplitude == 0 (a gaussian waist far below the pixel pitch on an
    even grid): RS still returns a hologram, WGS / CS-WGS raise
    DegenerateFieldError on the all-zero fields (solvers.py:117-119) and the
    metrics raise ZeroIlluminationError (metrics.py:37-38), as the reference."""
    p = hs.build_pupil(16, illumination="gaussian", waist=1e-9, seed=0)
    assert p.sum_amplitude == 0.0
    s = hs.SpotSet.from_points([[1e-5, 0.0, 0.0], [0.0, 2e-5, 1e-5]])
    holo, trace = hs.rs(p, s, seed=0)
    assert np.all(np.isfinite(holo.phase)) and trace.quality is None
    with pytest.raises(hs.DegenerateFieldError):
        hs.wgs(p, s, iterations=3)
    with pytest.raises(hs.DegenerateFieldError):
        hs.cswgs(p, s, iterations=4, compression=0.5)
    with pytest.raises(hs.ZeroIlluminationError):
        hs.quality_report(p, holo, s)
