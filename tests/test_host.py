"""Host-side logic of the drop-in API (no GPU needed).

Mirrors the reference unit tests for the pure-Python parts
(pkg/tests/test_optics.py, test_solvers.py, test_metrics.py).
"""

import hashlib
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import solvers
from conftest import GOLDEN


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ optics
def test_build_pupil_matches_reference(golden, pupils):
    for key, meta in golden["pupils"].items():
        p = pupils[key]
        assert p.active_count == meta["M"]
        assert p.sum_amplitude == meta["sum_amplitude"]
        assert sha(p.rows) == meta["sha_rows"]
        assert sha(p.cols) == meta["sha_cols"]
        assert sha(p.amplitude) == meta["sha_amp"]
        assert sha(p.permutation) == meta["sha_perm"]
        assert p.prism_coeff == meta["prism"] and p.lens_coeff == meta["lens"]
        path = os.path.join(GOLDEN, f"pupil_{key}.npz")
        if os.path.exists(path):
            d = np.load(path)
            assert np.array_equal(d["aperture"], p.aperture)


def test_pupil_validation():
    with pytest.raises(hs.InvalidParameterError):
        hs.build_pupil(1)
    with pytest.raises(hs.InvalidParameterError):
        hs.build_pupil(8, pitch=0)
    with pytest.raises(hs.InvalidParameterError):
        hs.build_pupil(8, illumination="laser")
    with pytest.raises(hs.InvalidParameterError):
        hs.build_pupil(8, illumination="gaussian", waist=-1)
    assert hs.build_pupil(8, illumination="uniform").waist is None


def test_pupil_arrays_readonly_and_image_roundtrip(pupils):
    p = pupils["p16g2"]
    with pytest.raises(ValueError):
        p.rows[0] = 3
    vals = np.arange(p.active_count, dtype=np.float64)
    img = p.image_from_storage(vals, fill=-1.0)
    assert np.array_equal(p.storage_from_image(img), vals)
    assert np.sum(img == -1.0) == 16 * 16 - p.active_count
    with pytest.raises(hs.InvalidParameterError):
        p.image_from_storage(vals[:-1])


def test_spotset_validation():
    with pytest.raises(hs.InvalidParameterError):
        hs.SpotSet(x=[], y=[], z=[], amplitude=[])
    with pytest.raises(hs.InvalidParameterError):
        hs.SpotSet(x=[0.0], y=[0.0, 1.0], z=[0.0], amplitude=[1.0])
    with pytest.raises(hs.InvalidParameterError):
        hs.SpotSet(x=[np.nan], y=[0.0], z=[0.0], amplitude=[1.0])
    with pytest.raises(hs.InvalidParameterError):
        hs.SpotSet(x=[0.0], y=[0.0], z=[0.0], amplitude=[0.0])
    s = hs.SpotSet.from_points([[1e-6, 2e-6, 3e-6]])
    assert s.count == 1 and np.array_equal(s.points(), [[1e-6, 2e-6, 3e-6]])


def test_hologram_validation(pupils):
    p = pupils["p8u1"]
    m = p.active_count
    with pytest.raises(hs.InvalidParameterError):
        hs.Hologram(np.zeros(m + 1), p)
    with pytest.raises(hs.InvalidParameterError):
        hs.Hologram(np.full(m, math.pi), p)
    with pytest.raises(hs.InvalidParameterError):
        hs.Hologram(np.full(m, np.inf), p)
    h = hs.Hologram(np.full(m, -math.pi), p)
    assert h.phase.flags.writeable is False


@settings(max_examples=200, deadline=None)
@given(st.floats(min_value=-1e6, max_value=1e6, allow_nan=False))
def test_wrap_phase_range_and_congruence(x):
    w = hs.wrap_phase(x)
    assert -math.pi <= w < math.pi
    assert abs(math.remainder(w - x, 2 * math.pi)) < 1e-6 * max(1.0, abs(x))


def test_wrap_phase_two_pi_shift_bitwise():
    x = np.round(np.linspace(-6, 6, 101) * 2**20) / 2**20
    assert np.array_equal(hs.wrap_phase(x), hs.wrap_phase(x + 2 * math.pi))


def test_phase_of_conventions():
    assert hs.phase_of(0.0, 0.0) == 0.0
    assert hs.phase_of(-1.0, 0.0) == -math.pi
    assert hs.phase_of(0.0, 1.0) == math.pi / 2


def test_compression_plan():
    p = hs.build_pupil(32, illumination="uniform")
    plan = hs.CompressionPlan.for_pupil(p, 0.3)
    assert plan.subset_size == math.ceil(0.3 * p.active_count)
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(hs.InvalidParameterError):
            hs.CompressionPlan.for_pupil(p, bad)


def test_spot_phase_formula(pupils):
    p = pupils["p16g2"]
    ph = hs.spot_phase(p, (1e-5, -2e-5, 3e-5), (p.xs, p.ys))
    want = p.prism_coeff * (1e-5 * p.xs - 2e-5 * p.ys) + p.lens_coeff * (p.xs**2 + p.ys**2) * 3e-5
    assert np.allclose(ph, want, rtol=1e-15, atol=0)


# --------------------------------------------------------------- workloads
def test_named_grids_match_reference(golden):
    for name in ("grid36", "grid100"):
        s = hs.named_spots(name)
        ref = golden[name]
        for k, v in (("x", s.x), ("y", s.y), ("z", s.z), ("a0", s.amplitude)):
            assert np.array_equal(v, np.array(ref[k])), (name, k)


def test_random_foci_match_golden():
    from conftest import load_solve
    d = load_solve("cfg3_random")
    s = hs.random_foci(100, 12345)
    assert np.array_equal(s.x, d["x"]) and np.array_equal(s.z, d["z"])


# ------------------------------------------------------------ solver host
def test_rebalance_known_answers():
    w, m, deg = hs.rebalance_weights(np.ones(2), np.array([2.0, 1.0]))
    assert np.allclose(w, [0.75, 1.5]) and not deg
    w, m, deg = hs.rebalance_weights(np.ones(3), np.array([0.0, 1.0, 2.0]))
    assert deg and m[0] == 1.0 * 1e-6
    with pytest.raises(hs.DegenerateFieldError):
        hs.rebalance_weights(np.ones(2), np.zeros(2))
    with pytest.raises(hs.DegenerateFieldError):
        hs.rebalance_weights(np.array([1e308, 1.0]), np.array([1e-300, 1.0]))


def test_predict_ops_and_budget():
    assert hs.predict_ops("rs", 100, 3) == 300
    assert hs.predict_ops("wgs", 100, 3, 7) == 2100
    assert hs.predict_ops("cswgs", 100, 3, 7, 0.3) == 600 + 30 * 3 * 5
    with pytest.raises(hs.InvalidParameterError):
        hs.predict_ops("gs", 1, 1)
    plan = hs.budget_controller("cswgs", 1000, 10, 5 * 1000 * 10, 1 / 16)
    assert plan.iterations == 2 + (3 * 1000 * 10) // (63 * 10)
    assert hs.budget_controller("wgs", 1000, 10, 10).over_budget
    with pytest.raises(hs.InvalidParameterError):
        hs.budget_controller("wgs", 1, 1, 0)


def test_window_sizes_and_golden_ops(golden):
    from conftest import load_solve
    for name, meta in golden["solves"].items():
        if meta["algorithm"] == "rs":
            continue
        d = load_solve(name)
        m = golden["pupils"][meta["pupil"]]["M"]
        sub = m if meta["algorithm"] == "wgs" else math.ceil(meta["compression"] * m)
        sizes = solvers.window_sizes(m, sub, meta["iterations"])
        assert sizes == list(d["sizes"])
        n = d["x"].shape[0]
        assert sum(sizes) * n == meta["ops"]
        assert hs.predict_ops(meta["algorithm"], m, n, meta["iterations"],
                              meta["compression"]) == meta["ops"]


def test_solver_config_validation():
    with pytest.raises(hs.InvalidParameterError):
        hs.SolverConfig("gs")
    with pytest.raises(hs.InvalidParameterError):
        hs.SolverConfig("wgs", iterations=0)
    with pytest.raises(hs.InvalidParameterError):
        hs.SolverConfig("cswgs", iterations=1)
    with pytest.raises(hs.InvalidParameterError):
        hs.SolverConfig("cswgs", iterations=4, compression=0.0)


def test_field_phases_conventions():
    f = np.array([0j, -1 + 0j, 1j, -1 - 0j])
    ph = solvers._field_phases(f)
    assert ph[0] == 0.0 and ph[1] == -math.pi and ph[2] == math.pi / 2


# ------------------------------------------------------------------ metrics
def test_metric_formulas():
    assert hs.efficiency([0.1, 0.2]) == pytest.approx(0.3)
    assert hs.uniformity([1.0, 1.0]) == 1.0
    assert hs.uniformity([1.0, 3.0]) == pytest.approx(0.5)
    with pytest.raises(hs.UndefinedUniformityError):
        hs.uniformity([0.0, 0.0])
    with pytest.raises(hs.UndefinedUniformityError):
        hs.efficiency([])
    s = hs.SpotSet.from_points([[0, 0, 0], [1e-6, 0, 0]], amplitude=[1.0, 2.0])
    assert np.allclose(hs.target_relative([1.0, 4.0], s), [1.0, 1.0])


# ------------------------------------------------------------ reduce_complex
def test_reduce_complex_matches_golden(golden):
    vals = np.load(os.path.join(GOLDEN, "reduce_values.npy"))
    for chunk, (re, im, n) in golden["reduce"].items():
        assert hs.reduce_complex(vals[:n], chunk=int(chunk)) == complex(re, im)
    assert hs.reduce_complex([]) == 0j
    assert hs.reduce_complex([1, 2, 3, 4], chunk=2) == 10
    with pytest.raises(hs.InvalidParameterError):
        hs.reduce_complex([1j], chunk=0)


# ---------------------------------------------------------------- renderer
def test_render_validation_before_device(pupils):
    p = pupils["p8u1"]
    holo = hs.Hologram(np.zeros(p.active_count), p)
    with pytest.raises(hs.InvalidParameterError):
        hs.render_plane(p, holo, window=1e-4, exposure="three_photon")
    with pytest.raises(hs.InvalidParameterError):
        hs.render_plane(p, holo, window=1e-4, resolution=0)
    with pytest.raises(hs.InvalidParameterError):
        hs.render_plane(p, holo, window=-1.0)
    with pytest.raises(hs.InvalidParameterError):
        hs.probe_intensities(p, holo, np.zeros((3, 2)))
    assert hs.probe_intensities(p, holo, np.zeros((0, 3))).shape == (0,)


# -------------------------------------------------------------------- LUT
def test_phase_lut_reference_behaviour(tmp_path):
    lut = hs.PhaseLut.default()
    assert lut.table[0] == -math.pi and lut.table[128] == 0.0
    assert int(lut.gray(math.pi - 1e-9)) == 0
    for p in np.linspace(-math.pi, math.pi - 1e-12, 997):
        assert abs(float(hs.wrap_phase(lut.phase(lut.gray(p)) - p))) <= math.pi / 256
    table = np.linspace(-math.pi, math.pi, 256, endpoint=False)[::-1]
    path = tmp_path / "lut.txt"
    path.write_text("\n".join(f"{v:.17g}" for v in table) + "\n")
    custom = hs.PhaseLut.from_file(path)
    assert custom.gray(np.array([table[3], table[77]])).tolist() == [3, 77]
    (tmp_path / "short.txt").write_text("0.0\n0.1\n")
    with pytest.raises(hs.InvalidParameterError):
        hs.PhaseLut.from_file(tmp_path / "short.txt")
