"""Reference API details on the device path: SpotTables arrays and
``tables=`` (kernels.py:61-76, 177-246), the host-driven ``wgs_step``
(solvers.py:132-163) and the device weight update's degeneracy semantics
(rebalance_weights, solvers.py:104-129; reference tests
pkg/tests/test_solvers.py:58-66, 221-224)."""

import ctypes
import math

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import _lib
from conftest import random_spots

pytestmark = pytest.mark.gpu


def test_spot_tables_arrays_match_reference(golden, golden_kernels, pupils):
    """spot_tables exposes gx_re/gx_im/gy_re/gy_im like the reference; the
    device builds them in fp64 (arguments in the reference's order), equal to
    the reference's tables up to libm last bits."""
    for case, pkey in golden["kernels"].items():
        g = lambda k: golden_kernels[f"{case}.{k}"]  # noqa: E731
        p = pupils[pkey]
        s = hs.SpotSet(x=g("x"), y=g("y"), z=g("z"), amplitude=np.ones(g("x").shape[0]))
        t = hs.spot_tables(p, s)
        assert t.count == s.count
        for k in ("gx_re", "gx_im", "gy_re", "gy_im"):
            arr = getattr(t, k)
            assert arr.shape == (p.side_px, s.count) and arr.dtype == np.float64
            assert not arr.flags.writeable
            assert np.max(np.abs(arr - g(k))) <= 4e-16, (case, k)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_caller_tables_are_used(pupils, rng, prec):
    """tables= is used as given (the reference never re-derives it from the
    spots): tables of spot set A passed with spot set B reproduce A's
    superposition and projection."""
    p = pupils["p64u0"]
    a, b = random_spots(rng, 5), random_spots(rng, 5)
    co = hs.SpotCoefficients(rng.uniform(0.3, 1.5, 5), rng.uniform(-3, 3, 5))
    with hs.precision(prec):
        ta = hs.spot_tables(p, a)
        want = hs.superpose(p, a, co)
        tab_a = hs.SpotTables(ta.gx_re, ta.gx_im, ta.gy_re, ta.gy_im, 5)
        got = hs.superpose(p, b, co, tables=tab_a)
        assert np.array_equal(got, want)
        holo = hs.Hologram(want, p)
        fa = hs.forward_project(p, holo, a)
        fb = hs.forward_project(p, holo, b, tables=tab_a)
        assert np.array_equal(fa, fb)
        # without tables= the plan goes back to B's own tables
        assert not np.array_equal(hs.forward_project(p, holo, b), fa)
        rep = hs.quality_report(p, holo, b, tables=tab_a)
        assert np.array_equal(rep.intensities, hs.spot_intensities(p, holo, a))
    with pytest.raises(hs.InvalidParameterError):
        hs.superpose(p, random_spots(rng, 4), hs.SpotCoefficients(np.ones(4), np.zeros(4)),
                     tables=tab_a)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_wgs_step_matches_oracle(pupils, rng, prec):
    """The host-driven iteration (device passes + host update) follows the
    reference schedule: five WGS steps equal the oracle's trace."""
    p = pupils["p64u0"]
    s = random_spots(rng, 4)
    n = s.count
    theta = np.random.default_rng(3).random(n) * (2.0 * math.pi)
    with hs.precision(prec):
        tab = hs.spot_tables(p, s)
        frag = hs.superpose(p, s, hs.SpotCoefficients(s.amplitude, theta), tables=tab)
        state = hs.WgsState(weights=np.ones(n), amplitudes=s.amplitude.copy(), thetas=theta,
                            hologram=hs.Hologram(frag, p))
        mags, ws = [], []
        for _ in range(5):
            state, m = hs.wgs_step(p, s, state, tables=tab)
            mags.append(m)
            ws.append(state.weights)
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, "wgs", 5, 1.0, 3)
    tol = 1e-9 if prec == "fp64" else 1e-4
    assert np.all(np.abs(np.array(mags) - r["mags"]) <= tol * r["mags"])
    assert np.all(np.abs(np.array(ws) - r["weights"]) <= tol * r["weights"])
    # and the device solve of the same run
    _, trace = hs.wgs(p, s, iterations=5, seed=3)
    assert np.allclose([x.magnitudes for x in trace.records], mags, rtol=1e-4, atol=0)


def _device_update(w, fields):
    lib = _lib.load()
    n = len(w)
    w = np.ascontiguousarray(w, dtype=np.float64)
    f = np.empty(2 * n)
    f[0::2], f[1::2] = np.real(fields), np.imag(fields)
    w_out, m_out = np.empty(n), np.empty(n)
    st, dg = ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.hs_debug_update(n, _lib.ptr(w), _lib.ptr(f), _lib.ptr(w_out), _lib.ptr(m_out),
                                   ctypes.byref(st), ctypes.byref(dg)))
    return w_out, m_out, st.value, bool(dg.value)


def test_device_update_semantics():
    # equal magnitudes keep the weights; (2, 1) -> (0.75, 1.5) exactly
    w, m, st, dg = _device_update([0.7, 0.7], [3.0, 3.0j])
    assert st == 0 and not dg and np.array_equal(w, [0.7, 0.7])
    w, m, st, dg = _device_update([1.0, 1.0], [2.0, 1.0])
    assert st == 0 and np.array_equal(w, [0.75, 1.5])
    # a zero magnitude is floored to min positive * 1e-6 and flagged
    w, m, st, dg = _device_update([1.0, 1.0], [0.0, 2.0j])
    assert st == 0 and dg and m[0] == 2.0 * hs.solvers.DEGENERACY_FLOOR and np.all(w > 0)
    want_w, want_m, want_flag = hs.rebalance_weights(np.ones(2), np.array([0.0, 2.0]))
    assert np.array_equal(w, want_w) and np.array_equal(m, want_m) and want_flag
    # all zero -> degenerate; overflow -> diverged (DegenerateFieldError both)
    _, _, st, _ = _device_update([1.0, 1.0], [0.0, 0.0])
    assert st == _lib.HS_EDEGENERATE
    _, _, st, _ = _device_update([1e308, 1.0], [1e-30, 1.0])
    assert st == _lib.HS_EDIVERGED
    # many spots: the host mirror of the reference update to the last bits
    # (device hypot and the fixed-order mean vs numpy's)
    rng = np.random.default_rng(5)
    f = rng.normal(size=300) + 1j * rng.normal(size=300)
    f[17] = 0.0
    w0 = rng.uniform(0.5, 2.0, 300)
    w, m, st, dg = _device_update(w0, f)
    hw, hm, hflag = hs.rebalance_weights(w0, np.hypot(f.real, f.imag))
    assert st == 0 and dg == hflag
    assert np.allclose(w, hw, rtol=1e-15, atol=0) and np.allclose(m, hm, rtol=1e-15, atol=0)
    assert m[17] > 0 and abs(m[17] - hm[17]) <= 1e-15 * hm[17]   # the floored magnitude
