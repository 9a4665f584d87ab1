"""Pin the CPU oracle (oracle/) against vectors produced by the reference.

The oracle restates the reference operation order, so every comparison here
is bitwise.  Fixtures: tests/golden/make_golden.py.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import load_solve


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_tables_superpose_forward_bitwise(golden, golden_kernels, pupils):
    for case, pkey in golden["kernels"].items():
        g = lambda k: golden_kernels[f"{case}.{k}"]  # noqa: E731
        p = pupils[pkey]
        tab = oracle.tables(p, g("x"), g("y"), g("z"))
        for name in ("gx_re", "gx_im", "gy_re", "gy_im"):
            assert np.array_equal(getattr(tab, name), g(name)), (case, name)
        assert np.array_equal(oracle.superpose(p, tab, g("amp"), g("theta")), g("superpose"))
        lo, hi = int(g("lo")), int(g("hi"))
        assert np.array_equal(oracle.superpose(p, tab, g("amp"), g("theta"), lo, hi),
                              g("superpose_range"))
        assert np.array_equal(oracle.forward(p, tab, g("phase")), g("fields"))
        assert np.array_equal(oracle.forward(p, tab, g("phase"), lo, hi, 37), g("fields_range"))


def test_tree_reduce_bitwise(golden):
    vals = np.load(__import__("conftest").GOLDEN + "/reduce_values.npy")
    for chunk, (re, im, n) in golden["reduce"].items():
        got = oracle.tree_reduce(vals[:n], int(chunk))
        assert got == complex(re, im)


@pytest.mark.parametrize("name", ["wgs_p64", "cswgs_p48", "rs_p64", "cswgs_p64_i2",
                                  "cswgs_p64_c1", "wgs_grid36_256", "cswgs_grid36_256",
                                  "cfg1"])
def test_solver_bitwise(golden, pupils, name):
    meta = golden["solves"][name]
    d = load_solve(name)
    p = pupils[meta["pupil"]]
    r = oracle.solve(p, d["x"], d["y"], d["z"], d["a0"], meta["algorithm"], meta["iterations"],
                     meta["compression"], meta["seed"])
    assert sha(r["phase"]) == meta["phase_sha"]
    assert r["ops"] == meta["ops"]
    assert list(r["sizes"]) == list(d["sizes"])
    assert np.array_equal(r["weights"], d["weights"])
    assert np.array_equal(r["mags"], d["mags"])
    e, u, inten, rel = oracle.quality(p, r["tables"], r["phase"], d["a0"])
    assert e == meta["e"] and u == meta["u"]
    assert np.array_equal(inten, d["intensities"])


def test_schedule_matches_trace_sizes(golden):
    """Window schedule restatement vs recorded subset sizes."""
    for name, meta in golden["solves"].items():
        if meta["algorithm"] == "rs":
            continue
        d = load_solve(name)
        m = golden["pupils"][meta["pupil"]]["M"]
        import math
        sub = m if meta["algorithm"] == "wgs" else math.ceil(meta["compression"] * m)
        sizes = [w[1] - w[0] for _, w in oracle.schedule(m, sub, meta["iterations"])]
        assert sizes == list(d["sizes"])
