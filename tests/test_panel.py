"""Rectangular full panels (``build_panel``, e.g. the paper's 1920 x 1152
SLM) -- host geometry and the oracle, on CPU.

The reference only builds circular apertures (optics.py:150-214); its
kernels and solvers read nothing but the Pupil's storage-order arrays, so
``tests/golden/make_panel.py`` runs the reference's own solvers on our panel
geometry.  The oracle must reproduce those runs bit for bit, as it does for
the circular golden cases (test_oracle_golden.py).
"""

import os

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from paper_2003_05293_b200.errors import InvalidParameterError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "panel.npz")
CASES = ["wgs_40x24", "cswgs_64x36", "rs_96x64", "cswgs_96x64", "cswgs_320x192"]


def panel_case(name):
    g = np.load(GOLDEN)
    d = {k.split(".", 1)[1]: g[k] for k in g.files if k.startswith(name + ".")}
    waist = float(d["waist"])
    ill = dict(illumination="uniform") if waist < 0 else dict(illumination="gaussian", waist=waist)
    p = hs.build_panel(int(d["w"]), int(d["h"]), seed=7, **ill)
    s = hs.SpotSet(x=d["x"], y=d["y"], z=d["z"], amplitude=d["a0"])
    return p, s, d


def test_panel_geometry():
    p = hs.build_panel(1920, 1152)
    assert p.panel == (1152, 1920) and p.side_px == 1920
    assert p.active_count == 1920 * 1152
    assert (p.rows.min(), p.rows.max(), p.cols.min(), p.cols.max()) == (384, 1535, 0, 1919)
    # centred: coordinates symmetric about the panel centre, same rule as build_pupil
    assert p.xs.min() == -p.xs.max() and p.ys.min() == -p.ys.max()
    assert np.array_equal(p.xs, (p.cols - 959.5) * 9.2e-6)
    # seeded permutation of the row-major panel pixels
    q = hs.build_panel(1920, 1152)
    assert np.array_equal(p.permutation, q.permutation)
    assert sorted(p.permutation[:5].tolist()) != list(range(5))
    img = p.panel_from_storage(np.ones(p.active_count))
    assert img.shape == (1152, 1920) and np.all(img == 1)
    assert p.geometry_signature() != hs.build_pupil(1920).geometry_signature()


def test_panel_validation():
    with pytest.raises(InvalidParameterError):
        hs.build_panel(1920, 1151)       # unequal parity: cannot centre on the grid
    with pytest.raises(InvalidParameterError):
        hs.build_panel(1, 4)
    with pytest.raises(InvalidParameterError):
        hs.build_panel(8, 4, illumination="gaussian", waist=0.0)


def test_portrait_panel_is_transposed_band():
    p = hs.build_panel(24, 40, illumination="uniform")
    assert p.panel == (40, 24) and p.side_px == 40
    assert (p.cols.min(), p.cols.max(), p.rows.min(), p.rows.max()) == (8, 31, 0, 39)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_on_panels(name):
    p, s, d = panel_case(name)
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, str(d["algorithm"]), int(d["iterations"]),
                     float(d["compression"]), int(d["seed"]))
    assert np.array_equal(r["phase"], d["phase"])
    assert r["ops"] == int(d["ops"])
    assert list(r["sizes"]) == list(d["sizes"])
    assert np.array_equal(r["weights"], d["weights"])
    assert np.array_equal(r["mags"], d["mags"])
    e, u, inten, _ = oracle.quality(p, r["tables"], r["phase"], s.amplitude)
    assert e == float(d["e"]) and u == float(d["u"])
    assert np.array_equal(inten, d["intensities"])
