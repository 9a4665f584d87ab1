"""The C-ABI library: builds, loads and exports every declared symbol.

No compute calls here (they need a GPU); on a host without a device the
product must refuse loudly instead of falling back to the CPU.
"""

import ctypes
import os
import re

import pytest

import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import _lib, build
from conftest import ROOT, has_gpu


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "holospots_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    lib = _lib.load()
    assert isinstance(lib, ctypes.CDLL)


def test_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    decl = declared_symbols()
    assert decl, "header parse failed"
    assert sorted(_lib.EXPORTS) == decl
    for name in decl:
        assert hasattr(lib, name), name


def test_max_spots():
    assert _lib.load().hs_max_spots() == 4096   # above 1024 spots: fp64 passes


def test_sm100a_cubin_present():
    """The .so carries sm_100a SASS (no PTX-JIT, no other arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_device():
    p = hs.build_pupil(8, illumination="uniform", seed=1)
    spots = hs.SpotSet.from_points([[1e-6, 0.0, 0.0]])
    with pytest.raises(hs.DeviceError):
        hs.rs(p, spots)
    with pytest.raises(hs.DeviceError):
        hs.superpose(p, spots, hs.SpotCoefficients([1.0], [0.0]))


def test_error_mapping():
    for code, cls in ((1, hs.InvalidParameterError), (2, hs.GeometryMismatchError),
                      (3, hs.DegenerateFieldError), (4, hs.DegenerateFieldError),
                      (5, hs.DeviceError), (6, hs.ZeroIlluminationError),
                      (7, hs.UndefinedUniformityError)):
        with pytest.raises(cls):
            _lib.check(code)
    _lib.check(0)
