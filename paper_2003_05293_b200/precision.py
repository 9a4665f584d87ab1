"""Scoped precision mode of the pixel passes (see ``set_precision``).

    with hs.precision("fp64"):
        holo, trace = hs.wgs(pupil, spots, iterations=30)
"""

from __future__ import annotations

import contextlib

from . import _lib


@contextlib.contextmanager
def precision(mode: str):
    """Run the enclosed calls with pixel-pass precision ``mode``
    ("auto", "fp32" or "fp64"), restoring the previous mode afterwards."""
    prev = _lib.get_precision()
    _lib.set_precision(mode)
    try:
        yield
    finally:
        _lib.set_precision(prev)
