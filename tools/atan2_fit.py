"""Fit of the fp32 atan2 used by the final pass (csrc/hs_kernels.cuh hs_atan2).

    python tools/atan2_fit.py

atan(r) / r = P(r^2) on r in [0, 1], degree 8, least squares with Lawson
reweighting towards minimax; prints the coefficients and the max |error|
of the fp32 Horner evaluation (with the octant fix-ups) against float64
arctan2 over 2M random points, next to numpy's fp32 arctan2.
"""
import numpy as np

r = np.concatenate([np.linspace(0, 1, 20001), np.cos(np.linspace(0, np.pi / 2, 20000))])
s = r * r
y = np.where(r > 0, np.arctan(r) / np.where(r > 0, r, 1), 1.0)
V = np.vander(s, 9, increasing=True)
w = np.ones_like(s)
for _ in range(30):
    c, *_ = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)
    e = np.abs(V @ c - y)
    w = w * np.sqrt(e / e.max() + 1e-12)
    w /= w.mean()
c = c.astype(np.float32)


def atan2_fast(yv, xv):
    ax, ay = np.abs(xv), np.abs(yv)
    mx, mn = np.maximum(ax, ay), np.minimum(ax, ay)
    rr = (mn / mx).astype(np.float32)
    ss = (rr * rr).astype(np.float32)
    p = np.full_like(ss, c[-1])
    for k in range(len(c) - 2, -1, -1):
        p = (p * ss + c[k]).astype(np.float32)
    a = (rr * p).astype(np.float32)
    a = np.where(ay > ax, (np.float32(np.pi / 2) - a).astype(np.float32), a)
    a = np.where(xv < 0, (np.float32(np.pi) - a).astype(np.float32), a)
    return np.copysign(a, yv)


rng = np.random.default_rng(0)
ys = rng.standard_normal(2_000_000).astype(np.float32)
xs = rng.standard_normal(2_000_000).astype(np.float32)
ref = np.arctan2(ys.astype(np.float64), xs.astype(np.float64))
print("coefficients (s^0 .. s^8):", c.tolist())
print("max |err| fit:", float(np.max(np.abs(atan2_fast(ys, xs) - ref))),
      " numpy fp32 arctan2:", float(np.max(np.abs(np.arctan2(ys, xs) - ref))))
