"""Per-iteration accuracy of the device solver against the CPU oracle.

    python tools/accuracy_probe.py [case ...]      # on a GPU box

For each case prints, per iteration, the largest relative deviation of the
trace magnitudes and weights from the oracle's (fp64, bit-exact with the
reference), and the final per-spot intensity / e / u deviations.  Kernel
variants are selected with the plan's environment knobs (HS_UMMA,
HS_UMMA_MAXN), so run it once per variant.  The oracle is the checker here.
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
import paper_2003_05293_b200 as hs  # noqa: E402

G = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def pupil(key):
    return hs.build_pupil(**G["pupils"][key]["kwargs"])


def rand_spots(n, seed, xy=1e-4, z=5e-5, amp="rand"):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.5, 1.5, n) if amp == "rand" else np.ones(n)
    return hs.SpotSet(x=rng.uniform(-xy, xy, n), y=rng.uniform(-xy, xy, n),
                      z=rng.uniform(-z, z, n), amplitude=a)


CASES = {
    "wgs600r": ("p256u0", lambda: rand_spots(600, 1600), "wgs", 3, 1.0, 7),
    "wgs600u": ("p256u0", lambda: rand_spots(600, 1600, amp="one"), "wgs", 3, 1.0, 7),
    "wgs200": ("p256u0", lambda: rand_spots(200, 1200), "wgs", 3, 1.0, 7),
    "cswgs200": ("p256u0", lambda: rand_spots(200, 1200), "cswgs", 4, 0.25, 7),
    "cswgs120": ("p256u0", lambda: rand_spots(120, 1120), "cswgs", 4, 0.25, 7),
    "wgs1000_512": ("p512g0", lambda: rand_spots(1000, 4, xy=1.5e-4), "wgs", 10, 1.0, 0),
    # near the precision "auto" threshold (512 pixels per spot)
    "wgs400_512": ("p512g0", lambda: rand_spots(400, 40, xy=1.5e-4), "wgs", 10, 1.0, 0),
    "cswgs200_512": ("p512g0", lambda: rand_spots(200, 20, xy=1.5e-4), "cswgs", 10, 0.5, 0),
    "cswgs130_512": ("p512g0", lambda: rand_spots(130, 13), "cswgs", 20, 1 / 3, 0),
}


def report(name, mags, w, r, inten=None, want_inten=None, eu=None, want_eu=None):
    em = np.max(np.abs(mags - r["mags"]) / r["mags"], axis=1)
    ew = np.max(np.abs(w - r["weights"]) / r["weights"], axis=1)
    out = {"case": name, "mags_rel_per_iter": [float(f"{v:.3g}") for v in em],
           "weights_rel_per_iter": [float(f"{v:.3g}") for v in ew],
           "env": {k: os.environ[k] for k in ("HS_UMMA", "HS_UMMA_MAXN", "HS_PRECISION")
                   if k in os.environ}}
    if inten is not None:
        out["inten_rel"] = float(np.max(np.abs(inten - want_inten) / want_inten))
        out["de"], out["du"] = abs(eu[0] - want_eu[0]), abs(eu[1] - want_eu[1])
    print(json.dumps(out), flush=True)


def run_case(name):
    if name == "cfg4":
        d = dict(np.load(os.path.join(ROOT, "tests", "golden", "solve_cfg4_wgs1000.npz")))
        p = pupil("p1152g0")
        s = hs.SpotSet(x=d["x"], y=d["y"], z=d["z"], amplitude=d["a0"])
        t = time.time()
        holo, trace = hs.wgs(p, s, iterations=30, seed=0)
        rep = hs.quality_report(p, holo, s)
        mags = np.array([x.magnitudes for x in trace.records])
        w = np.array([x.weights for x in trace.records])
        report(name, mags, w, d, rep.intensities, d["intensities"],
               (rep.efficiency, rep.uniformity), (float(d["e"]), float(d["u"])))
        return
    key, mk, alg, iters, c, seed = CASES[name]
    p, s = pupil(key), mk()
    holo, trace = hs.solve(p, s, hs.SolverConfig(alg, iterations=iters, compression=c, seed=seed))
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, alg, iters, c, seed)
    mags = np.array([x.magnitudes for x in trace.records])
    w = np.array([x.weights for x in trace.records])
    rep = hs.quality_report(p, holo, s)
    e, u, inten, _ = oracle.quality(p, r["tables"], r["phase"], s.amplitude)
    report(name, mags, w, r, rep.intensities, inten, (rep.efficiency, rep.uniformity), (e, u))




def golden_rows(min_iters=0):
    """The reference demo table (compression_runs.csv rows 2-41): |de|, |du|."""
    p = pupil("p256u0")
    frames = G["grid36_frames"]
    for row in G["compression_runs"]:
        if row["iterations"] < min_iters:
            continue
        f = frames[row["seed"]]
        s = hs.SpotSet(x=f["x"], y=f["y"], z=f["z"], amplitude=f["a0"])
        cfg = hs.SolverConfig(row["algorithm"], iterations=row["iterations"],
                              compression=row["c"], seed=row["seed"])
        holo, trace = hs.solve(p, s, cfg)
        rep = hs.quality_report(p, holo, s)
        r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, row["algorithm"], row["iterations"],
                         row["c"], row["seed"])
        mags = np.array([x.magnitudes for x in trace.records])
        em = np.max(np.abs(mags - r["mags"]) / r["mags"], axis=1)
        print(json.dumps({"alg": row["algorithm"], "c": row["c"], "I": row["iterations"],
                          "seed": row["seed"], "de": abs(rep.efficiency - row["e"]),
                          "du": abs(rep.uniformity - row["u"]),
                          "mags_rel_first": [float(f"{v:.3g}") for v in em[:4]],
                          "mags_rel_max": float(em.max()),
                          "mags_rel_argmax": int(em.argmax())}), flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or list(CASES) + ["cfg4"]):
        if c.startswith("golden"):
            golden_rows(int(c[6:] or 0))
        else:
            run_case(c)
