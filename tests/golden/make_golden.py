"""Generate golden fixtures by running the reference ``holospots`` package.

Run in the build container (where /root/reference exists):

    NUMBA_NUM_THREADS=8 python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` and ``tests/golden/golden.json``.  The
fixtures pin the oracle (``oracle/``) and the product; nothing at test
time reads /root/reference.
"""

import csv
import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_NUM_THREADS", "8")

import holospots as hs  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_foci(n, seed, xy=100e-6, z=50e-6):
    """Same draw order as paper_2003_05293_b200.workloads.random_foci."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-xy, xy, n)
    y = rng.uniform(-xy, xy, n)
    zz = rng.uniform(-z, z, n)
    return hs.SpotSet(x=x, y=y, z=zz, amplitude=np.ones(n))


def test_spots(rng, n, xy=6e-5, z=2e-4):
    """Reference conftest.random_spots (pkg/tests/conftest.py:40-42)."""
    return hs.SpotSet(x=rng.uniform(-xy, xy, n), y=rng.uniform(-xy, xy, n),
                      z=rng.uniform(-z, z, n), amplitude=rng.uniform(0.3, 2.0, n))


def spots_dict(s):
    return dict(x=s.x, y=s.y, z=s.z, a0=s.amplitude)


summary = {"pupils": {}, "solves": {}, "kernels": {}}

# ---------------------------------------------------------------- pupils
PUPILS = {
    "p8u1": dict(side_px=8, illumination="uniform", seed=1),
    "p16g2": dict(side_px=16, illumination="gaussian", waist=6e-5, seed=2),
    "p48g2": dict(side_px=48, illumination="gaussian", waist=2e-4, seed=2),
    "p64u0": dict(side_px=64, illumination="uniform", seed=0),
    "p256u0": dict(side_px=256, illumination="uniform", seed=0),
    "p512g0": dict(side_px=512, illumination="gaussian", waist=6e-3, seed=0),
    "p1152g0": dict(side_px=1152, illumination="gaussian", waist=6e-3, seed=0),
}
pupils = {}
for key, kw in PUPILS.items():
    p = hs.build_pupil(**kw)
    pupils[key] = p
    summary["pupils"][key] = dict(
        kwargs=kw, M=int(p.active_count), sum_amplitude=float(p.sum_amplitude),
        sha_rows=sha(p.rows), sha_cols=sha(p.cols), sha_amp=sha(p.amplitude),
        sha_perm=sha(p.permutation), prism=p.prism_coeff, lens=p.lens_coeff)
    if p.side_px <= 64:
        np.savez_compressed(os.path.join(HERE, f"pupil_{key}.npz"), rows=p.rows,
                            cols=p.cols, amplitude=p.amplitude,
                            permutation=p.permutation, aperture=p.aperture)

# ------------------------------------------------------- kernel vectors
rng = np.random.default_rng(20031)
kcases = {}
for i, key in enumerate(["p8u1", "p16g2", "p48g2", "p64u0"]):
    p = pupils[key]
    for n in (1, 3, 7):
        s = test_spots(rng, n)
        amp = rng.uniform(0.0, 2.0, n)
        theta = rng.uniform(-9.0, 9.0, n)
        tab = hs.spot_tables(p, s)
        frag = hs.superpose(p, s, hs.SpotCoefficients(amp, theta))
        m = p.active_count
        lo, hi = int(m // 5), int(m - m // 7)
        frag_rng = hs.superpose(p, s, hs.SpotCoefficients(amp, theta), (lo, hi))
        phase = hs.wrap_phase(rng.uniform(-4.0, 4.0, m))
        holo = hs.Hologram(phase, p)
        fields = hs.forward_project(p, holo, s)
        fields_rng = hs.forward_project(p, holo, s, (lo, hi), chunk=37)
        inten = hs.spot_intensities(p, holo, s)
        name = f"k_{key}_n{n}"
        kcases[name] = dict(pupil=key, **spots_dict(s), amp=amp, theta=theta,
                            gx_re=tab.gx_re, gx_im=tab.gx_im, gy_re=tab.gy_re,
                            gy_im=tab.gy_im, superpose=frag, lo=lo, hi=hi,
                            superpose_range=frag_rng, phase=phase,
                            fields=fields, fields_range=fields_rng,
                            intensities=inten)
np.savez_compressed(os.path.join(HERE, "kernels.npz"),
                    **{f"{c}.{k}": v for c, d in kcases.items()
                       for k, v in d.items() if k != "pupil"})
summary["kernels"] = {c: d["pupil"] for c, d in kcases.items()}

# reduce_complex vectors
rvals = rng.normal(size=5000) + 1j * rng.normal(size=5000)
summary["reduce"] = {str(ch): [hs.reduce_complex(rvals[:nn], chunk=ch).real,
                               hs.reduce_complex(rvals[:nn], chunk=ch).imag, nn]
                     for ch, nn in ((4, 17), (7, 5000), (32, 1025), (1024, 5000))}
np.save(os.path.join(HERE, "reduce_values.npy"), rvals)

# ---------------------------------------------------------------- solves
SUB = 97  # phase subsample stride for the large cases


def run(name, pupil_key, spots, algorithm, iterations=1, compression=1.0,
        seed=0, full_phase=False):
    p = pupils[pupil_key]
    cfg = hs.SolverConfig(algorithm, iterations=iterations,
                          compression=compression, seed=seed)
    holo, trace = hs.solve(p, spots, cfg, workers=8)
    rep = hs.quality_report(p, holo, spots, workers=8)
    idx = np.arange(0, p.active_count, 1 if full_phase else SUB)
    rec_w = np.array([r.weights for r in trace.records]) if trace.records else \
        np.zeros((0, spots.count))
    rec_m = np.array([r.magnitudes for r in trace.records]) if trace.records else \
        np.zeros((0, spots.count))
    np.savez_compressed(
        os.path.join(HERE, f"solve_{name}.npz"), **spots_dict(spots),
        phase_idx=idx, phase=holo.phase[idx], weights=rec_w, mags=rec_m,
        sizes=np.array([r.subset_size for r in trace.records], dtype=np.int64),
        intensities=rep.intensities, relative=rep.target_relative)
    summary["solves"][name] = dict(
        pupil=pupil_key, algorithm=algorithm, iterations=iterations,
        compression=compression, seed=seed, ops=int(trace.operation_count),
        degenerate=bool(trace.degenerate), e=rep.efficiency, u=rep.uniformity,
        phase_sha=sha(holo.phase), full_phase=full_phase)
    print(f"{name}: e={rep.efficiency:.6f} u={rep.uniformity:.6f} "
          f"ops={trace.operation_count}", flush=True)


rng = np.random.default_rng(7)
run("wgs_p64", "p64u0", test_spots(rng, 5), "wgs", 8, seed=9, full_phase=True)
run("cswgs_p48", "p48g2", test_spots(rng, 4), "cswgs", 7, 0.25, seed=1,
    full_phase=True)
run("rs_p64", "p64u0", test_spots(rng, 6), "rs", seed=3, full_phase=True)
run("cswgs_p64_i2", "p64u0", test_spots(rng, 3), "cswgs", 2, 0.3, seed=2,
    full_phase=True)
run("cswgs_p64_c1", "p64u0", test_spots(rng, 3), "cswgs", 5, 1.0, seed=4,
    full_phase=True)
grid36 = hs.named_scenario("grid36").spot_set()
run("wgs_grid36_256", "p256u0", grid36, "wgs", 5, seed=0)
run("cswgs_grid36_256", "p256u0", grid36, "cswgs", 12, 0.125, seed=0)
run("cfg1", "p512g0", random_foci(10, 12345), "cswgs", 10, 1 / 8, seed=0)
run("cfg2_rs", "p1152g0", random_foci(100, 12345), "rs", seed=0)
grid100 = hs.named_scenario("grid100").spot_set()
run("cfg3_grid100", "p1152g0", grid100, "cswgs", 20, 1 / 16, seed=0)
run("cfg3_random", "p1152g0", random_foci(100, 12345), "cswgs", 20, 1 / 16, seed=0)

# ------------------------------------- reference demo golden table (rows 2-41)
rows = []
with open("/root/reference/pkg/demos/output/compression_runs.csv") as fh:
    for i, row in enumerate(csv.DictReader(fh)):
        if i >= 40:  # rows 42-51 (c <= 2^-7) are chaotic
            break
        rows.append(dict(algorithm=row["algorithm"], c=float(row["c"]),
                         iterations=int(row["iterations"]), ops=int(row["ops"]),
                         e=float(row["efficiency"]), u=float(row["uniformity"]),
                         seed=int(row["seed"])))
summary["compression_runs"] = rows
summary["grid36"] = spots_dict_list = {k: v.tolist() for k, v in
                                       spots_dict(grid36).items()}
summary["grid100"] = {k: v.tolist() for k, v in spots_dict(grid100).items()}
# compare_at_budget runs seed k on rotation frame k (bench.py:183-200)
summary["grid36_frames"] = [{k: v.tolist() for k, v in spots_dict(f).items()}
                            for f in hs.rotation_sweep(hs.named_scenario("grid36"), 5)]

with open(os.path.join(HERE, "golden.json"), "w") as fh:
    json.dump(summary, fh, indent=1, default=float)
print("wrote", HERE)
