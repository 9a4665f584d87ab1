"""Multi-GPU sharding logic (one process per GPU).

Two decompositions:

* **Batch data parallelism** (configs 3 / 5): independent patterns are split
  into contiguous per-rank ranges. There is no data-path collective; each
  rank owns its own plan and device.
* **Pixel sharding of one hologram** (config 4): the fixed chunk list of a
  pass (tiles for full-range passes, sorted-window chunks for compressed
  ones) is split across ranks **at fold-group boundaries** (groups of
  ``GROUP`` chunks, the first level of the device fold tree,
  csrc/hs_kernels.cuh ``kGroup``). Every group is then folded by exactly one
  rank, in the device order. The exchange is an all-gather of the
  ``ngroups x np`` complex128 group partials. Every rank folds them in group
  order, so the fields are bitwise identical on every rank and identical to
  the single-GPU result for any world size.

``fold_groups`` / ``fold_fields`` restate the device fold on the host so the
gloo tests can check the invariance without a GPU.
"""

from __future__ import annotations

import numpy as np

GROUP = 32  # chunks per first-level fold group (kGroup in hs_kernels.cuh)


def shard_patterns(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pattern range [first, first + count) of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def shard_groups(nchunks: int, world: int) -> list[tuple[int, int]]:
    """Per-rank chunk ranges aligned to fold groups, balanced by chunk count."""
    if world < 1:
        raise ValueError("world must be >= 1")
    ngroups = -(-nchunks // GROUP)
    bounds = []
    for r in range(world + 1):
        g = (r * ngroups) // world
        bounds.append(min(g * GROUP, nchunks))
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def fold_groups(partials: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Group partials of chunks [lo, hi) (group-aligned): fp64 sums of the
    fp32 chunk partials in chunk order, one row per group."""
    part = np.asarray(partials)
    out = []
    for g0 in range(lo, hi, GROUP):
        acc = np.zeros(part.shape[1], dtype=np.complex128)
        for c in range(g0, min(g0 + GROUP, hi)):
            acc = acc + part[c].astype(np.complex128)
        out.append(acc)
    return np.array(out).reshape(-1, part.shape[1])


def fold_fields(group_partials: np.ndarray) -> np.ndarray:
    """Second fold level: groups summed in group order (fp64)."""
    acc = np.zeros(group_partials.shape[1], dtype=np.complex128)
    for row in group_partials:
        acc = acc + row
    return acc


def sharded_fields(partials: np.ndarray, world: int, rank: int, all_gather) -> np.ndarray:
    """Fields of one pass computed by ``world`` ranks.

    Rank ``rank`` folds its groups, ``all_gather(local) -> list`` exchanges
    the group partials (rank order = group order), and every rank folds the
    same sequence.
    """
    lo, hi = shard_groups(partials.shape[0], world)[rank]
    local = fold_groups(partials, lo, hi)
    gathered = all_gather(local)
    return fold_fields(np.concatenate([g for g in gathered if g.size], axis=0))


# ---------------------------------------------------------------- device path
def solve_sharded(pupil, spots, config, rank: int, world: int, all_gather, device=None,
                  exchange: str = "p2p"):
    """Row-sharded solve of one pattern across ``world`` processes.

    Every rank calls this with the same ``spots`` / ``config``.
    ``exchange="p2p"`` (default, one node): the ranks swap CUDA IPC handles once through
    ``all_gather`` and every pass exchanges its group partials over peer
    memory on the device (csrc/hs_xchg.cuh) -- no host round trip.
    ``exchange="host"`` (e.g. across nodes): ``all_gather(obj) -> list``
    (rank order) carries the per-pass group partials (``ngroups x np``
    complex128 per pass) through the host.  Either
    way the phase slabs are gathered at the end, and the result
    ``(Hologram, SolverTrace)`` is identical on every rank and bitwise equal
    to :func:`paper_2003_05293_b200.solve` on one GPU with precision "fp32":
    the sharded passes are the fp32 kernels (n <= 1024; precision "fp64"
    raises InvalidParameterError).  Row sharding pays for large, well-
    conditioned problems (config 4: 1042 pixels per spot), which precision
    "auto" runs in fp32 on one GPU as well.
    """
    import time

    from . import _lib
    from .optics import CompressionPlan, Hologram
    from .solvers import (SolverConfig, SolverTrace, StepRecord, _ALG_CODE, _raise_status,
                          _theta0, window_sizes)

    if not isinstance(config, SolverConfig):
        raise TypeError("config must be a SolverConfig")
    t0 = time.perf_counter()
    m, n = pupil.active_count, spots.count
    subset = m
    if config.algorithm == "cswgs":
        subset = CompressionPlan.for_pupil(pupil, config.compression).subset_size
    iters = 0 if config.algorithm == "rs" else config.iterations
    plan = _lib.plan_for(pupil, device)
    plan.set_spots(spots)
    plan.shard_begin(_ALG_CODE[config.algorithm], iters, subset, _theta0(config.seed, n),
                     rank, world)
    passes = 1 if config.algorithm == "rs" else iters + 1
    if exchange == "p2p":
        handles = all_gather(plan.p2p_setup())
        try:
            plan.p2p_open(handles)
            plan.p2p_solve()  # all passes as one captured graph (hs_shard_p2p_solve)
            plan.sync()
        finally:
            all_gather(None)  # every rank finished reading its peers' buffers
            plan.p2p_close()
    elif exchange == "host":
        for j in range(passes):
            local, g_lo, g_hi, ngroups = plan.shard_pass(j)
            pieces = all_gather((g_lo, g_hi, local))
            order = sorted(pieces, key=lambda t: t[0])
            groups = np.concatenate([t[2] for t in order if t[2].shape[1]], axis=1)
            if groups.shape[1] != ngroups:
                raise RuntimeError(f"group exchange incomplete: {groups.shape[1]} of {ngroups}")
            plan.shard_update(j, groups)
    else:
        raise ValueError(f"unknown exchange {exchange!r}")
    status, deg = plan.status()
    # every rank raises together: a failed rank (or a peer abort seen by the
    # exchange) must not leave the others waiting in the phase exchange
    codes = all_gather(int(status[0]))
    bad = [c for c in codes if c != 0]
    if bad:
        _raise_status(int(status[0]) or bad[0])
    mine = plan.phases()[0]
    slabs = all_gather(mine)
    phase = np.full(m, np.nan)
    for sl in slabs:
        own = ~np.isnan(sl)
        phase[own] = sl[own]
    if np.isnan(phase).any():
        raise RuntimeError("phase slabs do not cover the pupil")
    holo = Hologram(phase, pupil)
    e, u, inten, rel, _ = plan.quality_batch()
    from .metrics import QualityReport
    fused = QualityReport(float(e[0]), float(u[0]), inten[0].copy(), rel[0].copy())
    if config.algorithm == "rs":
        return holo, SolverTrace("rs", (), m * n, time.perf_counter() - t0, False, holo, fused)
    w, mg = plan.trace(iters)
    records, ops = [], 0
    first = int(deg[0])
    for j, size in enumerate(window_sizes(m, subset, iters), start=1):
        ops += size * n
        records.append(StepRecord(j, w[0, j - 1].copy(), mg[0, j - 1].copy(), size, ops,
                                  bool(first and j >= first)))
    return holo, SolverTrace(config.algorithm, tuple(records), ops, time.perf_counter() - t0,
                             bool(first), holo, fused)
