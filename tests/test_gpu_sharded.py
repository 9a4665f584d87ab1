"""Row-sharded solve (distributed.solve_sharded) with 2 processes on the one
GPU of the test box, exchanging group partials over gloo.  Results must be
bitwise identical to the single-process solve."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import distributed as D

pytestmark = pytest.mark.gpu

CASES = {
    "cswgs_tile": (dict(side_px=256, illumination="gaussian", waist=1e-3, seed=0), 36, "cswgs", 8, 0.125),
    "wgs_rowrun": (dict(side_px=96, illumination="uniform", seed=3), 200, "wgs", 4, 1.0),
    "rs_tile": (dict(side_px=128, illumination="uniform", seed=1), 20, "rs", 1, 1.0),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spots(n, seed):
    return hs.random_foci(n, seed, xy=8e-5, z=3e-5)


def _worker(rank, world, port, case, out, exchange="host"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pk, n, alg, iters, c = CASES[case]
        pupil = hs.build_pupil(**pk)
        cfg = hs.SolverConfig(alg, iterations=iters, compression=c, seed=5)

        def all_gather(obj):
            res = [None] * world
            dist.all_gather_object(res, obj)
            return res

        holo, trace = D.solve_sharded(pupil, _spots(n, 11), cfg, rank, world, all_gather, device=0,
                                      exchange=exchange)
        np.savez(f"{out}.{rank}.npz", phase=holo.phase, e=trace.quality.efficiency,
                 u=trace.quality.uniformity,
                 mags=np.array([r.magnitudes for r in trace.records]).reshape(-1),
                 ops=trace.operation_count)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["host", "p2p"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_sharded_solve_bitwise(tmp_path, case, exchange):
    """host: group partials through gloo; p2p: through CUDA IPC peer memory
    written by the publish kernel (two processes share the one GPU here)."""
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), case, out, exchange), nprocs=2, join=True)
    pk, n, alg, iters, c = CASES[case]
    pupil = hs.build_pupil(**pk)
    # the row-sharded solve runs the fp32 passes (these small pupils would
    # run fp64 under precision "auto")
    with hs.precision("fp32"):
        holo, trace = hs.solve(pupil, _spots(n, 11), hs.SolverConfig(alg, iters, c, seed=5))
    for rank in range(2):
        r = np.load(f"{out}.{rank}.npz")
        assert np.array_equal(r["phase"], holo.phase), case
        assert float(r["e"]) == trace.quality.efficiency and float(r["u"]) == trace.quality.uniformity
        assert np.array_equal(r["mags"], np.array([x.magnitudes for x in trace.records]).reshape(-1))
        assert int(r["ops"]) == trace.operation_count
