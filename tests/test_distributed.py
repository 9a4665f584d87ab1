"""Multi-process (gloo, world_size 2) tests of the sharding logic.

The device fold is restated on the host (distributed.fold_groups /
fold_fields); these tests check that splitting a pass across ranks at fold
group boundaries yields bitwise the single-rank fields, and that batch
sharding covers every pattern exactly once.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_05293_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_patterns_cover_exactly_once():
    for total in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                f, c = D.shard_patterns(total, world, r)
                seen.extend(range(f, f + c))
            assert seen == list(range(total))


def test_shard_groups_aligned_and_balanced():
    for nchunks in (1, 31, 32, 33, 538, 552, 1170):
        for world in (1, 2, 4, 8):
            rng = D.shard_groups(nchunks, world)
            assert rng[0][0] == 0 and rng[-1][1] == nchunks
            for (a, b), (c, d) in zip(rng, rng[1:]):
                assert b == c
            for a, b in rng:
                assert a % D.GROUP == 0 and (b % D.GROUP == 0 or b == nchunks)


def test_single_rank_fold_equals_sharded_fold_in_process():
    rng = np.random.default_rng(0)
    part = (rng.normal(size=(552, 112)) + 1j * rng.normal(size=(552, 112))).astype(np.complex64)
    want = D.fold_fields(D.fold_groups(part, 0, part.shape[0]))
    for world in (2, 4, 8):
        pieces = [D.fold_groups(part, lo, hi) for lo, hi in D.shard_groups(552, world)]
        got = D.fold_fields(np.concatenate([p for p in pieces if p.size]))
        assert np.array_equal(got, want)


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)  # same partials on every rank
        part = (rng.normal(size=(300, 48)) + 1j * rng.normal(size=(300, 48))).astype(np.complex64)

        def all_gather(local):
            out = [None] * world
            dist.all_gather_object(out, local)
            return out

        fields = D.sharded_fields(part, world, rank, all_gather)
        # batch sharding: each rank sums its own pattern ids; all-reduce
        first, count = D.shard_patterns(10, world, rank)
        ids = [list(range(first, first + count))]
        gathered = [None] * world
        dist.all_gather_object(gathered, ids)
        if rank == 0:
            np.save(result_path, fields)
            with open(result_path + ".ids", "w") as fh:
                fh.write(repr(sum((g[0] for g in gathered), [])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_fields_bitwise(tmp_path):
    path = str(tmp_path / "fields.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got = np.load(path)
    rng = np.random.default_rng(123)
    part = (rng.normal(size=(300, 48)) + 1j * rng.normal(size=(300, 48))).astype(np.complex64)
    want = D.fold_fields(D.fold_groups(part, 0, 300))
    assert np.array_equal(got, want)
    assert open(path + ".ids").read() == repr(list(range(10)))
