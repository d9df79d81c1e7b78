"""Multi-process batch driver on the CPU (gloo, world size 2): sharding, the
atlas all-reduce and the stats all-gather, with a deterministic fake per-pair
worker standing in for the GPU registration."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_05117_b200 import batch

N_PAIRS = 7
SHAPE = (6, 5)


def fake_pair(i):
    rng = np.random.default_rng(100 + i)
    return rng.random(SHAPE), rng.random(SHAPE)


def fake_register(src, tgt):
    warped = torch.from_numpy(0.5 * (src + tgt))
    row = [float(src.sum()), float(tgt.sum()), 0.01, 3.0, 0.9, 1.1, 0.0, 0.0, 4.0]
    return row, warped


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = batch.register_batch(fake_pair, n_pairs=N_PAIRS, register_fn=fake_register)
        out[rank] = (res.stats, res.atlas.numpy(), res.pairs_done)
    finally:
        dist.destroy_process_group()


def expected():
    stats = np.array([fake_register(*fake_pair(i))[0] for i in range(N_PAIRS)])
    atlas = sum(0.5 * (s + t) for s, t in (fake_pair(i) for i in range(N_PAIRS))) / N_PAIRS
    return stats, atlas


def test_shard_round_robin():
    assert batch.shard(7, 0, 2) == [0, 2, 4, 6]
    assert batch.shard(7, 1, 2) == [1, 3, 5]
    assert batch.shard(2, 3, 4) == []
    assert sorted(sum((batch.shard(10, r, 3) for r in range(3)), [])) == list(range(10))


def test_single_process_matches_definition():
    res = batch.register_batch(fake_pair, n_pairs=N_PAIRS, register_fn=fake_register)
    st, at = expected()
    np.testing.assert_allclose(res.stats, st)
    np.testing.assert_allclose(res.atlas.numpy(), at)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world(world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    st, at = expected()
    for r in range(world):
        stats, atlas, mine = out[r]
        assert mine == batch.shard(N_PAIRS, r, world)
        np.testing.assert_allclose(stats, st)   # every rank sees the full table
        np.testing.assert_allclose(atlas, at)   # and the same atlas average
