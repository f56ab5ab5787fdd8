"""Multi-process (gloo, world_size 2) tests of the sharding and the single
all-gather of the multi-GPU path; the device ranking itself is covered by
the GPU tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_01143_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    blocks = rng.integers(1, 64, size=(n, 3))
    cost = shard.config_cost(blocks, np.full(n, 26))
    mine = shard.shard_indices(cost, world, rank)
    m = shard.pad_to(n, world)
    # "records": global index and a value derived from it, padded
    rec = torch.full((m, 2), -1.0, dtype=torch.float64)
    rec[: len(mine), 0] = torch.from_numpy(mine.astype(np.float64))
    rec[: len(mine), 1] = torch.from_numpy((mine * 7 + 1).astype(np.float64))
    g = shard.gather_records(rec, world)
    shards = [shard.shard_indices(cost, world, r) for r in range(world)]
    gi = shard.global_index(shards, m)
    out_q.put((rank, g.numpy(), gi, cost))
    dist.destroy_process_group()


def test_shard_partition_is_exact_and_balanced():
    n = 1001
    cost = shard.config_cost(np.random.default_rng(1).integers(1, 64, size=(n, 3)), np.full(n, 26))
    parts = [shard.shard_indices(cost, 4, r) for r in range(4)]
    allidx = np.concatenate(parts)
    assert sorted(allidx.tolist()) == list(range(n))
    loads = [cost[p].sum() for p in parts]
    assert max(loads) / min(loads) < 1.1


def test_gloo_world2_all_gather_reassembles_every_config():
    world, n = 2, 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    g0, gi = res[0][1], res[0][2]
    assert np.array_equal(g0, res[1][1])  # identical on both ranks
    valid = gi >= 0
    assert sorted(gi[valid].tolist()) == list(range(n))
    assert np.array_equal(g0[valid, 0], gi[valid].astype(float))
    assert np.array_equal(g0[valid, 1], gi[valid] * 7 + 1.0)
