"""Multi-rank host logic on CPU (gloo, world_size 2): batch sharding, max-over-
ranks timing aggregation and the optional result gather used by bench.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_6238_b200.dist import gather_shards, max_over_ranks, shard_range


def test_shard_range_partitions():
    for batch in [0, 1, 7, 4096, 4097]:
        for world in [1, 2, 3, 8]:
            parts = [shard_range(batch, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == batch
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # timing rule: max over ranks
        t = max_over_ranks(1.0 + rank)
        # each rank computes its shard of a toy batch; rank 0 gathers
        batch, n = 11, 3
        a, b = shard_range(batch, rank, world)
        local = torch.arange(a, b, dtype=torch.float64)[:, None] * torch.ones(n) \
            + 1j * torch.arange(a, b, dtype=torch.float64)[:, None]
        full = gather_shards(local.to(torch.complex128), batch)
        q.put((rank, t, None if full is None else full.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_and_gather():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert all(r[1] == pytest.approx(2.0) for r in res)
    full = res[0][2]
    expect = np.arange(11)[:, None] * np.ones(3) + 1j * np.arange(11)[:, None]
    np.testing.assert_array_equal(full, expect)
    assert res[1][2] is None
