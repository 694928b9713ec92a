"""Multi-rank host logic on CPU (gloo, world size 2): character sharding and the
max-over-ranks / sum-over-ranks reduction bench.py uses."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import hsgen


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for scaling in ("weak", "strong"):
            c0, n = bench.shard(1_000_001, rank, world, scaling)
            out[scaling] = (c0, n)
        # each rank "times" a different duration; the job time is the max, joints the sum
        ms, joints = bench.reduce_over_ranks(10.0 + 5.0 * rank, 1000 * (rank + 1), world, "cpu")
        out["reduced"] = (ms, joints)
        # every rank regenerates its own shard from the counter RNG: same bits as a
        # single process generating the union
        c0, n = bench.shard(6, rank, world, "strong")
        out["poses"] = hsgen.local_poses(5, 64, n, char0=c0, type_=0)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # weak: each rank owns a full crowd at a disjoint global offset
    assert res[0]["weak"] == (0, 1_000_001) and res[1]["weak"] == (1_000_001, 1_000_001)
    # strong: contiguous, disjoint, covering split
    (a0, an), (b0, bn) = res[0]["strong"], res[1]["strong"]
    assert a0 == 0 and a0 + an == b0 and b0 + bn == 1_000_001
    for r in range(world):
        assert res[r]["reduced"] == (15.0, 3000)
    union = np.concatenate([res[0]["poses"], res[1]["poses"]])
    assert np.array_equal(union, hsgen.local_poses(5, 64, 6))
