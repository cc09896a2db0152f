"""World-size-2 gloo tests of the N>1 host logic on CPU: shard ranges, the
count reduction and the max-time reduction.  Each rank classifies its shard
with the oracle (test infrastructure; the GPU ranks run the CUDA path)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_2108_04791_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # strong scaling over a fixed array
        n = 100_003
        lo, hi = shard.strong_shard(rank, world, n)
        N = workloads.generate("C5", start=lo, count=hi - lo)
        c = int(oracle.isprime(N, threads=1).sum())
        total = shard.reduce_count(c)
        # weak scaling: each rank a full batch of the generator stream
        m = 40_000
        wlo, whi = shard.weak_shard(rank, world, m)
        W = workloads.generate("C5", start=wlo, count=whi - wlo)
        wc = int(oracle.isprime(W, threads=1).sum())
        wtotal = shard.reduce_count(wc)
        tmax = shard.reduce_max(float(rank + 1) * 1.5)
        q.put((rank, total, wtotal, tmax, lo, hi))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_counts():
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
    res.sort()
    n = 100_003
    whole = int(oracle.isprime(workloads.generate("C5", count=n)).sum())
    weak_whole = int(oracle.isprime(workloads.generate("C5", count=2 * 40_000)).sum())
    for rank, total, wtotal, tmax, lo, hi in res:
        assert total == whole
        assert wtotal == weak_whole
        assert tmax == 3.0
    assert res[0][4] == 0 and res[0][5] == res[1][4] and res[1][5] == n


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_ranges_cover_exactly_once(world):
    for n in (0, 1, 7, 4096, 100_003, 2**32):
        spans = [shard.strong_shard(r, world, n) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    assert shard.weak_shard(3, 8, 10) == (30, 40)
    with pytest.raises(ValueError):
        shard.strong_shard(world, world, 10)
