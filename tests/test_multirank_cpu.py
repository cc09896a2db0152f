"""World-size-2 gloo tests of the N>1 host logic on CPU: shard ranges (weak,
strong, and C4's value-range split), bench.py's per-rank batch selection and
golden totals, the count reduction and the max-time reduction.  Each rank
classifies its shard with the oracle (test infrastructure; the GPU ranks run
the CUDA path)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
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


def _worker_bench_split(rank, world, port, q):
    """bench.py's multi-GPU batch selection, scaled down: C4's value-range
    split over [0, 2^22) (each rank sieves only its window), the strong split
    of a fixed C2 prefix, and the weak C1 batches against the golden
    per-rank counts -- each rank classifies its batch with the oracle and the
    counts are summed over gloo like bench.py sums them over NCCL."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, a, b = bench.shard_input("C4", "weak", rank, world)
        assert kind == "iota" and (a, b) == shard.value_range_shard(rank, world, 0, 1 << 32)
        va, vb = shard.value_range_shard(rank, world, 0, 1 << 22)
        c4 = shard.reduce_count(int(oracle.dense_range(va, vb - va).sum()))
        m = 1 << 18
        sa, sb = shard.strong_shard(rank, world, m)
        c2 = shard.reduce_count(int(oracle.isprime(workloads.generate("C2", start=sa, count=sb - sa),
                                                   threads=1).sum()))
        kind, wa, wb = bench.shard_input("C1", "weak", rank, world)
        assert kind == "gen" and wb - wa == workloads.CONFIGS["C1"][1]
        c1 = shard.reduce_count(int(oracle.isprime(workloads.generate("C1", start=wa, count=wb - wa),
                                                   threads=1).sum()))
        q.put((rank, c4, c2, c1, (va, vb)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_value_range_and_strong_split():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_bench_split, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pi_2_22 = 295947
    c2_whole = int(oracle.isprime(workloads.generate("C2", count=1 << 18)).sum())
    wc = bench.load_weak_counts()
    for rank, c4, c2, c1, _ in res:
        assert c4 == pi_2_22
        assert c2 == c2_whole
        assert c1 == wc["C1"][0] + wc["C1"][1] == bench.expected_total("C1", "weak", 2, bench.load_counts(), wc)
    assert res[0][4] == (0, 1 << 21) and res[1][4] == (1 << 21, 1 << 22)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_batches_cover_and_totals(world):
    """bench.py's batches: strong and C4 batches tile the fixed array / value
    range exactly once; weak batches are consecutive full batches; the golden
    totals are the full count (strong, C4) or the sum of per-rank counts."""
    counts, wc = bench.load_counts(), bench.load_weak_counts()
    for cfg in ("C1", "C2", "C3", "C4", "C5"):
        n = workloads.CONFIGS[cfg][1]
        for mode in ("weak", "strong"):
            spans = [bench.shard_input(cfg, mode, r, world) for r in range(world)]
            sc = bench.scaling_of(cfg, mode)
            if sc == "strong":
                assert spans[0][1] == 0 and spans[-1][2] == n
                assert all(x[2] == y[1] for x, y in zip(spans, spans[1:]))
                assert bench.expected_total(cfg, mode, world, counts, wc) == counts[cfg]
                assert bench.global_units(cfg, mode, world) == n
            else:
                assert [(x[1], x[2]) for x in spans] == [(r * n, (r + 1) * n) for r in range(world)]
                assert bench.global_units(cfg, mode, world) == n * world
                assert bench.expected_total(cfg, mode, world, counts, wc) == sum(wc[cfg][r] for r in range(world))
            assert all(x[0] == ("iota" if cfg == "C4" else "gen") for x in spans)
    assert wc["C1"][0] == counts["C1"] and wc["C5"][0] == counts["C5"]
