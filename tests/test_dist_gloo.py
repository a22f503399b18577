"""Multi-process (world_size 2, gloo, CPU) coverage of the replica path: request
sharding and the sum-tokens / max-time throughput reduction bench.py uses."""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_11305_b200.replicas import reduce_throughput, shard_bounds


def test_shard_bounds_cover_and_balance():
    for n in (0, 1, 7, 16, 33):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, out) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(10, rank, world)
    tokens = 100.0 * (hi - lo)          # each rank "generates" 100 tokens per request
    ms = 50.0 + 25.0 * rank              # rank 1 is slower
    tot, mx = reduce_throughput(tokens, ms, dist)
    out[rank] = (lo, hi, tot, mx)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replica_reduction():
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][:2] == (0, 5) and res[1][:2] == (5, 10)
    for r in (0, 1):
        assert res[r][2] == 1000.0 and res[r][3] == 75.0   # sum of tokens, max of times


def test_single_process_identity():
    assert reduce_throughput(12.0, 3.0, None) == (12.0, 3.0)
