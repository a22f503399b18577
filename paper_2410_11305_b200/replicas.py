"""Request-sharded replicas: one process per GPU, each owning a full model
copy and a contiguous shard of the request list; no data-path collective.

The only cross-rank communication is the benchmark's timing reduction: tokens are
summed over ranks and the device time is the max over ranks, so the reported
whole-job throughput is (sum of tokens) / (slowest rank's time).
"""

from __future__ import annotations


def shard_bounds(n_requests: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of n_requests for this rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n_requests, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def reduce_throughput(tokens: float, ms: float, dist=None) -> tuple[float, float]:
    """(sum of tokens over ranks, max device ms over ranks); identity without torch.distributed."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(tokens), float(ms)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([tokens], dtype=torch.float64, device=dev)
    m = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return float(t.item()), float(m.item())
