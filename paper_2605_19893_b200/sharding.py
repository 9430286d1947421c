"""Multi-GPU plumbing for the verify path: request sharding, no collectives on
the data path.

Requests are independent (the reference's engine runs one request per
engine; groups and layers are pure functions), so N GPUs split the requests
and each runs its own `nsa_verify` calls.  torch.distributed is used only to
agree on timing: the step time is the MAX over ranks of each rank's
device-measured time, and throughput is all units processed / that time.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def request_shard(total: int, world: int, rank: int) -> range:
    """Contiguous, balanced request ids of `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def request_seed(request: int, layer: int = 0) -> int:
    """Seed of a request's synthetic data: a function of the GLOBAL request id,
    so every shard sees distinct requests and a run is independent of N."""
    return 1234 + 1000 * request + layer


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """Max of a per-rank scalar (device time) over the process group."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device: torch.device | None = None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(units_this_rank: float, ms_this_rank: float,
                   device: torch.device | None = None) -> tuple[float, float]:
    """(whole-job units/s, max-over-ranks ms): all ranks' units over the slowest
    rank's time -- the weak-scaling aggregate bench.py reports."""
    units = sum_over_ranks(units_this_rank, device)
    ms = max_over_ranks(ms_this_rank, device)
    return units / (ms * 1e-3), ms
