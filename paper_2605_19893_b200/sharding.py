"""Multi-GPU plumbing for the verify path: request sharding and KV-head-group
sharding, no collectives on the data path.

Requests are independent (the reference's engine runs one request per
engine; groups and layers are pure functions), so N GPUs split the requests
and each runs its own `nsa_verify` calls.  With fewer requests than GPUs a
request is split by KV-head group: every shard routes over all heads (the
reference sums the selection mass over all Hq heads,
nsa_attention.cpp:51-63, so the index sets need every head's compressed
keys -- SURVEY 8e option i, replicated routing) and attends only its KV
heads.  torch.distributed is used only to agree on timing: the step time is
the MAX over ranks of each rank's device-measured time, and throughput is
all units processed / that time.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def request_shard(total: int, world: int, rank: int) -> range:
    """Contiguous, balanced request ids of `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


@dataclass(frozen=True)
class Shard:
    """One rank's piece of one request: KV heads [head_begin, head_begin + head_count)."""
    request: int
    head_begin: int
    head_count: int
    n_kv_heads: int

    @property
    def whole(self) -> bool:
        return self.head_begin == 0 and self.head_count == self.n_kv_heads

    @property
    def fraction(self) -> float:
        """Share of the request's query-tokens this shard completes."""
        return self.head_count / self.n_kv_heads

    def kv_heads(self):
        """(begin, count) for nsa_verify(kv_heads=...), None for the whole request."""
        return None if self.whole else (self.head_begin, self.head_count)


def shard_plan(total_requests: int, world: int, rank: int, n_kv_heads: int) -> list[Shard]:
    """This rank's shards.  total >= world: whole requests, contiguous and
    balanced (request_shard).  total < world: each request gets a contiguous
    group of ranks (sizes differ by at most 1) that splits its KV heads into
    contiguous, balanced ranges; a group larger than n_kv_heads is refused."""
    if world < 1 or not 0 <= rank < world or total_requests < 1 or n_kv_heads < 1:
        raise ValueError("bad shard arguments")
    if total_requests >= world:
        return [Shard(r, 0, n_kv_heads, n_kv_heads) for r in request_shard(total_requests, world, rank)]
    # ranks of request r: request_shard(world, total_requests, r) -- which request owns this rank
    for r in range(total_requests):
        ranks = request_shard(world, total_requests, r)
        if rank in ranks:
            n = len(ranks)
            if n > n_kv_heads:
                raise ValueError(f"{n} ranks cannot split {n_kv_heads} KV heads")
            heads = request_shard(n_kv_heads, n, rank - ranks.start)
            return [Shard(r, heads.start, len(heads), n_kv_heads)]
    raise AssertionError("unreachable")


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
