"""N>1 path on CPU: request sharding and max-over-ranks timing with a
world_size-2 gloo group (the GPU runs use the same helpers over NCCL)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19893_b200 import sharding as S


def test_request_shard_partitions():
    for total in (0, 1, 7, 64, 65):
        for world in (1, 2, 4, 8):
            got = [list(S.request_shard(total, world, r)) for r in range(world)]
            flat = [x for g in got for x in g]
            assert flat == list(range(total))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        S.request_shard(4, 2, 2)


def test_seeds_depend_on_global_request():
    assert S.request_seed(3) != S.request_seed(4)
    assert S.request_seed(3, 1) != S.request_seed(3, 2)
    # shards of a 2-GPU run see the same data as the 1-GPU run for the same ids
    ids2 = [i for r in range(2) for i in S.request_shard(8, 2, r)]
    assert [S.request_seed(i) for i in ids2] == [S.request_seed(i) for i in range(8)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = S.request_shard(64, world, rank)
        ms = 2.0 + rank  # rank 1 is the slow one
        value, ms_max = S.job_throughput(len(shard) * 9, ms)
        out[rank] = (list(shard), ms_max, value, S.max_over_ranks(10.0 * (rank + 1)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharding_and_timing():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    shards = [res[r][0] for r in range(world)]
    assert sorted(x for s in shards for x in s) == list(range(64))
    assert not set(shards[0]) & set(shards[1])
    for r in range(world):
        _, ms_max, value, mx = res[r]
        assert ms_max == 3.0                       # max over ranks, not rank-local
        assert value == pytest.approx(64 * 9 / 3e-3)  # all units / slowest rank
        assert mx == 20.0
