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


def test_shard_plan_requests_and_head_groups():
    """total >= world: whole requests (request_shard); total < world: each
    request's rank group splits its KV heads into contiguous balanced ranges."""
    for total, world in ((64, 8), (64, 2), (8, 8), (4, 8), (1, 8), (3, 8), (1, 2), (5, 4)):
        got = [S.shard_plan(total, world, r, 8) for r in range(world)]
        cover = {}
        for r, shards in enumerate(got):
            assert shards, (total, world, r)
            for s in shards:
                cover.setdefault(s.request, []).append((s.head_begin, s.head_count))
        assert sorted(cover) == list(range(total))
        for req, ranges in cover.items():
            heads = sorted(h for b, n in ranges for h in range(b, b + n))
            assert heads == list(range(8)), (total, world, req, ranges)
        units = sum(s.fraction for shards in got for s in shards)
        assert units == pytest.approx(total)
    with pytest.raises(ValueError):
        S.shard_plan(1, 16, 0, 8)  # 16 ranks cannot split 8 KV heads


def _bench_dry(*args):
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", *args],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_gpus2_spawns_two_ranks_over_gloo():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks
    (torch.distributed.run, 127.0.0.1 rendezvous), each rank takes its shard of
    the C4 requests, and rank 0 prints one line with n_gpus 2 and the
    whole-job throughput over the slowest rank's time."""
    d = _bench_dry("--gpus", "2")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["ctx"] == 131072 and d["config"]["total_requests"] == 64
    plan = d["shard_plan"]
    assert len(plan) == 2
    reqs = [s[0] for rank in plan for s in rank]
    assert sorted(reqs) == list(range(64)) and len(set(reqs)) == 64
    assert d["ms_per_step"] == 1.25  # max over ranks of the stand-in times (1.0, 1.25)
    assert d["value"] == pytest.approx(64 * 9 / 1.25e-3)


def test_bench_head_group_sharding_dry_run():
    """Fewer requests than ranks: the request's KV heads are split across its ranks."""
    d = _bench_dry("--gpus", "2", "--total-requests", "1")
    assert d["shard_plan"] == [[[0, 0, 4]], [[0, 4, 4]]]
    assert "KV-head-group" in d["config"]["parallelism"]
    assert d["value"] == pytest.approx(9 / 1.25e-3)


def test_bench_single_gpu_default_is_c2():
    d = _bench_dry()
    assert d["n_gpus"] == 1 and d["config"]["ctx"] == 65536 and d["config"]["layers"] == 32
    assert d["metric"] == ("verified query-tokens/s at 64K ctx, 8-tok draft; achieved HBM GB/s "
                           "vs peak")
