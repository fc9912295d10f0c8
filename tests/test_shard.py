"""Multi-GPU sharding logic on CPU: the partition, and the gloo world-size-2
run of the same rank-local code path bench.py uses (no GPU needed)."""
from __future__ import annotations

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_08608_b200.shard import max_over_ranks, partition


@pytest.mark.parametrize("B,Hkv,world", [(1, 8, 1), (1, 8, 2), (1, 8, 8), (2, 16, 4), (3, 5, 4),
                                         (1, 1, 2)])
def test_partition_covers_disjoint_balanced(B, Hkv, world):
    shards = partition(B, Hkv, world)
    units = [u for s in shards for u in s.units]
    assert sorted(units) == [(b, h) for b in range(B) for h in range(Hkv)]
    sizes = [len(s.units) for s in shards]
    assert max(sizes) - min(sizes) <= 1


def test_gqa_groups_stay_whole():
    # C5: 64 query heads over 8 KV heads on 8 GPUs -> one KV head (8 q heads) each
    shards = partition(1, 8, 8)
    for r, s in enumerate(shards):
        assert s.units == ((0, r),)
        assert s.batch_heads(8) == [(0, 8 * r + g) for g in range(8)]


def test_weak_scaling_batch_ranges():
    # bench.py: global batch 2 * world, 16 heads -> whole batches per rank
    for world in (1, 2, 4, 8):
        shards = partition(2 * world, 16, world)
        assert [s.batch_range(16) for s in shards] == [(2 * r, 2 * r + 2) for r in range(world)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = partition(2 * world, 16, world)[rank]
        # every rank sees a disjoint shard; gather to check coverage
        mine = torch.tensor([b * 16 + h for b, h in shard.units])
        got = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(got, mine)
        t = max_over_ranks(1.5 + rank)
        out[rank] = (sorted(torch.cat(got).tolist()), t)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_and_max_timing():
    world = 2
    port = 29500 + (os.getpid() % 2000)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        units, t = res[r]
        assert units == list(range(2 * world * 16))
        assert t == 2.5  # max over ranks of 1.5 + rank
