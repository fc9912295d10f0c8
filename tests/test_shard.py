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


@pytest.mark.parametrize("B,Hkv,world", [(1, 8, 2), (1, 8, 8), (4, 16, 2), (3, 16, 2), (3, 5, 4)])
def test_calls_are_rectangles_covering_the_shard(B, Hkv, world):
    for s in partition(B, Hkv, world):
        got = sorted((b, kv) for b0, b1, kv0, kv1 in s.calls(Hkv)
                     for b in range(b0, b1) for kv in range(kv0, kv1))
        assert got == sorted(s.units)
        for b0, b1, kv0, kv1 in s.calls(Hkv):
            # partial head ranges only within one batch (keeps the LSE view contiguous)
            assert b1 - b0 == 1 or (kv0, kv1) == (0, Hkv)
    # C5 on 2/4/8 ranks: one call per rank over a contiguous KV-head range
    for world in (2, 4, 8):
        assert [s.calls(8) for s in partition(1, 8, world)] == [
            [(0, 1, 8 // world * r, 8 // world * (r + 1))] for r in range(world)]


def _oracle_fwd(port):
    """A fwd with api.fwd's signature on CPU tensors, one oracle call per (b, h)."""
    import numpy as np

    def fwd(q, k, v, out, lse, causal=False):
        B, N, H, D = q.shape
        g = H // k.shape[2]
        for b in range(B):
            for h in range(H):
                o, l, _ = port.flash_fwd(q[b, :, h].numpy(), k[b, :, h // g].numpy(),
                                         v[b, :, h // g].numpy(), causal=causal, tile=(64, 64))
                out[b, :, h] = torch.from_numpy(np.ascontiguousarray(o))
                lse[b, h] = torch.from_numpy(l)
    return fwd


def _views_worker(rank, world, port_no, out):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import oracle as O
    from paper_2407_08608_b200.shard import shard_forward
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, N, H, Hkv, D = 1, 96, 8, 4, 16
        gen = torch.Generator().manual_seed(7)
        q = torch.randn(B, N, H, D, generator=gen, dtype=torch.float64)
        k, v = (torch.randn(B, N, Hkv, D, generator=gen, dtype=torch.float64) for _ in range(2))
        o = torch.zeros_like(q)
        lse = torch.zeros(B, H, N, dtype=torch.float64)
        shard = partition(B, Hkv, world)[rank]
        calls = shard_forward(_oracle_fwd(O.Port()), q, k, v, o, lse, shard, Hkv, causal=True)
        # the whole job = the sum of the ranks' disjoint slices (zeros elsewhere)
        dist.all_reduce(o)
        dist.all_reduce(lse)
        out[rank] = (calls, o, lse)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_ranks_compute_their_head_slices(port):
    """The bench's rank-local path (shard_forward over strided views) on two
    gloo ranks, each running the CPU oracle on its KV-head groups: the union of
    the slices equals the single-process result bitwise."""
    import numpy as np
    world = 2
    port_no = 31500 + (os.getpid() % 2000)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_views_worker, args=(world, port_no, out), nprocs=world, join=True)
        res = dict(out)
    gen = torch.Generator().manual_seed(7)
    q = torch.randn(1, 96, 8, 16, generator=gen, dtype=torch.float64)
    k, v = (torch.randn(1, 96, 4, 16, generator=gen, dtype=torch.float64) for _ in range(2))
    o = torch.zeros_like(q)
    lse = torch.zeros(1, 8, 96, dtype=torch.float64)
    _oracle_fwd(port)(q, k, v, o, lse, causal=True)
    for r in range(world):
        calls, o_r, l_r = res[r]
        assert calls == 1
        assert torch.equal(o_r, o) and torch.equal(l_r, lse)
    assert np.isfinite(lse.numpy()).all()
