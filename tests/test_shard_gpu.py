"""C5 (Llama-3-70B attention: 64 query / 8 KV heads, N 8192, d 128) sharded by
KV-head group exactly as bench.py --workload c5 runs it: two processes (gloo,
both on cuda:0 — the box has one GPU), each calling fa3b_fwd through
shard_forward on strided views of its heads only. The union of the two ranks'
slices must equal the single-call output bitwise, in BF16 and in FP8 (K5
operands and per-block scales sliced the same way)."""
from __future__ import annotations

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B, N, H, HKV, D = 1, 8192, 64, 8, 128


def _inputs(fp8):
    from paper_2407_08608_b200 import api
    gen = torch.Generator(device="cuda").manual_seed(70)
    q = torch.randn(B, N, H, D, device="cuda", generator=gen).bfloat16()
    k, v = (torch.randn(B, N, HKV, D, device="cuda", generator=gen).bfloat16() for _ in range(2))
    if not fp8:
        return (q, k, v), {}
    (q8, sq), (k8, sk) = (api.fp8_prepare(x, block_rows=128, hadamard=True, seed=5) for x in (q, k))
    v8, sv = api.fp8_prepare(v, block_rows=128, hadamard=False)
    return (q8, k8, v8), dict(q_scale=sq, k_scale=sk, v_scale=sv)


def _worker(rank, world, port, fp8, out):
    from paper_2407_08608_b200 import api
    from paper_2407_08608_b200.shard import partition, shard_forward
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        (q, k, v), scales = _inputs(fp8)
        o = torch.zeros(B, N, H, D, device="cuda", dtype=torch.bfloat16)
        lse = torch.zeros(B, H, N, device="cuda", dtype=torch.float32)
        calls = shard_forward(api.fwd, q, k, v, o, lse, partition(B, HKV, world)[rank], HKV,
                              causal=True, **scales)
        torch.cuda.synchronize()
        o_h, l_h = o.float().cpu(), lse.cpu()
        dist.all_reduce(o_h)  # disjoint slices, zeros elsewhere: the sum is the union
        dist.all_reduce(l_h)
        out[rank] = (calls, o_h, l_h)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16", "e4m3"])
def test_c5_head_sharded_two_ranks_bitwise(cuda, fp8):
    from paper_2407_08608_b200 import api
    world = 2
    port = 33500 + (os.getpid() % 2000) + int(fp8)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, fp8, out), nprocs=world, join=True)
        res = dict(out)
    (q, k, v), scales = _inputs(fp8)
    o, lse = api.fwd(q, k, v, causal=True, **scales)
    for r in range(world):
        calls, o_r, l_r = res[r]
        assert calls == 1
        assert torch.equal(o_r, o.float().cpu())
        assert torch.equal(l_r, lse.cpu())
