"""Batch x head sharding across GPUs.

Attention has no exchange step between (batch, head) units, so multi-GPU
runs partition the units and never call a data-path collective. Units are
(batch, KV-head) pairs, each carrying its whole GQA group of query heads, so
K/V are never duplicated across GPUs. The partition is contiguous in
(batch-major, kv-head) order and balanced to within one unit.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    units: tuple  # ((batch, kv_head), ...)

    def batch_heads(self, group: int):
        """(batch, query head) pairs this shard computes."""
        return [(b, kv * group + g) for b, kv in self.units for g in range(group)]

    def batch_range(self, heads_kv: int):
        """(first batch, last batch + 1) when the shard is whole batches, else None."""
        if not self.units or len(self.units) % heads_kv or self.units[0][1] != 0:
            return None
        return self.units[0][0], self.units[-1][0] + 1


def partition(batch: int, heads_kv: int, world: int) -> list[Shard]:
    if batch <= 0 or heads_kv <= 0 or world <= 0:
        raise ValueError("partition: batch, heads_kv and world must be positive")
    units = [(b, h) for b in range(batch) for h in range(heads_kv)]
    base, extra = divmod(len(units), world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(Shard(r, tuple(units[start:start + n])))
        start += n
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank time over the process group (the timing rule for
    multi-GPU numbers); identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
