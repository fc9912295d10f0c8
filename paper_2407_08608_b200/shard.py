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

    def calls(self, heads_kv: int):
        """The shard as a few rectangular (b0, b1, kv0, kv1) blocks of the
        [batch, kv-head] grid, each one fa3b_fwd on strided views
        q[b0:b1, :, kv0*g:kv1*g], k/v[b0:b1, :, kv0:kv1] (no copies): runs of
        consecutive KV heads within a batch, with runs of whole batches merged."""
        runs = []
        for b, kv in self.units:
            if runs and runs[-1][0] == b and runs[-1][2] == kv:
                runs[-1][2] = kv + 1
            else:
                runs.append([b, kv, kv + 1])
        out = []
        for b, kv0, kv1 in runs:
            whole = kv0 == 0 and kv1 == heads_kv
            if (whole and out and out[-1][1] == b and out[-1][2] == 0
                    and out[-1][3] == heads_kv):
                out[-1] = (out[-1][0], b + 1, 0, heads_kv)
            else:
                out.append((b, b + 1, kv0, kv1))
        return out


def shard_forward(fwd, q, k, v, o, lse, shard: Shard, heads_kv: int, **kw) -> int:
    """Run this rank's part of one forward: one ``fwd`` call (api.fwd or any
    function with its signature) per block of ``shard.calls``, on strided
    views into the full [B, N, H, D] tensors, writing into views of ``o`` and
    ``lse`` [B, H, N]. FP8 scale tensors ([B, H(kv), blocks], passed as
    q_scale / k_scale / v_scale) are sliced the same way. No copies, no
    collectives. Returns the number of calls."""
    g = q.shape[2] // heads_kv
    n = 0
    for b0, b1, kv0, kv1 in shard.calls(heads_kv):
        extra = dict(kw)
        for name, per_q in (("q_scale", True), ("k_scale", False), ("v_scale", False)):
            if kw.get(name) is not None:
                lo, hi = (kv0 * g, kv1 * g) if per_q else (kv0, kv1)
                extra[name] = kw[name][b0:b1, lo:hi]
        fwd(q[b0:b1, :, kv0 * g:kv1 * g], k[b0:b1, :, kv0:kv1], v[b0:b1, :, kv0:kv1],
            out=o[b0:b1, :, kv0 * g:kv1 * g], lse=lse[b0:b1, kv0 * g:kv1 * g], **extra)
        n += 1
    return n


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
