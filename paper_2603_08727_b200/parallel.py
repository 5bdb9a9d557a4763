"""Multi-GPU plumbing: unit sharding and the one prefill exchange.

A unit is (sequence, layer, KV head); units are independent given rho (R11, R20), so the
decode loop needs no collective.  Ranks take sequence-major blocks first, then KV heads
(minimising the number of ranks per sequence).  When a sequence's KV heads span ranks,
Eq. 3's column sums must be summed over them before the moments (collective C1):
arkv_prefill_begin -> all_reduce(colsum) -> arkv_prefill_finish.
"""
from __future__ import annotations

from typing import Dict


def shard_units(batch: int, n_kv_heads: int, world: int, rank: int) -> Dict[str, int]:
    """Sequence-major block partition of batch x n_kv_heads units over `world` ranks.
    Returns {seq_lo, seq_hi, kvh_lo, kvh_hi} (half-open).  If world <= batch, every rank
    holds whole sequences (world must divide batch); otherwise each sequence is split over
    world / batch ranks by KV head (which must divide n_kv_heads)."""
    if world <= batch:
        if batch % world:
            raise ValueError("world must divide batch")
        per = batch // world
        return dict(seq_lo=rank * per, seq_hi=(rank + 1) * per, kvh_lo=0, kvh_hi=n_kv_heads)
    if world % batch:
        raise ValueError("batch must divide world")
    rps = world // batch            # ranks per sequence
    if n_kv_heads % rps:
        raise ValueError("ranks per sequence must divide n_kv_heads")
    hp = n_kv_heads // rps
    seq = rank // rps
    j = rank % rps
    return dict(seq_lo=seq, seq_hi=seq + 1, kvh_lo=j * hp, kvh_hi=(j + 1) * hp)


def sequence_group_ranks(batch: int, world: int, rank: int):
    """Ranks that share this rank's sequences (the C1 all-reduce group)."""
    if world <= batch:
        return [rank]
    rps = world // batch
    base = (rank // rps) * rps
    return list(range(base, base + rps))


def sequence_group(batch: int, world: int, rank: int):
    """The process group of the ranks sharing this rank's sequence (C1), or None when the
    rank holds whole sequences.  Every rank creates every group, in the same order
    (torch.distributed.new_group is collective)."""
    import torch.distributed as dist
    if world <= batch:
        return None
    mine = None
    rps = world // batch
    for r0 in range(0, world, rps):
        ranks = list(range(r0, r0 + rps))
        g = dist.new_group(ranks)
        if rank in ranks:
            mine = g
    return mine


def prefill_sharded(cache, q_win, k, v, group=None, rho_override=None):
    """Prefill of a KV-head shard: local passes + column sums, C1 all-reduce over the
    ranks sharing the sequences, then moments / rho / ingest / tailor."""
    import torch.distributed as dist
    colsum = cache.arkv_prefill_begin(q_win, k)
    if group is not None:
        dist.all_reduce(colsum, op=dist.ReduceOp.SUM, group=group)
    return cache.arkv_prefill_finish(k, v, colsum, rho_override=rho_override)
