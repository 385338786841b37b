"""Multi-GPU sharding of the SentenceKV hot path.

Every (sequence b, KV head g) unit is independent through P1-P3 and D1-D4 (selection is ranked per
KV head, reading A9/A15), so ranks split the units with no exchange on the data path.  The one
collective is an all-gather of the per-head attention outputs of each layer (the next layer's
output projection needs every head), done with torch.distributed (NCCL over NVLink on B200).

A plan splits the KV heads into `head_shards` contiguous groups and the batch into `batch_shards`
contiguous groups; rank r holds batch shard r // head_shards and head shard r % head_shards.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    batch: int
    kv_heads: int
    q_heads: int
    batch_shards: int
    head_shards: int

    @property
    def grp(self) -> int:
        return self.q_heads // self.kv_heads

    @property
    def batch_count(self) -> int:
        return self.batch // self.batch_shards

    @property
    def kv_head_count(self) -> int:
        return self.kv_heads // self.head_shards

    @property
    def batch_begin(self) -> int:
        return (self.rank // self.head_shards) * self.batch_count

    @property
    def kv_head_begin(self) -> int:
        return (self.rank % self.head_shards) * self.kv_head_count

    @property
    def q_head_begin(self) -> int:
        return self.kv_head_begin * self.grp

    @property
    def q_head_count(self) -> int:
        return self.kv_head_count * self.grp

    def ctx_kwargs(self) -> dict:
        """Arguments of paper_2504_00970_b200.SentenceKV for this rank's shard."""
        return dict(batch=self.batch, kv_heads=self.kv_heads, q_heads=self.q_heads,
                    kv_head_begin=self.kv_head_begin, kv_head_count=self.kv_head_count,
                    batch_begin=self.batch_begin, batch_count=self.batch_count)


def plan(batch: int, kv_heads: int, q_heads: int, world: int, rank: int, strategy: str = "heads") -> ShardPlan:
    """Shard plan for `world` ranks.

    strategy "heads": KV heads over as many ranks as divide G (the rest of the ranks split the batch);
    "batch": batch over the ranks (heads kept whole while B allows, else heads take the rest).
    Raises ValueError when the shapes cannot be split evenly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if q_heads % kv_heads:
        raise ValueError("q_heads must be a multiple of kv_heads")
    divisors = [h for h in range(world, 0, -1) if world % h == 0]
    if strategy == "heads":
        hs = next(h for h in divisors if kv_heads % h == 0)
        bs = world // hs
    elif strategy == "batch":
        bs = next((b for b in divisors if batch % b == 0), 1)
        hs = world // bs
    else:
        raise ValueError(f"unknown strategy {strategy}")
    if kv_heads % hs or batch % bs:
        raise ValueError(f"cannot split B={batch}, G={kv_heads} over {world} ranks ({bs} x {hs})")
    return ShardPlan(world, rank, batch, kv_heads, q_heads, bs, hs)


def assemble(gathered: torch.Tensor, p: ShardPlan) -> torch.Tensor:
    """Rank-major all-gather result [world][B_loc][Hq_loc][d] -> [B][Hq][d]."""
    d = gathered.shape[-1]
    x = gathered.view(p.batch_shards, p.head_shards, p.batch_count, p.q_head_count, d)
    return x.permute(0, 2, 1, 3, 4).reshape(p.batch, p.q_heads, d)


def all_gather_outputs(out_local: torch.Tensor, p: ShardPlan, group=None, gathered: torch.Tensor = None):
    """The per-layer exchange: all-gather every rank's attention output (fp32 [B_loc][Hq_loc][d])
    into `gathered` ([world][B_loc][Hq_loc][d], rank-major; allocated if None) and return it.
    Use assemble() for the [B][Hq][d] view."""
    import torch.distributed as dist

    if gathered is None:
        gathered = torch.empty((p.world,) + tuple(out_local.shape), dtype=out_local.dtype, device=out_local.device)
    if p.world == 1:
        gathered[0].copy_(out_local)
        return gathered
    # concatenated along dim 0 (the form every backend accepts), viewed as [world][...]
    flat = gathered.view((p.world * out_local.shape[0],) + tuple(out_local.shape[1:]))
    dist.all_gather_into_tensor(flat, out_local.contiguous(), group=group)
    return gathered
