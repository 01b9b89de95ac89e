"""Sharding of the path across GPUs of one node (one process per GPU).

The path shards by prompt (batch) and by KV head:
  * batch sharding: each rank owns whole prompts and runs K1..K5 alone --
    no collective at all (replicas on disjoint data);
  * KV-head sharding: K1, K3, K4, K5 are local to the rank's heads, but K2's
    gamma' is a mean over ALL query heads of a layer (reference
    sparsity.py:41-43).  The one exchange step: every rank writes its heads'
    integer below-threshold counts into a zeroed [B, L, Hq] buffer and the
    ranks sum it (NCCL all-reduce over NVLink; gloo in the CPU tests).
    Integer sums are exact and order-free, so every rank then runs K2 on
    identical counts and gets the unsharded budgets bit for bit -- unlike an
    all-reduce of float gamma sums, which would change numpy's pairwise
    summation order.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ValidationError


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    num_kv_heads: int       # global Hkv
    group_size: int         # G = Hq / Hkv

    def __post_init__(self):
        if not 0 <= self.rank < self.world:
            raise ValidationError(f"rank: must be in [0, {self.world}), got {self.rank}")
        if self.num_kv_heads % self.world:
            raise ValidationError(
                f"world: {self.world} ranks cannot split {self.num_kv_heads} KV heads evenly")

    @property
    def kv_per_rank(self) -> int:
        return self.num_kv_heads // self.world

    @property
    def kv_range(self) -> tuple[int, int]:
        lo = self.rank * self.kv_per_rank
        return lo, lo + self.kv_per_rank

    @property
    def q_range(self) -> tuple[int, int]:
        lo, hi = self.kv_range
        return lo * self.group_size, hi * self.group_size

    @property
    def num_query_heads(self) -> int:
        return self.num_kv_heads * self.group_size


def shard_batch(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous prompt range [lo, hi) of `rank` (sizes differ by at most one)."""
    if not 0 <= rank < world:
        raise ValidationError(f"rank: must be in [0, {world}), got {rank}")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def exchange_head_counts(local_counts, shard: HeadShard, group=None):
    """Sum the per-head below-threshold counts of all ranks.

    local_counts: int64 tensor [B, L, Hq_local] (this rank's heads).
    Returns int64 [B, L, Hq] identical on every rank.
    """
    import torch
    import torch.distributed as dist

    b, l, hq_local = local_counts.shape
    lo, hi = shard.q_range
    if hq_local != hi - lo:
        raise ValidationError(f"local_counts: expected {hi - lo} heads, got {hq_local}")
    full = torch.zeros((b, l, shard.num_query_heads), dtype=torch.int64, device=local_counts.device)
    full[:, :, lo:hi] = local_counts
    if shard.world > 1:
        if full.is_cuda and dist.get_backend(group) == "gloo":
            host = full.cpu()     # gloo reduces host memory (the CPU tests' backend)
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            full.copy_(host)
        else:
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full
