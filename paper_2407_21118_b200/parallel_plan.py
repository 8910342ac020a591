"""Head-group sharding plan for one decode step across ranks.

Head groups are independent until the per-layer output sum: with B_v folded
into W_o (attention.py:214-221), rank k owning groups G_k produces

    out_k = sum_{i in heads(G_k)} ctx_i @ wo_fused[o_off[i]:o_off[i+1]]

and the layer output is sum_k out_k -- one all-reduce of [B x d] per layer,
which also replicates x for the next layer.  Everything a rank needs is the
slice of W_q columns of its heads, its groups' (A_k, B_k, A_v) factors, the
wo_fused rows of its heads and its groups' latent stores.

Batch sharding (replicas) needs no collective at all; bench.py uses it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class GroupShard:
    rank: int
    world: int
    k_groups: tuple  # key groups owned
    v_groups: tuple  # value groups owned
    heads: tuple     # heads whose softmax/value path this rank computes


def plan_groups(n_heads: int, s_k: int, s_v: int, world: int, rank: int) -> GroupShard:
    """Contiguous partition of head groups.  Key and value granularities may
    differ (attention.py:210-211); heads are assigned by the coarser grouping
    so that a rank owns whole K and V groups for every head it scores."""
    if world < 1 or not (0 <= rank < world):
        raise ValidationError(f"bad rank {rank} of world {world}")
    s = max(s_k, s_v)
    if s % s_k or s % s_v or n_heads % s:
        raise ValidationError(f"group sizes {s_k}/{s_v} do not nest for {n_heads} heads")
    n_blocks = n_heads // s
    if n_blocks % world:
        raise ValidationError(f"{n_blocks} head blocks do not split over {world} ranks")
    per = n_blocks // world
    heads = tuple(range(rank * per * s, (rank + 1) * per * s))
    kg = tuple(sorted({h // s_k for h in heads}))
    vg = tuple(sorted({h // s_v for h in heads}))
    return GroupShard(rank=rank, world=world, k_groups=kg, v_groups=vg, heads=heads)


def shard_layer_arrays(wq: np.ndarray, wo_fused: np.ndarray, o_off, ak, bk, av, bv,
                       head_dim: int, shard: GroupShard):
    """Slice one layer's arrays to a shard (host-side, offline)."""
    dh = head_dim
    cols = np.concatenate([np.arange(h * dh, (h + 1) * dh) for h in shard.heads])
    rows = np.concatenate([np.arange(o_off[h], o_off[h + 1]) for h in shard.heads])
    return dict(
        wq=wq[:, cols],
        wo_fused=wo_fused[rows, :],
        ak=[ak[g] for g in shard.k_groups], bk=[bk[g] for g in shard.k_groups],
        av=[av[g] for g in shard.v_groups], bv=[bv[g] for g in shard.v_groups],
    )


def allreduce_sum(t, group=None):
    """Sum of partial layer outputs over the ranks (the only exchange)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
