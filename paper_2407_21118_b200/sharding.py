"""Head-group sharding of the GPU engine.

Rank k of `world` owns the contiguous head block of ``parallel_plan.plan_groups``
(whole key and value groups): its slice of the layer GEMV rows (W_q columns,
or wq_fused columns with rope off, plus its groups' A_k / A_v), its groups'
B_k, the wo_fused rows of its heads and its groups' latent stores.  A decode
step on a shard produces the partial layer output
``sum_{i in heads_k} ctx_i @ wo_fused_i``; the layer output is the sum over
ranks -- one all-reduce of [B x d] per layer (``_Session.allreduce``), which
also replicates x for the next layer.  Nothing else crosses ranks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .attention import (FusedWeights, LatentKVCache, LayerFused, _SideStore, _head_offsets,
                        _round_up, _torch)
from .errors import ValidationError
from .model import AttentionConfig, DecomposedLayer, LayerKV
from .parallel_plan import plan_groups


@dataclass(frozen=True)
class ShardedAttentionConfig(AttentionConfig):
    """AttentionConfig of one shard: n_heads is the LOCAL head count, d_model
    stays the full model width (x and the layer output are replicated)."""

    world: int = 1
    rank: int = 0

    def __post_init__(self):
        if self.d_model != self.world * self.n_heads * self.head_dim:
            raise ValidationError(f"d_model {self.d_model} != world*local_heads*head_dim")
        if self.layers < 1:
            raise ValidationError(f"layers must be >= 1, got {self.layers}")


def _shard_layer(L: LayerFused, dec: LayerKV, n: int, dh: int, rope: bool, shard, dev):
    # pure index slicing on whatever device L lives on (host-testable);
    # shard_engine itself requires CUDA via the cache it builds
    import torch
    h0, h1 = shard.heads[0], shard.heads[-1] + 1
    kg, vg = list(shard.k_groups), list(shard.v_groups)
    rk, rv = list(L.key_ranks), list(L.value_ranks)
    qdim = L.qdim or n * dh
    q_off = _head_offsets(rk, L.s_k, n)
    if rope:
        q_rows = torch.arange(h0 * dh, h1 * dh, device=dev)
    else:
        q_rows = torch.arange(q_off[h0], q_off[h1], device=dev)
    lat_k = np.concatenate([[0], np.cumsum(rk)])
    lat_v = np.concatenate([[0], np.cumsum(rv)])
    k_rows = torch.arange(qdim + int(lat_k[kg[0]]), qdim + int(lat_k[kg[-1] + 1]), device=dev)
    v_base = qdim + int(lat_k[-1])
    v_rows = torch.arange(v_base + int(lat_v[vg[0]]), v_base + int(lat_v[vg[-1] + 1]), device=dev)
    w1 = L.w1.index_select(0, torch.cat([q_rows, k_rows, v_rows])).contiguous()
    bk = L.bk[kg[0]:kg[-1] + 1].contiguous()
    o_off = _head_offsets(rv, L.s_v, n)
    ko = o_off[h1] - o_off[h0]
    ko_pad = _round_up(ko, 8)
    woT = torch.zeros(L.woT.shape[0], ko_pad, dtype=L.woT.dtype, device=dev)
    woT[:, :ko] = L.woT[:, o_off[h0]:o_off[h1]]
    n_loc = h1 - h0
    rk_s, rv_s = tuple(rk[g] for g in kg), tuple(rv[g] for g in vg)
    i32 = lambda v: torch.tensor(list(v), dtype=torch.int32, device=dev)
    lk = np.concatenate([[0], np.cumsum(rk_s)[:-1]]).astype(int)
    lv = np.concatenate([[0], np.cumsum(rv_s)[:-1]]).astype(int)
    qd = n_loc * dh if rope else int(q_off[h1] - q_off[h0])
    fl = LayerFused(
        wq_fused=None, wo_fused=None,
        q_offsets=_head_offsets(rk_s, L.s_k, n_loc), o_offsets=_head_offsets(rv_s, L.s_v, n_loc),
        key_ranks=rk_s, value_ranks=rv_s, s_k=L.s_k, s_v=L.s_v, rk_pad=L.rk_pad, rv_pad=L.rv_pad,
        ko_pad=ko_pad, w1=w1, bk=bk, woT=woT, ranks_k_dev=i32(rk_s), latoff_k_dev=i32(lk),
        ranks_v_dev=i32(rv_s), latoff_v_dev=i32(lv),
        o_off_dev=i32(_head_offsets(rv_s, L.s_v, n_loc)), qdim=qd,
        q_off_dev=i32(_head_offsets(rk_s, L.s_k, n_loc)))
    key = DecomposedLayer(dec.key.granularity, tuple(dec.key.groups[g] for g in kg),
                          dec.key.d_model, dh, n_loc)
    value = DecomposedLayer(dec.value.granularity, tuple(dec.value.groups[g] for g in vg),
                            dec.value.d_model, dh, n_loc)
    return fl, LayerKV(key=key, value=value)


def shard_engine(fused: FusedWeights, cache: LatentKVCache, rank: int, world: int):
    """Slice a (fused weights, cache) pair to the head block of `rank`.

    Returns (fused_shard, cache_shard) whose config is a
    ShardedAttentionConfig; the cache shard copies the owned groups' rows.
    """
    cfg = cache.config
    n, dh = cfg.n_heads, cfg.head_dim
    layers, decs = [], []
    for li, L in enumerate(fused.layers):
        dec = cache.decomposed[li]
        shard = plan_groups(n, dec.key.granularity.group_size, dec.value.granularity.group_size,
                            world, rank)
        fl, dl = _shard_layer(L, dec, n, dh, cfg.rope, shard, cache.device)
        layers.append(fl)
        decs.append((dl, shard))
    n_loc = len(decs[0][1].heads)
    scfg = ShardedAttentionConfig(cfg.d_model, n_loc, dh, layers=cfg.layers, rope=cfg.rope,
                                  rope_base=cfg.rope_base, world=world, rank=rank)
    fs = FusedWeights(layers=tuple(layers), config=scfg, dtype=fused.dtype,
                      theta_dev=fused.theta_dev, theta=fused.theta)
    cs = LatentKVCache([d for d, _ in decs], scfg, cache.bits, dtype=cache.dtype,
                       batch=cache.batch, capacity=cache.capacity, device=cache.device,
                       score_kernel=cache.score_kernel)
    for li, (_, shard) in enumerate(decs):
        stores = list(cs._stores[li])
        for side, groups in ((0, shard.k_groups), (1, shard.v_groups)):
            src, dst = cache._stores[li][side], stores[side]
            if dst.r_pad != src.r_pad:
                # non-uniform ranks: the shard's widest group may be narrower
                # than the source store's row; keep the source row width
                dst = _SideStore(dst.ranks, dst.bits, src.r_pad, dst.batch, dst.cap, dst.dtype,
                                 cache.device)
                stores[side] = dst
            g0, g1 = groups[0], groups[-1] + 1
            dst.rows.copy_(src.rows[:, g0:g1])
            for k in ("scales", "zps", "scales64", "zps64"):
                if getattr(src, k) is not None:
                    getattr(dst, k).copy_(getattr(src, k)[:, g0:g1])
        cs._stores[li] = tuple(stores)
    cs.t = cache.t
    return fs, cs


def attach_allreduce(target, fn) -> None:
    """Install the per-layer partial-output reduction on a shard: fn(x)
    reduces the [B x d] layer output in place on the current stream (e.g. an
    NCCL all-reduce).  ``target`` is the shard's LatentKVCache (or a session
    of it); the hook is kept on the cache, so sessions rebuilt after capacity
    growth keep reducing.  The step graph is re-captured with it."""
    cache = target if isinstance(target, LatentKVCache) else target.cache
    cache._allreduce = fn
    if cache._session is not None:
        cache._session.allreduce = fn
        cache._session.graph = None
