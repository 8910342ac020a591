"""Head-group shard slicing on the host, CPU tensors only.

shard_engine's per-layer slicing (_shard_layer) must give rank k exactly the
GEMV rows of its heads / groups, its groups' B_k and the wo_fused columns of
its heads, with rank offsets recomputed; the union over ranks must cover the
layer exactly once.
"""

import numpy as np
import pytest
import torch

from paper_2407_21118_b200.attention import LayerFused, _head_offsets
from paper_2407_21118_b200.errors import ValidationError
from paper_2407_21118_b200.model import (AttentionConfig, DecomposedLayer, Granularity,
                                         GroupFactors, LayerKV)
from paper_2407_21118_b200.parallel_plan import plan_groups
from paper_2407_21118_b200.sharding import ShardedAttentionConfig, _shard_layer


def _layer(n=8, dh=4, s=2, ranks_k=(3, 2, 4, 1), ranks_v=(2, 3, 1, 2), rope=True):
    d = n * dh
    G = n // s
    qd = d if rope else int(_head_offsets(ranks_k, s, n)[-1])
    rows = qd + sum(ranks_k) + sum(ranks_v)
    w1 = torch.arange(rows * d, dtype=torch.float32).reshape(rows, d)
    ko = int(_head_offsets(ranks_v, s, n)[-1])
    woT = torch.arange(d * ko, dtype=torch.float32).reshape(d, ko)
    bk = torch.arange(G * 8 * s * dh, dtype=torch.float32).reshape(G, 8, s * dh)
    i32 = lambda v: torch.tensor(list(v), dtype=torch.int32)
    L = LayerFused(wq_fused=None, wo_fused=None, q_offsets=_head_offsets(ranks_k, s, n),
                   o_offsets=_head_offsets(ranks_v, s, n), key_ranks=tuple(ranks_k),
                   value_ranks=tuple(ranks_v), s_k=s, s_v=s, rk_pad=8, rv_pad=8, ko_pad=ko, w1=w1,
                   bk=bk, woT=woT, ranks_k_dev=i32(ranks_k), latoff_k_dev=i32([0] * G),
                   ranks_v_dev=i32(ranks_v), latoff_v_dev=i32([0] * G),
                   o_off_dev=i32(_head_offsets(ranks_v, s, n)), qdim=qd,
                   q_off_dev=i32(_head_offsets(ranks_k, s, n)))
    gran = Granularity.group_head(s)
    kg = tuple(GroupFactors(np.zeros((d, r)), np.zeros((r, s * dh)), r) for r in ranks_k)
    vg = tuple(GroupFactors(np.zeros((d, r)), np.zeros((r, s * dh)), r) for r in ranks_v)
    dec = LayerKV(DecomposedLayer(gran, kg, d, dh, n), DecomposedLayer(gran, vg, d, dh, n))
    return L, dec, n, dh, s


@pytest.mark.parametrize("rope", [True, False])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_shards_partition_the_layer(rope, world):
    L, dec, n, dh, s = _layer(rope=rope)
    rk, rv = L.key_ranks, L.value_ranks
    qd = L.qdim
    lat_k = np.concatenate([[0], np.cumsum(rk)])
    lat_v = np.concatenate([[0], np.cumsum(rv)])
    seen_rows, seen_cols = [], []
    for r in range(world):
        sh = plan_groups(n, s, s, world, r)
        fl, dl = _shard_layer(L, dec, n, dh, rope, sh, torch.device("cpu"))
        h0, h1 = sh.heads[0], sh.heads[-1] + 1
        kg, vg = sh.k_groups, sh.v_groups
        q_off = _head_offsets(rk, s, n)
        q_rows = list(range(h0 * dh, h1 * dh)) if rope else list(range(q_off[h0], q_off[h1]))
        k_rows = list(range(qd + lat_k[kg[0]], qd + lat_k[kg[-1] + 1]))
        v_base = qd + lat_k[-1]
        v_rows = list(range(v_base + lat_v[vg[0]], v_base + lat_v[vg[-1] + 1]))
        want = L.w1[q_rows + k_rows + v_rows]
        assert torch.equal(fl.w1, want)
        assert fl.qdim == len(q_rows)
        assert torch.equal(fl.bk, L.bk[kg[0]:kg[-1] + 1])
        o_off = _head_offsets(rv, s, n)
        assert torch.equal(fl.woT[:, :o_off[h1] - o_off[h0]], L.woT[:, o_off[h0]:o_off[h1]])
        assert fl.key_ranks == tuple(rk[g] for g in kg)
        assert fl.q_offsets == _head_offsets(fl.key_ranks, s, h1 - h0)
        assert len(dl.key.groups) == len(kg) and dl.key.n_heads == h1 - h0
        seen_rows += q_rows + k_rows + v_rows
        seen_cols += list(range(o_off[h0], o_off[h1]))
    assert sorted(seen_rows) == list(range(L.w1.shape[0]))  # every GEMV row exactly once
    assert sorted(seen_cols) == list(range(L.woT.shape[1]))


def test_sharded_config_validation():
    ShardedAttentionConfig(4096, 8, 128, layers=1, rope=True, world=4, rank=1)
    with pytest.raises(ValidationError):
        ShardedAttentionConfig(4096, 8, 128, layers=1, world=2)
    with pytest.raises(ValidationError):
        plan_groups(32, 4, 4, 3, 0)  # 8 head blocks do not split over 3 ranks
    assert AttentionConfig(4096, 32, 128, layers=1).d_model == 4096
