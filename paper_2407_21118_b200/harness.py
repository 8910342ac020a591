"""Synthetic-input and direct-fill helpers for parity tests and the bench.

The reference fills caches token by token (palu_prefill is O(T^2),
attention.py:469-494).  For long contexts the bench and tests fill the
latent store directly with rows H_g = X @ A_g, exactly what T
calls of _append_latents (attention.py:343-347) would store for fixed
inputs.  Rows are computed in fp64 on the GPU and written in the cache's own
format: raw storage dtype, or quantised with the same bit-exact device
quantiser the decode step uses (palu_quantize_rows + palu_pack_rows).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .attention import FP_BITS, LatentKVCache, _ptr, _stream, _torch
from .model import (AttentionConfig, DecomposedLayer, Granularity, GroupFactors, LayerKV,
                    LayerWeights, ModelWeights, as_array, fuse_hadamard)


def _fill_side(side, g, b, t0, h64):
    """Write fp64 latent rows h64 [T, r] into group g, batch b, rows t0.."""
    torch = _torch()
    T, r = h64.shape
    if side.bits == FP_BITS:
        side.rows[b, g, t0:t0 + T, :r].copy_(h64.to(side.rows.dtype))
        return
    codes = torch.empty(T, r, dtype=torch.uint8, device=h64.device)
    s64 = torch.empty(T, dtype=torch.float64, device=h64.device)
    z64 = torch.empty(T, dtype=torch.int64, device=h64.device)
    st = _stream()
    _lib.call("palu_quantize_rows", _ptr(h64.contiguous()), T, r, side.bits, _ptr(codes), _ptr(s64),
              _ptr(z64), st)
    full = torch.zeros(T, side.r_pad, dtype=torch.uint8, device=h64.device)
    full[:, :r] = codes
    packed = torch.empty(T, side.r_pad * side.bits // 8, dtype=torch.uint8, device=h64.device)
    _lib.call("palu_pack_rows", _ptr(full), T, side.r_pad, side.bits, _ptr(packed), st)
    side.rows[b, g, t0:t0 + T].copy_(packed)
    side.scales[b, g, t0:t0 + T].copy_(s64.float())
    side.zps[b, g, t0:t0 + T].copy_(z64.float())
    side.scales64[b, g, t0:t0 + T].copy_(s64)
    side.zps64[b, g, t0:t0 + T].copy_(z64)


def fill_cache_direct(cache: LatentKVCache, li: int, x_rows, b: int | None = None,
                      chunk: int = 8192) -> None:
    """Append rows x_rows @ A_g (every group, both sides) at the cache tail of
    layer li (batch row b, or all rows).  Advances nothing: call
    ``set_cache_t`` once every layer is filled."""
    torch = _torch()
    kv = cache.decomposed[li]
    K, V = cache._stores[li]
    dev = cache.device
    x = torch.from_numpy(np.asarray(x_rows, np.float64)) if isinstance(x_rows, np.ndarray) else x_rows
    x = x.to(dev, torch.float64)
    T = x.shape[0]
    cache.reserve(cache.t + T)
    K, V = cache._stores[li]
    bs = range(cache.batch) if b is None else [b]
    for side, dec in ((K, kv.key), (V, kv.value)):
        for g, gf in enumerate(dec.groups):
            a = torch.from_numpy(as_array(gf.a)).to(dev)
            for c0 in range(0, T, chunk):
                h = x[c0:c0 + chunk] @ a
                for bb in bs:
                    _fill_side(side, g, bb, cache.t + c0, h)


def set_cache_t(cache: LatentKVCache, t: int) -> None:
    cache.t = t
    if cache._session is not None:
        cache._session.t_dev.fill_(t)


# ---------------------------------------------------------------------------
# Seeded synthetic model; same seeds/scales as
# oracle.palu_oracle.synth_layer, generated on the GPU.
# ---------------------------------------------------------------------------
_MASK = (1 << 64) - 1


def random_matrix_gpu(rows: int, cols: int, seed: int, row0: int = 0, device=None):
    """core.py:331-356 counter-based uniform [-1, 1) matrix, bit-exact, on the GPU.

    uint64 arithmetic is emulated in int64 torch ops (wrapping multiply and
    logical shifts), so the values equal the reference's bit for bit.
    """
    torch = _torch()
    dev = device or torch.device("cuda")

    def s64(v):
        v &= _MASK
        return v - (1 << 64) if v >= (1 << 63) else v

    def lsr(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)

    def mix(z):
        z = z + s64(0x9E3779B97F4A7C15)
        z = (z ^ lsr(z, 30)) * s64(0xBF58476D1CE4E5B9)
        z = (z ^ lsr(z, 27)) * s64(0x94D049BB133111EB)
        return z ^ lsr(z, 31)

    base = s64(seed ^ (0 * 0x517CC1B727220A95))
    r = (torch.arange(row0, row0 + rows, dtype=torch.int64, device=dev) + 1) * s64(0xD6E8FEB86659FD93)
    c = (torch.arange(cols, dtype=torch.int64, device=dev) + 1) * s64(0xA5A5A5A5B4B4B4B5)
    state = mix(base ^ r)[:, None] ^ c[None, :]
    h = mix(state)
    u = lsr(h, 11).double() * (2.0 ** -53)
    return 2.0 * u - 1.0


def synth_model(d, n_heads, head_dim, s_k, ranks_k, s_v, ranks_v, seed, layers=1,
                hadamard_fused=False, rope=True, rope_base=10000.0, with_kv=True, host=True):
    """Seeded synthetic weights and factors (oracle.synth_layer conventions).

    Returns (weights, decomposed, config) built from this package's types
    with fp64 numpy payloads (``host=True``).
    """
    torch = _torch()
    sq = 1.0 / math.sqrt(d)
    gk, gv = n_heads // s_k, n_heads // s_v
    rk = [ranks_k] * gk if isinstance(ranks_k, int) else list(ranks_k)
    rv = [ranks_v] * gv if isinstance(ranks_v, int) else list(ranks_v)

    def gran(s):
        if s == 1:
            return Granularity.multi_head()
        if s == n_heads:
            return Granularity.joint_head(n_heads)
        return Granularity.group_head(s)

    def rm(r, c, sd):
        return random_matrix_gpu(r, c, sd).cpu().numpy()

    wl, dl = [], []
    for li in range(layers):
        sd = seed + 101 * li if li else seed
        z = np.zeros((d, d))
        lw = LayerWeights(wq=rm(d, d, sd) * sq,
                          wk=rm(d, d, sd + 1) * sq if with_kv else z,
                          wv=rm(d, d, sd + 2) * sq if with_kv else z,
                          wo=rm(d, d, sd + 3) * sq)
        kg = [GroupFactors(a=rm(d, r, sd + 1000 + 2 * g) * sq,
                           b=rm(r, s_k * head_dim, sd + 1001 + 2 * g) / math.sqrt(r), rank=r)
              for g, r in enumerate(rk)]
        vg = [GroupFactors(a=rm(d, r, sd + 2000 + 2 * g) * sq,
                           b=rm(r, s_v * head_dim, sd + 2001 + 2 * g) / math.sqrt(r), rank=r)
              for g, r in enumerate(rv)]
        key = DecomposedLayer(gran(s_k), tuple(kg), d, head_dim, n_heads)
        value = DecomposedLayer(gran(s_v), tuple(vg), d, head_dim, n_heads)
        if hadamard_fused:
            key, value = fuse_hadamard(key).layer, fuse_hadamard(value).layer
        wl.append(lw)
        dl.append(LayerKV(key=key, value=value))
    config = AttentionConfig(d, n_heads, head_dim, layers=layers, rope=rope, rope_base=rope_base)
    return ModelWeights(layers=tuple(wl)), dl, config


# ---------------------------------------------------------------------------
# Bench-scale synthetic engine: weights generated directly on the GPU in the
# kernels' layouts (no fp64 host copies of a 32-layer model), latent caches
# filled with rows of the same statistics as x @ A for x ~ U[-1, 1).
# ---------------------------------------------------------------------------
def _shape_only(rows: int, cols: int):
    """Zero-stride placeholder with the right shape (validation only)."""
    return np.broadcast_to(np.float64(0.0), (rows, cols))


def synthetic_engine(d=4096, n_heads=32, head_dim=128, s=4, rank_k=256, rank_v=256, layers=32,
                     batch=1, context=65536, extra=64, bits=16, dtype="bfloat16", seed=0,
                     rope_base=10000.0, rope=True, kv_heads=0):
    """Return (weights, fused, cache) for a Llama-2-7B-shaped Palu model.

    Random-init weights of that architecture (uniform, scaled as SURVEY
    8(d)); the cache holds ``context`` tokens per sequence.  kv_heads > 0:
    GQA (Mistral-7B: 8 KV heads) as the MHA-equivalent layer -- one group per
    KV head (s = n_heads / kv_heads), its B_k / B_v columns replicated across
    the group's query heads.
    """
    if kv_heads:
        s = n_heads // kv_heads
    import torch as _t
    from .attention import FusedWeights, LayerFused, _dt, _head_offsets, _rank_pad, _round_up, theta_table

    torch = _torch()
    code, tdt = _dt(dtype)
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    G = n_heads // s

    def per_layer(r):
        # int (uniform) | per-layer tuples of per-group ranks (rank_plan.kv_plan)
        return [tuple([r] * G)] * layers if isinstance(r, int) else [tuple(int(x) for x in t) for t in r]

    ranks_k_l, ranks_v_l = per_layer(rank_k), per_layer(rank_v)

    def U(*shape, scale):
        return ((torch.rand(*shape, generator=g, device=dev, dtype=torch.float32) * 2 - 1) * scale)

    i32 = lambda v: torch.tensor(list(v), dtype=torch.int32, device=dev)
    fl, wl, dl = [], [], []
    gran = Granularity.group_head(s) if 1 < s < n_heads else (
        Granularity.multi_head() if s == 1 else Granularity.joint_head(n_heads))
    for li in range(layers):
        rk, rv = ranks_k_l[li], ranks_v_l[li]
        rk_pad, rv_pad = _round_up(max(rk), 128), _round_up(max(rv), 128)
        ko = s * sum(rv)
        ko_pad = _round_up(ko, 8)
        lat_k = [sum(rk[:i]) for i in range(G)]
        lat_v = [sum(rv[:i]) for i in range(G)]
        qdim = d if rope else s * sum(rk)  # rope off: w1 starts with wq_fused^T
        n1 = qdim + sum(rk) + sum(rv)
        w1 = U(n1, d, scale=1.0 / math.sqrt(d)).to(tdt)
        bk = torch.zeros(G, rk_pad, s * head_dim, device=dev, dtype=tdt)
        for gg, r in enumerate(rk):
            if kv_heads:  # one KV head's B columns replicated over its query heads
                bk[gg, :r] = U(r, head_dim, scale=1.0 / math.sqrt(r)).repeat(1, s).to(tdt)
            else:
                bk[gg, :r] = U(r, s * head_dim, scale=1.0 / math.sqrt(r)).to(tdt)
        # wo_fused rows: (B_v block @ W_o block); entries ~ scale of a product
        woT = torch.zeros(d, ko_pad, device=dev, dtype=tdt)
        woT[:, :ko] = U(d, ko, scale=1.0 / math.sqrt(3.0 * d)).to(tdt)
        fl.append(LayerFused(wq_fused=None, wo_fused=None,
                             q_offsets=_head_offsets(rk, s, n_heads),
                             o_offsets=_head_offsets(rv, s, n_heads), key_ranks=rk, value_ranks=rv,
                             s_k=s, s_v=s, rk_pad=rk_pad, rv_pad=rv_pad, ko_pad=ko_pad, w1=w1, bk=bk,
                             woT=woT, ranks_k_dev=i32(rk), latoff_k_dev=i32(lat_k),
                             ranks_v_dev=i32(rv), latoff_v_dev=i32(lat_v),
                             o_off_dev=i32(_head_offsets(rv, s, n_heads)), qdim=qdim,
                             q_off_dev=i32(_head_offsets(rk, s, n_heads))))
        sh = _shape_only(d, d)
        wl.append(LayerWeights(sh, sh, sh, sh))
        kg = tuple(GroupFactors(_shape_only(d, r), _shape_only(r, s * head_dim), r) for r in rk)
        vg = tuple(GroupFactors(_shape_only(d, r), _shape_only(r, s * head_dim), r) for r in rv)
        dl.append(LayerKV(DecomposedLayer(gran, kg, d, head_dim, n_heads),
                          DecomposedLayer(gran, vg, d, head_dim, n_heads)))
    config = AttentionConfig(d, n_heads, head_dim, layers=layers, rope=rope, rope_base=rope_base)
    theta = theta_table(head_dim, rope_base)
    fused = FusedWeights(layers=tuple(fl), config=config, dtype=dtype,
                         theta_dev=torch.from_numpy(theta).to(dev), theta=theta)
    cache = LatentKVCache(dl, config, bits, dtype=dtype, batch=batch, capacity=context + extra)
    # fill: latent entries ~ x @ A with x ~ U[-1,1), A ~ U/sqrt(d): std 1/3
    for li in range(layers):
        for side in cache._stores[li]:
            for gg in range(side.G):
                r = side.ranks[gg]
                for b in range(batch):
                    for c0 in range(0, context, 16384):
                        T = min(16384, context - c0)
                        h = torch.randn(T, r, generator=g, device=dev, dtype=torch.float32) / 3.0
                        if side.bits == FP_BITS:
                            side.rows[b, gg, c0:c0 + T, :r].copy_(h.to(side.rows.dtype))
                        else:
                            _fill_side(side, gg, b, c0, h.double())
    set_cache_t(cache, context)
    return ModelWeights(layers=tuple(wl)), fused, cache
