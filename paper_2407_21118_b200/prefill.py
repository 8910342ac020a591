"""Batched prompt prefill on the GPU.

The reference builds a cache by T sequential decode steps (palu_prefill,
attention.py:469-494): O(T^2) work spread over T dependent steps.  Its result
is fully determined layer by layer: layer l's latents are x_l(t) A_g for every
prompt token, stored (and, for bits < 16, quantised per token) in order, and
layer l + 1's input at token t is layer l's decode output at t -- causal
attention of the rotated query at t over the stored keys 0..t.  So a prompt
prefill is one causal attention pass per layer over all T tokens:

  1. Y = X W1^T (the layer's stacked [W_q | A_k | A_v] rows: one GEMM);
  2. the latent rows go into the cache through the same device quantiser and
     packer the decode step's append uses (bit-exact codes for fp64 inputs);
  3. per group, the STORED rows (dequantised as quant.py:106-107) are
     reconstructed K = H B_g, rotated at positions 0..T-1 (fp64 angles),
     scored against the rotated queries with a causal mask, softmaxed, and
     the value path applies p H_v and wo_fused (Eq. 5);
  4. the layer output is the next layer's X.

The GEMMs and the softmax run through torch (cuBLAS / library kernels, fp32
accumulation); this is the one-time prompt pass, not the decode hot path.
Parity: the caches equal token-by-token prefill's (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import math

import numpy as np

from .attention import FP_BITS, LatentKVCache, _torch, build_fused
from .errors import ValidationError


def _unpack_rows(packed, cols: int, bits: int):
    """LE bitstream rows (quant.py:156-169 order) -> uint8 codes [T, cols], on the GPU."""
    torch = _torch()
    T, nb = packed.shape
    shifts = torch.arange(8, device=packed.device, dtype=torch.uint8)
    bitplane = ((packed.unsqueeze(-1) >> shifts) & 1).reshape(T, nb * 8)[:, : cols * bits]
    w = (1 << torch.arange(bits, device=packed.device)).to(torch.int32)
    return (bitplane.reshape(T, cols, bits).to(torch.int32) * w).sum(-1)


def _stored_rows(side, g: int, b: int, t1: int):
    """Rows 0..t1-1 of group g as the cache holds them, dequantised, fp32 [t1, r]."""
    torch = _torch()
    r = side.ranks[g]
    if side.bits == FP_BITS:
        return side.rows[b, g, :t1, :r].float()
    codes = _unpack_rows(side.rows[b, g, :t1], side.r_pad, side.bits)[:, :r].float()
    return (codes - side.zps64[b, g, :t1, None].float()) * side.scales64[b, g, :t1, None].float()


def _rope(x, positions, theta):
    """attention.py:105-112 on [n, T, d_h] rows at fp64-reduced angles."""
    torch = _torch()
    ang = positions.double()[:, None] * theta[None, :].double()
    c, s = torch.cos(ang).float(), torch.sin(ang).float()
    half = x.shape[-1] // 2
    lo, hi = x[..., :half], x[..., half:]
    return torch.cat([lo * c - hi * s, lo * s + hi * c], dim=-1)


def prefill_batched(weights, fused, cache: LatentKVCache, prompt) -> None:
    """Append a prompt of T tokens to ``cache`` (batch row 0 .. B-1 share it)
    with one causal attention pass per layer; advances cache.t by T."""
    torch = _torch()
    from .harness import _fill_side

    cfg = cache.config
    if not cfg.rope:
        raise ValidationError("batched prefill implements the rope-on path")
    X = torch.as_tensor(np.asarray(prompt, dtype=np.float64), device=cache.device).float()
    if X.ndim != 2 or X.shape[1] != cfg.d_model:
        raise ValidationError(f"prompt must be (T, {cfg.d_model})")
    T = X.shape[0]
    t0 = cache.t
    cache.reserve(t0 + T)
    n, dh, d = cfg.n_heads, cfg.head_dim, cfg.d_model
    theta = fused.theta_dev
    pos = torch.arange(t0, t0 + T, device=cache.device)
    kpos = torch.arange(0, t0 + T, device=cache.device)
    causal = kpos[None, :] <= pos[:, None]  # [T, t0 + T]
    scale = 1.0 / math.sqrt(dh)
    for li, L in enumerate(fused.layers):
        K, V = cache._stores[li]
        Y = X @ L.w1.float().T  # [T, d + sum r_k + sum r_v]
        q = _rope(Y[:, :d].reshape(T, n, dh).transpose(0, 1), pos, theta)  # [n, T, dh]
        sk = sum(L.key_ranks)
        lat_k, lat_v = Y[:, d:d + sk], Y[:, d + sk:]
        for side, lat, ranks in ((K, lat_k, L.key_ranks), (V, lat_v, L.value_ranks)):
            o = 0
            for g, r in enumerate(ranks):
                h = lat[:, o:o + r].double()
                for b in range(cache.batch):
                    _fill_side(side, g, b, t0, h)
                o += r
        out = torch.zeros(T, d, device=cache.device)
        for g in range(K.G):
            hk = _stored_rows(K, g, 0, t0 + T)
            keys = (hk @ L.bk[g, :K.ranks[g]].float()).reshape(t0 + T, L.s_k, dh).transpose(0, 1)
            keys = _rope(keys, kpos, theta)
            for p_ in range(L.s_k):
                i = g * L.s_k + p_
                logits = (q[i] @ keys[p_].T) * scale
                probs = torch.softmax(logits.masked_fill(~causal, float("-inf")), dim=-1)
                gv = i // L.s_v
                hv = _stored_rows(V, gv, 0, t0 + T)
                ctx = probs @ hv  # [T, r_v]
                o0, o1 = L.o_offsets[i], L.o_offsets[i + 1]
                out += ctx @ L.woT[:, o0:o1].float().T
        X = out
    cache.t = t0 + T
    if cache._session is not None:
        cache._session.t_dev.fill_(cache.t)


def palu_prefill_batched(weights, decomposed, config, prompt, bits=FP_BITS, fused=None,
                         tile_len=None, *, dtype: str = "float32") -> LatentKVCache:
    """palu_prefill (attention.py:469-494) as one batched pass per layer."""
    if tile_len is not None and tile_len < 1:
        raise ValidationError(f"tile_len must be >= 1, got {tile_len}")
    tokens = np.asarray(prompt, dtype=np.float64)
    if tokens.ndim != 2 or tokens.shape[1] != config.d_model:
        raise ValidationError(f"prompt must be (T, {config.d_model})")
    if fused is None:
        fused = build_fused(weights, decomposed, config, dtype=dtype)
    cache = LatentKVCache(decomposed, config, bits, dtype=fused.dtype, capacity=max(tokens.shape[0], 8))
    prefill_batched(weights, fused, cache, tokens)
    return cache
