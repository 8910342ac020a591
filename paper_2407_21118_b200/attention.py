"""Drop-in GPU mirror of palu.attention's decode API (attention.py:34-515).

Same names, argument meaning and error behaviour as the reference:
``build_fused``, ``LatentKVCache``, ``palu_decode_step_rope``,
``palu_decode_step_quantized``, ``palu_prefill``, ``palu_decode``,
``reference_decode`` and ``rope_apply``.  The numpy stages of the reference
step are replaced by the CUDA kernels of libpalu_b200.so (C ABI,
include/palu_b200.h); torch only allocates device memory, provides streams
and captures CUDA graphs.  There is no CPU fallback: without a CUDA device
or the library every step raises.

Extras over the reference signatures (keyword-only, defaults keep the
reference behaviour):
  * ``dtype``: "float32" (fp32 storage and math; the C1 parity config) or
    "bfloat16" (bf16 weights/latents, fp32 accumulation; the perf path);
  * ``batch``: x_t may be (d,) or (B, d) -- B independent sequences;
  * ``capacity``: initial cache rows per sequence (grows by doubling);
  * ``score_kernel``: "auto" | "simt" | "tcgen05".
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ValidationError
from .model import (AttentionConfig, LayerKV, LayerWeights, ModelWeights, as_array,
                    validate_weights)

FP_BITS = 16
_APPEND_SPLIT = os.environ.get("PALU_APPEND_SPLIT") == "1"  # A/B diagnostics only
# PALU_APPEND_ABSORB=0: separate append and absorb launches (A/B diagnostics only)
_APPEND_ABSORB = os.environ.get("PALU_APPEND_ABSORB", "1") != "0"
# PALU_L2PF=1: L2 prefetch of the output projection during the score (measured slower; A/B)
_L2PF = os.environ.get("PALU_L2PF") == "1"
# replicated-B key groups (GQA as its MHA-equivalent layer): reconstruct K once
# per KV head (palu_rope_score_tc_rep); PALU_GQA_REP=0 keeps the per-head path
_GQA_REP = os.environ.get("PALU_GQA_REP", "1") != "0"
SUPPORTED_BITS = (2, 3, 4, 8)
DTYPES = ("float32", "bfloat16")


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_21118_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _ptr(t) -> int:
    return t.data_ptr() if t is not None else None


def _stream() -> int:
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream


def _dt(dtype: str):
    torch = _torch()
    if dtype not in DTYPES:
        raise ValidationError(f"dtype must be one of {DTYPES}, got {dtype!r}")
    return (_lib.DTYPE_F32, torch.float32) if dtype == "float32" else (_lib.DTYPE_BF16, torch.bfloat16)


def theta_table(head_dim: int, base: float) -> np.ndarray:
    """Rotary frequencies exactly as attention.py:108-109 evaluates them."""
    idx = np.arange(head_dim // 2, dtype=np.float64)
    return base ** (-2.0 * idx / head_dim)


def rope_apply(v, position: int, base: float = 10000.0) -> np.ndarray:
    """attention.py:93-102 (host helper; not on the decode hot path)."""
    vec = np.asarray(v, dtype=np.float64)
    if vec.ndim != 1:
        raise ValidationError("rope_apply expects a 1-D vector")
    if vec.shape[0] % 2 != 0:
        raise ValidationError(f"rope_apply requires even length, got {vec.shape[0]}")
    if position < 0:
        raise ValidationError("position must be non-negative")
    half = vec.shape[0] // 2
    ang = position * theta_table(vec.shape[0], base)
    c, s = np.cos(ang), np.sin(ang)
    lo, hi = vec[:half], vec[half:]
    return np.concatenate([lo * c - hi * s, lo * s + hi * c])


def _head_offsets(ranks, s: int, n_heads: int) -> tuple:
    """attention.py:171-176."""
    offs = [0]
    for i in range(n_heads):
        offs.append(offs[-1] + ranks[i // s])
    return tuple(offs)


# ---------------------------------------------------------------------------
# Fused, device-resident weights (attention.py:179-232)
# ---------------------------------------------------------------------------
@dataclass
class LayerFused:
    """attention.py:179-186 plus the device tensors the kernels consume.

    w1   [qdim + sum r_k + sum r_v, d]  rows: W_q columns (rope on, qdim = d) or
                                       wq_fused columns (rope off, qdim = sum_i r_k(i)),
                                       then A_k^T, A_v^T
    bk   [G_k, Rk_pad, s_k * d_h]    key up-projections, zero rows past rank
    woT  [d, Ko_pad]                 wo_fused^T (B_v folded into W_o, Eq. 5)
    """

    wq_fused: object
    wo_fused: object  # host fp64 wo_fused (attention.py:221) for inspection
    q_offsets: tuple
    o_offsets: tuple
    key_ranks: tuple
    value_ranks: tuple
    s_k: int = 0
    s_v: int = 0
    rk_pad: int = 0
    rv_pad: int = 0
    ko_pad: int = 0
    w1: object = None
    bk: object = None
    woT: object = None
    ranks_k_dev: object = None
    latoff_k_dev: object = None
    ranks_v_dev: object = None
    latoff_v_dev: object = None
    o_off_dev: object = None
    qdim: int = 0           # rows of w1 before the latents (d, or sum_i r_k(i) rope off)
    q_off_dev: object = None  # rope off: per-head offsets of q_lat inside y


@dataclass
class FusedWeights:
    layers: tuple
    config: AttentionConfig = None
    dtype: str = "float32"
    theta_dev: object = None
    theta: np.ndarray = None

    @property
    def dtype_code(self):
        return _lib.DTYPE_F32 if self.dtype == "float32" else _lib.DTYPE_BF16


def _rank_pad(r: int, dtype: str, bits: int = 16) -> int:
    """Row width of a latent store: bf16 rows are 128-byte swizzle blocks for
    the tcgen05 path; packed rows must be whole 16-byte TMA granules."""
    m = 64 if dtype == "bfloat16" else 32
    if bits != 16:
        m = max(m, {2: 64, 3: 128, 4: 32, 8: 32}[bits])
    return _round_up(max(r, 1), m)


def build_fused(weights, decomposed, config, *, dtype: str = "float32", device=None,
                prep: str = "host") -> FusedWeights:
    """attention.py:194-232, then upload in the kernels' layouts.

    Per head i of value group g: wo block = B_v[g][:, i-in-g] @ W_o[rows i];
    the key-side fusion into W_q only exists without rotary embedding.
    Offline prep runs once in fp64: on the host (prep="host", as the
    reference) or as batched fp64 GEMMs on the GPU (prep="gpu", offline.py).
    """
    if prep not in ("host", "gpu"):
        raise ValidationError(f"prep must be 'host' or 'gpu', got {prep!r}")
    torch = _torch()
    code, tdt = _dt(dtype)
    validate_weights(weights, config)
    if len(decomposed) != config.layers:
        raise ValidationError(f"{len(decomposed)} decomposed layers for {config.layers}-layer config")
    d, n, dh = config.d_model, config.n_heads, config.head_dim
    dev = device or torch.device("cuda", torch.cuda.current_device())
    _lib.load()
    layers = []
    for li, (lw, kv) in enumerate(zip(weights.layers, decomposed)):
        for dec, tag in ((kv.key, "key"), (kv.value, "value")):
            if dec.d_model != d or dec.n_heads != n or dec.head_dim != dh:
                raise ValidationError(f"layer {li} {tag} decomposition does not match the config")
        s_k = kv.key.granularity.group_size
        s_v = kv.value.granularity.group_size
        wq, wo = as_array(lw.wq), as_array(lw.wo)
        ak = [as_array(g.a) for g in kv.key.groups]
        bk = [as_array(g.b) for g in kv.key.groups]
        av = [as_array(g.a) for g in kv.value.groups]
        bv = [as_array(g.b) for g in kv.value.groups]
        o_blocks, q_blocks = [], []
        if prep == "gpu":
            from .offline import fused_blocks_gpu
            wo_fused, wq_gpu = fused_blocks_gpu(wq, wo, bk, bv, n, dh, s_k, s_v, config.rope, device=dev)
            if not config.rope:
                q_blocks = [wq_gpu]
        else:
            for i in range(n):
                gk, pk = divmod(i, s_k)
                gv, pv = divmod(i, s_v)
                if not config.rope:
                    q_blocks.append(wq[:, i * dh:(i + 1) * dh] @ bk[gk][:, pk * dh:(pk + 1) * dh].T)
                o_blocks.append(bv[gv][:, pv * dh:(pv + 1) * dh] @ wo[i * dh:(i + 1) * dh, :])
            wo_fused = np.concatenate(o_blocks, axis=0)
        key_ranks = tuple(g.rank for g in kv.key.groups)
        value_ranks = tuple(g.rank for g in kv.value.groups)
        rk_pad = _round_up(max(key_ranks), 128)  # covers every store width below
        rv_pad = _round_up(max(value_ranks), 128)
        ko = wo_fused.shape[0]
        ko_pad = _round_up(ko, 8)
        # rope off: the key reconstruction is absorbed into W_q (attention.py:219-220),
        # so the first rows of w1 produce q_lat directly
        wq_f = None if config.rope else np.concatenate(q_blocks, axis=1)
        first = wq.T if config.rope else wq_f.T
        w1 = np.concatenate([first] + [a.T for a in ak] + [a.T for a in av], axis=0)
        bk_pad = np.zeros((len(bk), rk_pad, s_k * dh))
        for g, b in enumerate(bk):
            bk_pad[g, :b.shape[0]] = b
        woT = np.zeros((d, ko_pad))
        woT[:, :ko] = wo_fused.T
        i32 = lambda v: torch.tensor(list(v), dtype=torch.int32, device=dev)
        lat_k = np.concatenate([[0], np.cumsum(key_ranks)[:-1]]).astype(int)
        lat_v = np.concatenate([[0], np.cumsum(value_ranks)[:-1]]).astype(int)
        layers.append(LayerFused(
            wq_fused=wq_f,
            wo_fused=wo_fused,
            q_offsets=_head_offsets(key_ranks, s_k, n),
            o_offsets=_head_offsets(value_ranks, s_v, n),
            key_ranks=key_ranks, value_ranks=value_ranks, s_k=s_k, s_v=s_v,
            rk_pad=rk_pad, rv_pad=rv_pad, ko_pad=ko_pad,
            w1=torch.from_numpy(w1).to(dev, tdt).contiguous(),
            bk=torch.from_numpy(bk_pad).to(dev, tdt).contiguous(),
            woT=torch.from_numpy(woT).to(dev, tdt).contiguous(),
            ranks_k_dev=i32(key_ranks), latoff_k_dev=i32(lat_k),
            ranks_v_dev=i32(value_ranks), latoff_v_dev=i32(lat_v),
            o_off_dev=i32(_head_offsets(value_ranks, s_v, n)),
            qdim=d if config.rope else int(_head_offsets(key_ranks, s_k, n)[-1]),
            q_off_dev=i32(_head_offsets(key_ranks, s_k, n)),
        ))
    theta = theta_table(dh, config.rope_base) if config.rope else np.zeros(max(dh // 2, 1))
    return FusedWeights(layers=tuple(layers), config=config, dtype=dtype,
                        theta_dev=torch.from_numpy(theta).to(dev), theta=theta)


# ---------------------------------------------------------------------------
# GPU latent cache (attention.py:235-331)
# ---------------------------------------------------------------------------
def _norm_bits(bits) -> tuple:
    """attention.py:292-300."""
    pair = (bits, bits) if isinstance(bits, (int, np.integer)) else tuple(bits)
    if len(pair) != 2:
        raise ValidationError(f"bits must be an int or a (key, value) pair, got {bits!r}")
    for b in pair:
        if b != FP_BITS and b not in SUPPORTED_BITS:
            raise ValidationError(f"bits must be one of {SUPPORTED_BITS}, got {b}")
    return int(pair[0]), int(pair[1])


@dataclass(frozen=True)
class QuantizedLatent:
    """quant.py:51-79 (export view of one group store)."""

    codes: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray
    bits: int

    @property
    def n_tokens(self) -> int:
        return self.codes.shape[0]

    @property
    def width(self) -> int:
        return self.codes.shape[1]


def _unpack_rows(packed: np.ndarray, cols: int, bits: int) -> np.ndarray:
    """Inverse of the per-row LE packing (quant.py:172-181 order)."""
    rows = packed.shape[0]
    bitsarr = np.unpackbits(packed, axis=1, bitorder="little")[:, : cols * bits]
    w = (1 << np.arange(bits)).astype(np.uint16)
    return (bitsarr.reshape(rows, cols, bits) * w).sum(axis=2).astype(np.uint8)


class _SideStore:
    """Device storage of one side (K or V) of one layer for all groups."""

    def __init__(self, ranks, bits, r_pad, batch, cap, dtype, dev):
        torch = _torch()
        self.ranks, self.bits, self.r_pad = tuple(ranks), bits, r_pad
        self.G = len(ranks)
        self.batch, self.cap, self.dtype = batch, cap, dtype
        _, tdt = _dt(dtype)
        shp = (batch, self.G, cap)
        if bits == FP_BITS:
            self.rows = torch.zeros(shp + (r_pad,), dtype=tdt, device=dev)
            self.scales = self.zps = self.scales64 = self.zps64 = None
        else:
            self.rows = torch.zeros(shp + (r_pad * bits // 8,), dtype=torch.uint8, device=dev)
            self.scales = torch.ones(shp, dtype=torch.float32, device=dev)
            self.zps = torch.zeros(shp, dtype=torch.float32, device=dev)
            self.scales64 = torch.ones(shp, dtype=torch.float64, device=dev)
            self.zps64 = torch.zeros(shp, dtype=torch.int64, device=dev)

    def grow(self, new_cap: int, t: int):
        torch = _torch()
        old = {k: getattr(self, k) for k in ("rows", "scales", "zps", "scales64", "zps64")}
        self.__init__(self.ranks, self.bits, self.r_pad, self.batch, new_cap, self.dtype,
                      old["rows"].device)
        for k, v in old.items():
            if v is not None:
                getattr(self, k)[:, :, :t].copy_(v[:, :, :t])
        del old
        torch.cuda.synchronize()

    def matrix(self, b: int, g: int, t: int) -> np.ndarray:
        """Dequantised fp64 rows of one group (attention.py:257-268)."""
        r = self.ranks[g]
        if self.bits == FP_BITS:
            return self.rows[b, g, :t, :r].double().cpu().numpy()
        q = self.quantized(b, g, t)
        return (q.codes.astype(np.float64) - q.zero_points[:, None].astype(np.float64)) * q.scales[:, None]

    def quantized(self, b: int, g: int, t: int) -> QuantizedLatent:
        if self.bits == FP_BITS:
            raise ValidationError("cache stores raw latents; no quantized form")
        r = self.ranks[g]
        packed = self.rows[b, g, :t].cpu().numpy()
        codes = _unpack_rows(packed, self.r_pad, self.bits)[:, :r] if t else np.zeros((0, r), np.uint8)
        return QuantizedLatent(codes=codes, scales=self.scales64[b, g, :t].cpu().numpy(),
                               zero_points=self.zps64[b, g, :t].cpu().numpy(), bits=self.bits)


class _GroupView:
    """Reference-compatible view of one group store (attention.py:235-281)."""

    def __init__(self, side: _SideStore, g: int, cache, b: int = 0):
        self._side, self._g, self._cache, self._b = side, g, cache, b
        self.rank = side.ranks[g]
        self.bits = side.bits

    def matrix(self) -> np.ndarray:
        return self._side.matrix(self._b, self._g, self._cache.t)

    def quantized_latent(self) -> QuantizedLatent:
        return self._side.quantized(self._b, self._g, self._cache.t)


class _LayerView:
    def __init__(self, cache, li):
        L = cache._stores[li]
        self.k_groups = [_GroupView(L[0], g, cache) for g in range(L[0].G)]
        self.v_groups = [_GroupView(L[1], g, cache) for g in range(L[1].G)]


class LatentKVCache:
    """attention.py:303-331 on the GPU.

    One latent store per head group per side per layer, in HBM with the
    layout of include/palu_b200.h.  ``bits`` 16 keeps raw rows in the
    storage dtype; 2/3/4/8 keeps per-token quantised, packed codes.  ``t``
    only grows.  A cache is owned by a single decode session.
    """

    def __init__(self, decomposed, config, bits=FP_BITS, *, dtype: str = "float32",
                 batch: int = 1, capacity: int | None = None, device=None,
                 score_kernel: str = "auto"):
        torch = _torch()
        k_bits, v_bits = _norm_bits(bits)
        if len(decomposed) != config.layers:
            raise ValidationError(f"{len(decomposed)} decomposed layers for {config.layers}-layer config")
        if batch < 1:
            raise ValidationError(f"batch must be >= 1, got {batch}")
        _dt(dtype)
        self.config = config
        self.decomposed = list(decomposed)
        self.bits = bits
        self.k_bits, self.v_bits = k_bits, v_bits
        self.dtype = dtype
        self.batch = batch
        self.t = 0
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        # whole 128-token tiles: every per-tile copy of the kernels (TMA boxes,
        # zero-point blocks) stays inside its own sequence/group rows
        cap = _round_up(max(int(capacity or 256), 8), 128)
        self.capacity = cap
        self._stores = []
        for kv in self.decomposed:
            rk, rv = kv.key.ranks, kv.value.ranks
            self._stores.append((
                _SideStore(rk, k_bits, _rank_pad(max(rk), dtype, k_bits), batch, cap, dtype,
                           self.device),
                _SideStore(rv, v_bits, _rank_pad(max(rv), dtype, v_bits), batch, cap, dtype,
                           self.device)))
        if score_kernel not in ("auto", "simt", "tcgen05", "fused"):
            raise ValidationError(f"score_kernel must be auto|simt|tcgen05|fused, got {score_kernel!r}")
        self.score_kernel = score_kernel
        self._session = None
        self._validated = None   # (weights, fused) of the last validated step
        self._allreduce = None   # head-group shard: per-layer partial-output reduction

    # reference-compatible accessors -------------------------------------
    @property
    def layers(self):
        return [_LayerView(self, li) for li in range(len(self._stores))]

    def hk(self, layer: int, b: int = 0) -> np.ndarray:
        K = self._stores[layer][0]
        return np.concatenate([K.matrix(b, g, self.t) for g in range(K.G)], axis=1)

    def hv(self, layer: int, b: int = 0) -> np.ndarray:
        V = self._stores[layer][1]
        return np.concatenate([V.matrix(b, g, self.t) for g in range(V.G)], axis=1)

    # capacity ------------------------------------------------------------
    def reserve(self, rows: int) -> None:
        if rows <= self.capacity:
            return
        new = self.capacity
        while new < rows:
            new *= 2
        for K, V in self._stores:
            K.grow(new, self.t)
            V.grow(new, self.t)
        self.capacity = new
        self._session = None


def _check_cache_fused(cache: LatentKVCache, fused: FusedWeights) -> None:
    """attention.py:334-340."""
    if fused.config is not None and fused.config.rope != cache.config.rope:
        raise ValidationError("fused weights were built for rope="
                              f"{fused.config.rope}, the cache config has rope={cache.config.rope}")
    if len(fused.layers) != len(cache._stores):
        raise ValidationError("cache and fused weights disagree on layer count")
    for li, lf in enumerate(fused.layers):
        kv = cache.decomposed[li]
        if lf.key_ranks != kv.key.ranks or lf.value_ranks != kv.value.ranks:
            raise ValidationError(f"cache/fused rank mismatch at layer {li}")
    if fused.dtype != cache.dtype:
        raise ValidationError(f"cache dtype {cache.dtype} != fused weights dtype {fused.dtype}")


def _value_tc_choice(bits: int, r_pad: int) -> bool:
    """Packed 2/4/8-bit values run on the int8 tensor pipe (palu_vq.cuh); 3-bit
    values keep the CUDA-core kernel unless PALU_VALUE_KERNEL=tc_quant (the
    converter-to-bf16 tcgen05 kernel, also forced for 2/4/8 bits with
    tc_quant_bf16).  PALU_VALUE_KERNEL=simt forces the CUDA-core kernel."""
    env = os.environ.get("PALU_VALUE_KERNEL", "")
    if bits == FP_BITS:
        return env != "simt"
    if bits not in (2, 3, 4, 8) or r_pad % 128 != 0 or env == "simt":
        return False
    return env in ("tc_quant", "tc_quant_bf16") or bits in (2, 4, 8)


def _validate_step(weights, fused, cache) -> None:
    """Validation before any mutation.  The (weights, fused) pair a cache was
    last validated with is remembered ON the cache (shapes and ranks of these
    objects cannot change), so repeated steps skip the per-layer checks (~50 us
    of Python per 32-layer step) and nothing outlives the cache."""
    v = cache._validated
    if v is not None and v[0] is weights and v[1] is fused:
        return
    _check_cache_fused(cache, fused)
    validate_weights(weights, cache.config)
    cache._validated = (weights, fused)


# ---------------------------------------------------------------------------
# The decode step engine
# ---------------------------------------------------------------------------
class _Session:
    """Device buffers + the per-step launch sequence for one (fused, cache) pair."""

    def __init__(self, fused: FusedWeights, cache: LatentKVCache, score_kernel: str = "auto",
                 use_graph: bool = True):
        torch = _torch()
        cfg = cache.config
        self.fused, self.cache, self.cfg = fused, cache, cfg
        self.B, self.d, self.n, self.dh = cache.batch, cfg.d_model, cfg.n_heads, cfg.head_dim
        dev = cache.device
        self.cap = cache.capacity
        self.rope = cfg.rope
        self.n1 = max(int(L.w1.shape[0]) for L in fused.layers)
        self.ko = max(L.ko_pad for L in fused.layers)
        rk = max(L.rk_pad for L in fused.layers)
        rv = max(L.rv_pad for L in fused.layers)
        self.x = torch.zeros(self.B, self.d, dtype=torch.float32, device=dev)
        self.y = torch.zeros(self.B, self.n1, dtype=torch.float32, device=dev)
        self.uw = torch.zeros(self.B * self.n * rk * self.dh, dtype=torch.float32, device=dev)
        self.ld_logits = _round_up(self.cap, 4)
        self.max_planes = 2  # rank splits of the tcgen05 score kernel
        self.plane = self.B * self.n * self.ld_logits
        self.logits = torch.zeros(self.max_planes, self.B, self.n, self.ld_logits,
                                  dtype=torch.float32, device=dev)
        self.ctx = torch.zeros(self.B, self.ko, dtype=torch.float32, device=dev)
        gv = max(len(L.value_ranks) for L in fused.layers)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        # split-T chunks: one wave of 2 CTAs per SM for the value stream (per-CTA
        # statistics and merge costs favour few, long chunks), <= 4096 tokens each
        self.n_chunks = max(-(-2 * sms // (gv * self.B)), -(-self.cap // 4096), 1)
        if os.environ.get("PALU_SV_CHUNKS"):  # tuning experiments only
            self.n_chunks = max(int(os.environ["PALU_SV_CHUNKS"]), -(-self.cap // 8192))
        ws = _lib.call("palu_softmax_value_workspace", self.B, self.n, rv, self.n_chunks)
        self.ws = torch.zeros(ws // 4 + 1, dtype=torch.float32, device=dev)
        self.t_dev = torch.tensor([cache.t], dtype=torch.int32, device=dev)
        self.x_host = torch.zeros(self.B, self.d, dtype=torch.float32).pin_memory()
        self.out_host = torch.zeros(self.B, self.d, dtype=torch.float32).pin_memory()
        # tcgen05 score path: bf16 raw keys, d_h 128, head pairs, R_pad in 64..256
        self.tc_layers = []
        c = cache
        for li, L in enumerate(fused.layers):
            K = cache._stores[li][0]
            ok = (cfg.rope and fused.dtype == "bfloat16" and K.bits in (FP_BITS, 2, 3, 4, 8)
                  and self.dh == 128 and L.s_k % 2 == 0 and K.r_pad % 64 == 0 and K.r_pad <= 256)
            if score_kernel in ("tcgen05", "fused") and not ok and cfg.rope:
                raise ValidationError(f"layer {li}: shape not supported by the tcgen05 score kernel")
            ks = _lib.call("palu_rope_score_tc_splits", L.s_k, K.r_pad) if ok else 0
            ok = ok and 1 <= ks <= 2
            if score_kernel == "tcgen05" and not ok:
                raise ValidationError(f"layer {li}: rank {K.r_pad} not supported by the tcgen05 kernel")
            self.tc_layers.append(ok and score_kernel != "simt")
        self.planes = [(_lib.call("palu_rope_score_tc_splits", L.s_k, c._stores[li][0].r_pad)
                        if self.tc_layers[li] else 1) for li, L in enumerate(fused.layers)]
        # fused score + softmax + value (grid-level role split): bf16 raw K and V,
        # K and V sharing the head grouping
        self.fused_layers = []
        for li, L in enumerate(fused.layers):
            K, V = c._stores[li]
            ok = (self.tc_layers[li] and K.bits == FP_BITS and V.bits == FP_BITS and L.s_v == L.s_k
                  and len(L.value_ranks) == len(L.key_ranks) and V.r_pad <= 512 and V.r_pad % 64 == 0
                  and score_kernel == "fused")
            self.fused_layers.append(ok)
        # rope off: tcgen05 latent-score kernel for bf16 raw keys
        self.ls_tc_layers = [
            (not cfg.rope and fused.dtype == "bfloat16"
             and c._stores[li][0].bits in (FP_BITS, 2, 3, 4, 8)
             and L.s_k <= 16 and c._stores[li][0].r_pad % 64 == 0 and c._stores[li][0].r_pad <= 256
             and score_kernel != "simt")
            for li, L in enumerate(fused.layers)]
        if score_kernel == "tcgen05" and not cfg.rope and not all(self.ls_tc_layers):
            raise ValidationError("shape not supported by the tcgen05 latent-score kernel")
        # tcgen05 softmax + value after the tcgen05 score kernel: bf16 raw V,
        # 64-column-aligned rows, up to 4 heads per value group
        self.value_tc_layers = []
        for li, L in enumerate(fused.layers):
            K, V = c._stores[li]
            self.value_tc_layers.append(
                (self.tc_layers[li] or self.ls_tc_layers[li]) and not self.fused_layers[li]
                and V.r_pad % 64 == 0 and V.r_pad <= 512 and L.s_v <= 4
                # quantised values: int8 tensor pipe for 2/4/8 bits (_value_tc_choice)
                and _value_tc_choice(V.bits, V.r_pad))
        self.ws_fused = None
        if any(self.fused_layers) or any(self.value_tc_layers):
            nbytes = max(_lib.call("palu_rope_attend_workspace", self.B, self.n, V.G, V.r_pad, self.cap)
                         for (K, V) in c._stores)
            self.ws_fused = torch.zeros(nbytes // 4 + 1, dtype=torch.float32, device=dev)
        self.score_sms = int(os.environ.get("PALU_SCORE_SMS", "0"))
        # replicated-B groups: every query head of a key group uses the same
        # B_k columns (one KV head); the score reconstructs K = H B once per
        # group and dots the rotated keys with the group's 4 rotated queries
        self.rep_bkt = [None] * len(fused.layers)
        self.qrot = None
        for li, L in enumerate(fused.layers):
            K = c._stores[li][0]
            if not (self.tc_layers[li] and not self.fused_layers[li] and _GQA_REP and K.bits == FP_BITS
                    and L.s_k == 4 and self.dh == 128 and _APPEND_ABSORB and not _APPEND_SPLIT):
                continue
            bkt = replicated_key_operand(L.bk, K.r_pad, L.s_k, self.dh)
            if bkt is None:
                continue
            self.rep_bkt[li] = bkt.unsqueeze(0).expand(self.B, -1, -1, -1).contiguous()
            if self.qrot is None:
                self.qrot = torch.zeros(self.B * self.n * self.dh, dtype=torch.float32, device=dev)
        self.uw_bf = None
        self.rope_tab = None
        if any(self.tc_layers):
            self.uw_bf = torch.zeros(self.B * self.n * 128 * rk, dtype=torch.bfloat16, device=dev)
            nf = _lib.call("palu_rope_table_floats", self.dh // 2, self.cap)
            self.rope_tab = torch.zeros(nf, dtype=torch.float32, device=dev)
            _lib.call("palu_rope_table", _ptr(fused.theta_dev), self.dh // 2, self.cap,
                      _ptr(self.rope_tab), _stream())
        self.use_graph = use_graph
        self.graph = None
        self.allreduce = None  # head-group shards: sum of partial layer outputs (sharding.py)
        self.eager_steps = 0
        self.score_kernel = score_kernel
        self.scale = 1.0 / math.sqrt(self.dh)

    # one layer = 8 stream-ordered launches ------------------------------
    def _layer(self, li: int, st: int):
        f, c = self.fused, self.cache
        L = f.layers[li]
        K, V = c._stores[li]
        B, d, n, dh = self.B, self.d, self.n, self.dh
        code = f.dtype_code
        x, y = self.x, self.y
        n1 = int(L.w1.shape[0])
        sk_sum = sum(L.key_ranks)
        qd = L.qdim if L.qdim else d
        self._proj(code, L.w1, n1, d, x, y, st)
        yp = y.data_ptr()
        # attention.py:343-347 + _GroupStore.append (:248-255), both sides in one launch
        # (PALU_APPEND_SPLIT=1: one launch per side, for A/B timing)
        assert K.cap == V.cap
        # rope on: the query absorption's output buffer and layout (UW K order
        # matches the converter's code order for int4 / int2 keys)
        if self.fused_layers[li]:
            uw_ptr, layout = _ptr(self.uw_bf), 1
        elif self.rep_bkt[li] is not None:
            uw_ptr, layout = _ptr(self.qrot), 4  # rotated queries only
        elif self.tc_layers[li]:
            uw_ptr, layout = _ptr(self.uw_bf), {4: 2, 2: 3}.get(K.bits, 1)
        else:
            uw_ptr, layout = _ptr(self.uw), 0
        absorbed = self.rope and _APPEND_ABSORB and not _APPEND_SPLIT
        if absorbed:
            # append and query absorption in one launch (both read only y and t)
            _lib.call("palu_append_absorb", code, K.bits, V.bits, yp + 4 * qd,
                      yp + 4 * (qd + sk_sum), B, self.n1, K.G, V.G, _ptr(L.ranks_k_dev),
                      _ptr(L.latoff_k_dev), _ptr(L.ranks_v_dev), _ptr(L.latoff_v_dev),
                      _ptr(K.rows), _ptr(K.scales), _ptr(K.zps), _ptr(K.scales64), _ptr(K.zps64),
                      _ptr(V.rows), _ptr(V.scales), _ptr(V.zps), _ptr(V.scales64), _ptr(V.zps64),
                      K.r_pad, V.r_pad, K.cap, yp, self.n1, n, dh, L.s_k, _ptr(L.bk), L.bk.shape[1],
                      _ptr(f.theta_dev), self.scale, uw_ptr, layout, _ptr(self.t_dev), st)
        elif _APPEND_SPLIT:
            for S, lat, rk, lo in ((K, yp + 4 * qd, L.ranks_k_dev, L.latoff_k_dev),
                                   (V, yp + 4 * (qd + sk_sum), L.ranks_v_dev, L.latoff_v_dev)):
                _lib.call("palu_latent_append", code, S.bits, lat, B, self.n1, S.G, _ptr(rk),
                          _ptr(lo), _ptr(S.rows), _ptr(S.scales), _ptr(S.zps), _ptr(S.scales64),
                          _ptr(S.zps64), S.r_pad, S.cap, _ptr(self.t_dev), st)
        else:
            _lib.call("palu_latent_append_kv", code, K.bits, V.bits, yp + 4 * qd,
                      yp + 4 * (qd + sk_sum), B, self.n1, K.G, V.G, _ptr(L.ranks_k_dev),
                      _ptr(L.latoff_k_dev), _ptr(L.ranks_v_dev), _ptr(L.latoff_v_dev),
                      _ptr(K.rows), _ptr(K.scales), _ptr(K.zps), _ptr(K.scales64), _ptr(K.zps64),
                      _ptr(V.rows), _ptr(V.scales), _ptr(V.zps), _ptr(V.scales64), _ptr(V.zps64),
                      K.r_pad, V.r_pad, K.cap, _ptr(self.t_dev), st)
        if not self.rope:
            # attention.py:380-388: latent-cache GEMV against q_lat (no reconstruction)
            if self.ls_tc_layers[li]:
                _lib.call("palu_latent_score_tc", K.bits, _ptr(K.rows), _ptr(K.scales),
                          _ptr(K.zps), B, n, L.s_k, K.G, K.r_pad, K.cap, yp, self.n1,
                          _ptr(L.q_off_dev), _ptr(L.ranks_k_dev), self.scale, _ptr(self.t_dev),
                          _ptr(self.logits), self.ld_logits, st)
            else:
                _lib.call("palu_latent_score", code, K.bits, _ptr(K.rows), _ptr(K.scales),
                          _ptr(K.zps), B, n, L.s_k, K.G, K.r_pad, K.cap, yp, self.n1,
                          _ptr(L.q_off_dev), _ptr(L.ranks_k_dev), self.scale, _ptr(self.t_dev),
                          _ptr(self.logits), self.ld_logits, st)
            self._value(li, st)
            return
        if not absorbed:
            _lib.call("palu_query_absorb", code, yp, B, self.n1, n, dh, L.s_k, _ptr(L.bk),
                      L.bk.shape[1], K.r_pad, _ptr(f.theta_dev), self.scale, _ptr(self.t_dev),
                      uw_ptr, layout, st)
        if self.fused_layers[li]:
            _lib.call("palu_rope_attend_tc", _ptr(K.rows), _ptr(V.rows), B, n, L.s_k, K.G, K.r_pad,
                      V.r_pad, K.cap, _ptr(self.uw_bf), _ptr(self.rope_tab), _ptr(self.t_dev),
                      _ptr(self.logits), self.ld_logits, _ptr(L.ranks_v_dev), _ptr(L.o_off_dev),
                      _ptr(self.ctx), self.ko, _ptr(self.ws_fused), self.score_sms, st)
            self._proj(code, L.woT, d, L.ko_pad, self.ctx, x, st)
            return
        if self.rep_bkt[li] is not None:
            _lib.call("palu_rope_score_tc_rep", _ptr(K.rows), B, n, K.G, K.r_pad, K.cap,
                      _ptr(self.rep_bkt[li]), _ptr(self.qrot), _ptr(self.rope_tab), _ptr(self.t_dev),
                      _ptr(self.logits), self.ld_logits, st)
        elif self.tc_layers[li]:
            if _L2PF:  # the output projection's weights ride into L2 during the score
                _lib.call("palu_rope_score_tc_pf", K.bits, _ptr(K.rows), _ptr(K.scales), _ptr(K.zps), B,
                          n, L.s_k, K.G, K.r_pad, K.cap, _ptr(self.uw_bf), _ptr(self.rope_tab),
                          _ptr(self.t_dev), _ptr(self.logits), self.ld_logits, _ptr(L.woT),
                          L.woT.numel() * L.woT.element_size(), st)
            else:
                _lib.call("palu_rope_score_tc", K.bits, _ptr(K.rows), _ptr(K.scales), _ptr(K.zps), B,
                          n, L.s_k, K.G, K.r_pad, K.cap, _ptr(self.uw_bf), _ptr(self.rope_tab),
                          _ptr(self.t_dev), _ptr(self.logits), self.ld_logits, st)
        else:
            _lib.call("palu_rope_score", code, K.bits, _ptr(K.rows), _ptr(K.scales), _ptr(K.zps),
                      B, n, dh, L.s_k, K.G, K.r_pad, K.cap, _ptr(self.uw), _ptr(f.theta_dev),
                      _ptr(self.t_dev), _ptr(self.logits), self.ld_logits, st)
        self._value(li, st)

    def _value(self, li: int, st: int):
        """Softmax + value path + wo_fused GEMV of layer li (attention.py:445-446, 350-362)."""
        f, c = self.fused, self.cache
        L = f.layers[li]
        K, V = c._stores[li]
        B, d, n = self.B, self.d, self.n
        code = f.dtype_code
        if self.value_tc_layers[li]:
            _lib.call("palu_value_tc", V.bits, _ptr(V.rows), _ptr(V.scales), _ptr(V.zps), B, n,
                      L.s_v, V.G, V.r_pad, V.cap, _ptr(self.logits), self.ld_logits,
                      _ptr(self.t_dev), _ptr(L.ranks_v_dev), _ptr(L.o_off_dev), _ptr(self.ctx),
                      self.ko, _ptr(self.ws_fused), st)
        else:
            _lib.call("palu_softmax_value", code, V.bits, _ptr(V.rows), _ptr(V.scales), _ptr(V.zps),
                      B, n, L.s_v, V.G, V.r_pad, _ptr(L.ranks_v_dev), _ptr(L.o_off_dev), V.cap,
                      _ptr(self.logits), self.ld_logits, self.planes[li], self.plane,
                      _ptr(self.t_dev), self.n_chunks, _ptr(self.ws), _ptr(self.ctx), self.ko, st)
        self._proj(code, L.woT, d, L.ko_pad, self.ctx, self.x, st)

    def _proj(self, code, W, N: int, K: int, xt, yt, st: int):
        """y[:, :N] = x[:, :K] @ W[:N, :K]^T (attention.py:344-347, 430, 361).

        Decode batches (B < 16) stream the weights once through palu_gemv.  For
        B >= 16 the projection is a plain GEMM and goes to cuBLAS (bf16 weights,
        x split into bf16 hi + lo rows, fp32 output: ~16 mantissa bits of x):
        palu_gemv would re-stream the weights once per 2-4 batch rows."""
        B = self.B
        if B >= 16 and code == _lib.DTYPE_BF16:
            torch = _torch()
            xs = xt[:, :K]
            hi = xs.to(torch.bfloat16)
            lo = (xs - hi.float()).to(torch.bfloat16)
            out = torch.mm(torch.cat([hi, lo]), W[:N, :K].t(), out_dtype=torch.float32)
            torch.add(out[:B], out[B:], out=yt[:, :N])
        else:
            _lib.call("palu_gemv", code, _ptr(W), N, K, _ptr(xt), B, xt.shape[1], _ptr(yt), yt.shape[1], 0, st)

    def launch_step(self):
        """All layers + t += 1 on the current stream (graph-capturable)."""
        st = _stream()
        for li in range(len(self.fused.layers)):
            self._layer(li, st)
            if self.allreduce is not None:
                self.allreduce(self.x)
        _lib.call("palu_advance", _ptr(self.t_dev), st)

    def profile_step(self) -> dict:
        """One eager step with CUDA events around every launch; returns
        {entry point: [ms per launch]} (the roofline's live kernel timing)."""
        torch = _torch()
        recs = []
        orig = _lib.call

        def timed(name, *args):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = orig(name, *args)
            b.record()
            recs.append((name, a, b))
            return rc

        _lib.call = timed
        try:
            # keep the device busy while the host enqueues the step, so each
            # event pair brackets the kernel alone rather than the host's
            # launch latency (which dominated the short kernels' numbers)
            torch.cuda._sleep(20_000_000)
            self.launch_step()
        finally:
            _lib.call = orig
        torch.cuda.synchronize()
        out = {}
        for name, a, b in recs:
            out.setdefault(name, []).append(a.elapsed_time(b))
        return out

    def step_device(self):
        """Run one step on self.x (device) -> self.x; graph replay after warm-up."""
        torch = _torch()
        if not self.use_graph or self.eager_steps < 1:
            self.launch_step()
            self.eager_steps += 1
            return
        if self.graph is None:
            import gc

            # dead sessions (cache <-> session cycles) own CUDA graphs whose
            # destruction is illegal while a capture is open: collect them now
            # and keep the collector off until the capture ends
            gc.collect()
            gc_was_enabled = gc.isenabled()
            gc.disable()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            try:
                with torch.cuda.stream(s):
                    # capture does not execute: t_dev is unchanged by the capture itself
                    with torch.cuda.graph(g, stream=s):
                        self.launch_step()
            except Exception:  # a collective that cannot be captured: run eagerly
                if gc_was_enabled:
                    gc.enable()
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
                self.use_graph = False
                self.launch_step()
                return
            if gc_was_enabled:
                gc.enable()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = g
        self.graph.replay()


def replicated_key_operand(bk, r_pad: int, s_k: int, dh: int):
    """B_k of every group as the reconstruct-once score's B operand, or None.

    bk: [G][rows >= r_pad][s_k * dh] (the fused B_k blocks, one d_h block per
    query head of the group).  When every head block of every group is the
    same (GQA as its MHA-equivalent layer: one KV head per group, SURVEY
    7.2-10), returns bf16/fp32 [G][dh][r_pad] with row c = column c of the
    group's KV-head block (K-major for tcgen05); otherwise None.
    """
    b = bk[:, :r_pad]
    if b.shape[-1] != s_k * dh:
        return None
    blocks = b.reshape(b.shape[0], r_pad, s_k, dh)
    if not bool((blocks == blocks[:, :, :1]).all()):
        return None
    return blocks[:, :, 0].transpose(1, 2).contiguous()


def _session(fused, cache, score_kernel=None) -> _Session:
    s = cache._session
    score_kernel = score_kernel or getattr(cache, "score_kernel", "auto")
    if (s is None or s.fused is not fused or s.cap != cache.capacity
            or s.score_kernel != score_kernel):
        s = _Session(fused, cache, score_kernel=score_kernel)
        # a shard's reduction survives session rebuilds (capacity growth,
        # another score kernel): without it every rank would silently return
        # only its partial output
        s.allreduce = cache._allreduce
        cache._session = s
    return s


def _validate_x(x_t, cache) -> np.ndarray:
    x = np.asarray(x_t, dtype=np.float64)
    d = cache.config.d_model
    if x.ndim == 1:
        if cache.batch != 1 or x.shape[0] != d:
            raise ValidationError(f"x_t must have shape ({d},) for a batch-1 cache, got {x.shape}")
    elif x.ndim != 2 or x.shape != (cache.batch, d):
        raise ValidationError(f"x_t must have shape ({cache.batch}, {d}), got {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValidationError("x_t must be finite")
    return x


def palu_decode_step_rope(weights, fused: FusedWeights, cache: LatentKVCache, x_t,
                          tile_len: int | None = None) -> np.ndarray:
    """attention.py:392-448 -- one decode step with online key reconstruction.

    Validation happens before any mutation (rope on, tile_len >= 1, ranks,
    weight shapes, x shape).  The kernels' token tiling is fixed; the
    reference guarantees the output is independent of tile_len
    (SPEC.md:402), so tile_len is validated and otherwise has no effect.
    """
    cfg = cache.config
    if not cfg.rope:
        raise ValidationError("palu_decode_step_rope requires a rope-on config")
    if tile_len is not None and tile_len < 1:
        raise ValidationError(f"tile_len must be >= 1, got {tile_len}")
    _validate_step(weights, fused, cache)
    x = _validate_x(x_t, cache)
    torch = _torch()
    cache.reserve(cache.t + 1)
    s = _session(fused, cache)
    s.x_host.copy_(torch.from_numpy(x.reshape(cache.batch, -1).astype(np.float32)))
    s.x.copy_(s.x_host, non_blocking=True)
    s.step_device()
    s.out_host.copy_(s.x, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cache.t += 1
    out = s.out_host.numpy().astype(np.float64)
    return out[0].copy() if np.asarray(x_t).ndim == 1 else out.copy()


def palu_decode_step_norope(weights, fused: FusedWeights, cache: LatentKVCache, x_t) -> np.ndarray:
    """attention.py:365-389 -- one decode step with both fusions active (rope off).

    q_lat_i = x @ wq_fused[:, q_off[i]:] comes out of the first rows of the
    layer GEMV; the score is a GEMV of the latent key cache against it (tcgen05
    streaming kernel for bf16 latents, CUDA cores otherwise); softmax, value
    path and wo_fused as in the rope-on step.  Validation before any mutation.
    """
    cfg = cache.config
    if cfg.rope:
        raise ValidationError("palu_decode_step_norope requires a rope-off config")
    _validate_step(weights, fused, cache)
    x = _validate_x(x_t, cache)
    torch = _torch()
    cache.reserve(cache.t + 1)
    s = _session(fused, cache)
    s.x_host.copy_(torch.from_numpy(x.reshape(cache.batch, -1).astype(np.float32)))
    s.x.copy_(s.x_host, non_blocking=True)
    s.step_device()
    s.out_host.copy_(s.x, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cache.t += 1
    out = s.out_host.numpy().astype(np.float64)
    return out[0].copy() if np.asarray(x_t).ndim == 1 else out.copy()


def palu_decode_step_quantized(weights, fused, cache, x_t, tile_len=None) -> np.ndarray:
    """attention.py:451-466: quantisation lives in the cache; dispatch by rope."""
    if cache.config.rope:
        return palu_decode_step_rope(weights, fused, cache, x_t, tile_len)
    return palu_decode_step_norope(weights, fused, cache, x_t)


def palu_prefill(weights, decomposed, config, prompt, bits=FP_BITS, fused=None, tile_len=None,
                 *, dtype: str = "float32", batched: bool = True) -> LatentKVCache:
    """attention.py:469-494: the cache after feeding the prompt.

    batched=True (rope on): one causal attention pass per layer over the
    whole prompt (prefill.py); batched=False: token-by-token decode steps,
    the reference's own schedule."""
    tokens = np.asarray(prompt, dtype=np.float64)
    if tokens.ndim != 2 or tokens.shape[1] != config.d_model:
        raise ValidationError(f"prompt must be (T, {config.d_model})")
    if tile_len is not None and tile_len < 1:
        raise ValidationError(f"tile_len must be >= 1, got {tile_len}")
    if batched and config.rope:
        from .prefill import palu_prefill_batched
        return palu_prefill_batched(weights, decomposed, config, tokens, bits, fused, tile_len, dtype=dtype)
    if fused is None:
        fused = build_fused(weights, decomposed, config, dtype=dtype)
    cache = LatentKVCache(decomposed, config, bits, dtype=fused.dtype,
                          capacity=max(tokens.shape[0], 8))
    for t in range(tokens.shape[0]):
        if config.rope:
            palu_decode_step_rope(weights, fused, cache, tokens[t], tile_len)
        else:
            palu_decode_step_norope(weights, fused, cache, tokens[t])
    return cache


def palu_decode(weights, decomposed, config, token_stream, bits=FP_BITS, tile_len=None,
                *, dtype: str = "float32"):
    """attention.py:497-515: decode a whole stream -> (outputs (T, d), cache)."""
    tokens = np.asarray(token_stream, dtype=np.float64)
    fused = build_fused(weights, decomposed, config, dtype=dtype)
    cache = LatentKVCache(decomposed, config, bits, dtype=dtype, capacity=max(tokens.shape[0], 8))
    outputs = np.zeros_like(tokens)
    for t in range(tokens.shape[0]):
        if config.rope:
            outputs[t] = palu_decode_step_rope(weights, fused, cache, tokens[t], tile_len)
        else:
            outputs[t] = palu_decode_step_norope(weights, fused, cache, tokens[t])
    return outputs, cache
