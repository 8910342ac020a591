"""CPU oracle for the Palu RoPE latent-KV decode path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy float64 restatement of the reference algorithm in
``/root/reference/pkg/src/palu`` for the one hot path this repository
accelerates (``palu_decode_step_rope`` and what it calls).  It exists to CHECK
the CUDA product path, never to BE it: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product package (``paper_2407_21118_b200``) never imports this file and
fails loudly when its CUDA library is missing.

Parity pin: every public function here is checked against fixtures generated
by running the reference itself (``tests/golden/make_golden.py``, committed
together with the ``.npz`` outputs) -- see ``tests/test_oracle_golden.py``.

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FP_BITS = 16  # attention.py:31 -- "16 bits" means a raw float64 store, not fp16
SUPPORTED_BITS = (2, 3, 4, 8)  # quant.py:28
_RANGE_FLOOR = 1e-8  # quant.py:27


# --------------------------------------------------------------------------
# core.py: counter-based seeded matrices and Hadamard construction
# --------------------------------------------------------------------------
_MIX_INC = np.uint64(0x9E3779B97F4A7C15)
_MIX_A = np.uint64(0xBF58476D1CE4E5B9)
_MIX_B = np.uint64(0x94D049BB133111EB)
_ROW_SALT = np.uint64(0xD6E8FEB86659FD93)
_COL_SALT = np.uint64(0xA5A5A5A5B4B4B4B5)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """core.py:324-328 (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + _MIX_INC
        z = (z ^ (z >> np.uint64(30))) * _MIX_A
        z = (z ^ (z >> np.uint64(27))) * _MIX_B
    return z ^ (z >> np.uint64(31))


def cell_uniform(seed: int, rows: int, cols: int, stream: int = 0,
                 row0: int = 0) -> np.ndarray:
    """core.py:331-343 -- uniform [0,1) keyed by (seed, stream, row, col).

    ``row0`` lets callers generate a row band of a larger matrix (the hash is
    per cell, so any band equals the same rows of the full matrix).
    """
    base = np.uint64((seed ^ (stream * 0x517CC1B727220A95)) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        r = (np.arange(row0, row0 + rows, dtype=np.uint64) + np.uint64(1)) * _ROW_SALT
        c = (np.arange(cols, dtype=np.uint64) + np.uint64(1)) * _COL_SALT
    state = _splitmix64(base ^ r[:, None]) ^ c[None, :]
    h = _splitmix64(state)
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_matrix(rows: int, cols: int, seed: int, row0: int = 0) -> np.ndarray:
    """core.py:346-356 (``spectrum=None`` branch): entries uniform on [-1, 1)."""
    if rows < 1 or cols < 1:
        raise ValueError(f"random_matrix dimensions must be positive, got {rows}x{cols}")
    return 2.0 * cell_uniform(seed, rows, cols, row0=row0) - 1.0


def _sylvester(block: int) -> np.ndarray:
    """core.py:282-288."""
    h = np.array([[1.0]])
    size = 1
    while size < block:
        h = np.block([[h, h], [h, -h]])
        size *= 2
    return h / math.sqrt(block)


def hadamard(dim: int) -> np.ndarray:
    """core.py:291-313: Sylvester blocks over the binary decomposition of dim."""
    if dim <= 0:
        raise ValueError(f"hadamard dimension must be positive, got {dim}")
    out = np.zeros((dim, dim))
    at, remaining = 0, dim
    while remaining:
        p = 1 << (remaining.bit_length() - 1)
        out[at:at + p, at:at + p] = _sylvester(p)
        at += p
        remaining -= p
    return out


def fuse_hadamard(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """quant.py:127-153 for one group: (A, B) -> (A R, R^T B)."""
    r = hadamard(a.shape[1])
    return a @ r, r.T @ b


# --------------------------------------------------------------------------
# quant.py: per-token asymmetric quantiser and LE bit-packing
# --------------------------------------------------------------------------
def round_half_away(x: np.ndarray) -> np.ndarray:
    """quant.py:31-32."""
    return np.where(x >= 0.0, np.floor(x + 0.5), np.ceil(x - 0.5))


def quantize_rows(x: np.ndarray, bits: int):
    """quant.py:87-99 -> (codes uint8, scales f64, zero_points int64)."""
    if bits not in SUPPORTED_BITS:
        raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
    x = np.asarray(x, dtype=np.float64)
    qmax = (1 << bits) - 1
    if x.size == 0:
        return (np.zeros(x.shape, dtype=np.uint8), np.ones(x.shape[0]),
                np.zeros(x.shape[0], dtype=np.int64))
    lo = x.min(axis=1)
    hi = x.max(axis=1)
    scales = np.maximum(hi - lo, _RANGE_FLOOR) / qmax
    zps = round_half_away(-lo / scales).astype(np.int64)
    q = round_half_away(x / scales[:, None]) + zps[:, None]
    codes = np.clip(q, 0, qmax).astype(np.uint8)
    return codes, scales, zps


def dequantize_rows(codes, scales, zps) -> np.ndarray:
    """quant.py:106-107 (and attention.py:265-268)."""
    return (np.asarray(codes).astype(np.float64) - np.asarray(zps, dtype=np.float64)[:, None]) \
        * np.asarray(scales)[:, None]


def pack_codes(codes: np.ndarray, bits: int) -> bytes:
    """quant.py:156-169: code i at bits [i*bits, (i+1)*bits) from the LSB of byte 0."""
    if bits not in SUPPORTED_BITS:
        raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size and flat.max() >= (1 << bits):
        raise ValueError(f"code exceeds {bits}-bit range")
    bit_cols = (flat[:, None] >> np.arange(bits, dtype=np.uint8)) & 1
    return np.packbits(bit_cols.reshape(-1), bitorder="little").tobytes()


def unpack_codes(data: bytes, count: int, bits: int) -> np.ndarray:
    """quant.py:172-181."""
    need = math.ceil(count * bits / 8)
    if len(data) < need:
        raise ValueError(f"packed payload too short: {len(data)} bytes for {count} codes")
    raw = np.frombuffer(data, dtype=np.uint8, count=need)
    stream = np.unpackbits(raw, bitorder="little")[: count * bits]
    weights = (1 << np.arange(bits)).astype(np.uint8)
    return (stream.reshape(count, bits) * weights).sum(axis=1).astype(np.uint8)


# --------------------------------------------------------------------------
# attention.py: RoPE, softmax, fusion, latent cache, decode steps
# --------------------------------------------------------------------------
def rope_rows(rows: np.ndarray, positions: np.ndarray, base: float) -> np.ndarray:
    """attention.py:105-112: half-split rotary, dim i pairs with i + d/2."""
    d = rows.shape[1]
    half = d // 2
    idx = np.arange(half, dtype=np.float64)
    angles = np.asarray(positions, dtype=np.float64)[:, None] * base ** (-2.0 * idx / d)
    cos, sin = np.cos(angles), np.sin(angles)
    lo, hi = rows[:, :half], rows[:, half:]
    return np.concatenate([lo * cos - hi * sin, lo * sin + hi * cos], axis=1)


def softmax(logits: np.ndarray) -> np.ndarray:
    """attention.py:115-118."""
    shifted = logits - logits.max()
    e = np.exp(shifted)
    return e / e.sum()


@dataclass
class OracleLayer:
    """One layer of weights and factors as plain arrays (attention.py:57-90).

    ``ak``/``bk``/``av``/``bv`` are per-group factor lists: A_g is d x r_g and
    B_g is r_g x (s * d_h) (decompose.py:75-118).
    """

    wq: np.ndarray
    wo: np.ndarray
    ak: list
    bk: list
    av: list
    bv: list
    s_k: int
    s_v: int
    wk: np.ndarray | None = None  # only the uncompressed baseline needs these
    wv: np.ndarray | None = None

    @property
    def key_ranks(self):
        return tuple(a.shape[1] for a in self.ak)

    @property
    def value_ranks(self):
        return tuple(a.shape[1] for a in self.av)


def head_offsets(ranks, s: int, n_heads: int) -> tuple[int, ...]:
    """attention.py:171-176: head i owns rank(group(i)) rows."""
    offs = [0]
    for i in range(n_heads):
        offs.append(offs[-1] + ranks[i // s])
    return tuple(offs)


def build_wo_fused(layer: OracleLayer, n_heads: int, head_dim: int) -> np.ndarray:
    """attention.py:214-225: wo block i = B_v[g][:, i-in-g] @ W_o[rows i]."""
    dh = head_dim
    blocks = []
    for i in range(n_heads):
        gv, pv = divmod(i, layer.s_v)
        bv = layer.bv[gv][:, pv * dh:(pv + 1) * dh]
        blocks.append(bv @ layer.wo[i * dh:(i + 1) * dh, :])
    return np.concatenate(blocks, axis=0)


def build_wq_fused(layer: OracleLayer, n_heads: int, head_dim: int) -> np.ndarray:
    """attention.py:217-220 (rope off only): wq block i = W_q[:, i] @ B_k[g][:, i-in-g]^T."""
    dh = head_dim
    blocks = []
    for i in range(n_heads):
        gk, pk = divmod(i, layer.s_k)
        bk = layer.bk[gk][:, pk * dh:(pk + 1) * dh]
        blocks.append(layer.wq[:, i * dh:(i + 1) * dh] @ bk.T)
    return np.concatenate(blocks, axis=1)


class GroupStoreOracle:
    """attention.py:235-268 restated over a preallocated array.

    Raw rows are kept as float64; quantised rows keep (codes, scale, zp) and
    are dequantised on read exactly as ``_GroupStore.matrix`` does.
    """

    def __init__(self, rank: int, bits: int, capacity: int = 16):
        self.rank, self.bits, self.n = rank, bits, 0
        cap = max(capacity, 1)
        if bits == FP_BITS:
            self.rows = np.zeros((cap, rank))
        else:
            self.codes = np.zeros((cap, rank), dtype=np.uint8)
            self.scales = np.ones(cap)
            self.zps = np.zeros(cap, dtype=np.int64)

    def _grow(self, need: int):
        cap = self.rows.shape[0] if self.bits == FP_BITS else self.codes.shape[0]
        if need <= cap:
            return
        new = max(need, 2 * cap)
        if self.bits == FP_BITS:
            self.rows = np.concatenate([self.rows, np.zeros((new - cap, self.rank))])
        else:
            self.codes = np.concatenate([self.codes, np.zeros((new - cap, self.rank), np.uint8)])
            self.scales = np.concatenate([self.scales, np.ones(new - cap)])
            self.zps = np.concatenate([self.zps, np.zeros(new - cap, np.int64)])

    def extend(self, rows: np.ndarray) -> None:
        """Append rows; quantised per token (attention.py:248-255)."""
        rows = np.atleast_2d(np.asarray(rows, dtype=np.float64))
        k = rows.shape[0]
        self._grow(self.n + k)
        if self.bits == FP_BITS:
            self.rows[self.n:self.n + k] = rows
        else:
            c, s, z = quantize_rows(rows, self.bits)
            self.codes[self.n:self.n + k] = c
            self.scales[self.n:self.n + k] = s
            self.zps[self.n:self.n + k] = z
        self.n += k

    def truncate(self, n: int) -> None:
        self.n = n

    def matrix(self) -> np.ndarray:
        """attention.py:257-268."""
        if self.bits == FP_BITS:
            return self.rows[:self.n]
        return dequantize_rows(self.codes[:self.n], self.scales[:self.n], self.zps[:self.n])


def norm_bits(bits) -> tuple[int, int]:
    """attention.py:292-300."""
    pair = (bits, bits) if isinstance(bits, int) else tuple(bits)
    if len(pair) != 2:
        raise ValueError(f"bits must be an int or a (key, value) pair, got {bits!r}")
    for b in pair:
        if b != FP_BITS and b not in SUPPORTED_BITS:
            raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {b}")
    return pair


@dataclass
class OracleCache:
    """attention.py:303-331: per layer, one store per K group and per V group."""

    layers: list
    bits: object = FP_BITS
    t: int = 0
    k_stores: list = field(default_factory=list)
    v_stores: list = field(default_factory=list)

    def __post_init__(self):
        kb, vb = norm_bits(self.bits)
        self.k_bits, self.v_bits = kb, vb
        self.k_stores = [[GroupStoreOracle(r, kb) for r in L.key_ranks] for L in self.layers]
        self.v_stores = [[GroupStoreOracle(r, vb) for r in L.value_ranks] for L in self.layers]

    def fill_direct(self, li: int, x_rows: np.ndarray) -> None:
        """Direct O(T) cache fill used by the bench/parity harness:
        append ``x_rows @ A_g`` for every group, same as T calls of
        ``_append_latents`` (attention.py:343-347) with fixed inputs."""
        L = self.layers[li]
        for a, st in zip(L.ak, self.k_stores[li]):
            st.extend(x_rows @ a)
        for a, st in zip(L.av, self.v_stores[li]):
            st.extend(x_rows @ a)

    def hk(self, li):
        return np.concatenate([s.matrix() for s in self.k_stores[li]], axis=1)

    def hv(self, li):
        return np.concatenate([s.matrix() for s in self.v_stores[li]], axis=1)


def append_latents(layer: OracleLayer, cache: OracleCache, li: int, x: np.ndarray) -> None:
    """attention.py:343-347: K groups first, then V groups."""
    for a, st in zip(layer.ak, cache.k_stores[li]):
        st.extend((x @ a)[None, :])
    for a, st in zip(layer.av, cache.v_stores[li]):
        st.extend((x @ a)[None, :])


def value_output(wo_fused, o_off, cache: OracleCache, li: int, probs, s_v: int, d: int):
    """attention.py:350-362."""
    out = np.zeros(d)
    hv = [st.matrix() for st in cache.v_stores[li]]
    for i, p in enumerate(probs):
        ctx = p @ hv[i // s_v]
        out += ctx @ wo_fused[o_off[i]:o_off[i + 1], :]
    return out


def decode_step_rope(layers, wo_fused_list, cache: OracleCache, x_t, n_heads: int,
                     head_dim: int, rope_base: float, tile_len=None,
                     return_logits: bool = False):
    """attention.py:392-448 -- one RoPE decode step over every layer.

    Appends (and quantises) the current token's latents first, rebuilds keys
    tile by tile as H_tile @ B_g, rotates them at their absolute positions,
    scores against the rotated query, softmaxes and applies the fused value
    path.  Mutates ``cache`` (one row per group per layer, then t += 1).
    """
    if tile_len is not None and tile_len < 1:
        raise ValueError(f"tile_len must be >= 1, got {tile_len}")
    x = np.asarray(x_t, dtype=np.float64)
    n, dh = n_heads, head_dim
    d = n * dh
    scale = 1.0 / math.sqrt(dh)
    pos_t = float(cache.t)
    all_logits = []
    for li, L in enumerate(layers):
        append_latents(L, cache, li, x)
        t_rows = cache.t + 1
        tile = t_rows if tile_len is None else tile_len
        queries = []
        for i in range(n):
            q = x @ L.wq[:, i * dh:(i + 1) * dh]
            queries.append(rope_rows(q[None, :], np.array([pos_t]), rope_base)[0])
        logits = np.zeros((n, t_rows))
        for g, st in enumerate(cache.k_stores[li]):
            h_all = st.matrix()
            b = L.bk[g]
            for start in range(0, t_rows, tile):
                stop = min(start + tile, t_rows)
                k_tile = h_all[start:stop] @ b
                positions = np.arange(start, stop, dtype=np.float64)
                for p in range(L.s_k):
                    head = g * L.s_k + p
                    k_head = rope_rows(k_tile[:, p * dh:(p + 1) * dh], positions, rope_base)
                    logits[head, start:stop] = k_head @ queries[head] * scale
        all_logits.append(logits)
        probs = [softmax(logits[i]) for i in range(n)]
        o_off = head_offsets(L.value_ranks, L.s_v, n)
        x = value_output(wo_fused_list[li], o_off, cache, li, probs, L.s_v, d)
    cache.t += 1
    return (x, all_logits) if return_logits else x


def decode_step_norope(layers, wq_fused_list, wo_fused_list, cache: OracleCache, x_t,
                       n_heads: int, head_dim: int):
    """attention.py:365-389 -- both fusions active (rope off)."""
    x = np.asarray(x_t, dtype=np.float64)
    n, dh = n_heads, head_dim
    d = n * dh
    scale = 1.0 / math.sqrt(dh)
    for li, L in enumerate(layers):
        append_latents(L, cache, li, x)
        q_off = head_offsets(L.key_ranks, L.s_k, n)
        hk = [st.matrix() for st in cache.k_stores[li]]
        probs = []
        for i in range(n):
            q_lat = x @ wq_fused_list[li][:, q_off[i]:q_off[i + 1]]
            probs.append(softmax(hk[i // L.s_k] @ q_lat * scale))
        o_off = head_offsets(L.value_ranks, L.s_v, n)
        x = value_output(wo_fused_list[li], o_off, cache, li, probs, L.s_v, d)
    cache.t += 1
    return x


# --------------------------------------------------------------------------
# Uncompressed baseline: attention.py:133-168 (reference_decode), one step
# over an explicit post-RoPE key cache.
# --------------------------------------------------------------------------
@dataclass
class DenseCacheOracle:
    keys: list  # per layer (t, d), rotary already applied
    values: list
    t: int = 0


def reference_step(wq, wk, wv, wo, cache: DenseCacheOracle, x_t, n_heads, head_dim,
                   rope: bool, rope_base: float):
    """attention.py:144-167 for a single token over every layer."""
    x = np.asarray(x_t, dtype=np.float64)
    n, dh = n_heads, head_dim
    d = n * dh
    t = cache.t
    for li in range(len(wq)):
        k_row = x @ wk[li]
        v_row = x @ wv[li]
        if rope:
            pos = np.array([t], dtype=np.float64)
            k_row = np.concatenate(
                [rope_rows(k_row[None, i * dh:(i + 1) * dh], pos, rope_base)[0] for i in range(n)])
        cache.keys[li] = np.vstack([cache.keys[li], k_row])
        cache.values[li] = np.vstack([cache.values[li], v_row])
        out = np.zeros(d)
        for h in range(n):
            sl = slice(h * dh, (h + 1) * dh)
            q = x @ wq[li][:, sl]
            if rope:
                q = rope_rows(q[None, :], np.array([t], dtype=np.float64), rope_base)[0]
            probs = softmax(cache.keys[li][:, sl] @ q / math.sqrt(dh))
            out += (probs @ cache.values[li][:, sl]) @ wo[li][sl, :]
        x = out
    cache.t += 1
    return x


# --------------------------------------------------------------------------
# Synthetic inputs: seeded, scaled uniform weights and factors.
# --------------------------------------------------------------------------
def synth_layer(d: int, n_heads: int, head_dim: int, s_k: int, ranks_k, s_v: int, ranks_v,
                seed: int, hadamard_fused: bool = False, with_kv: bool = False) -> OracleLayer:
    """Seeded synthetic layer: W = U[-1,1)/sqrt(d), A_g = U/sqrt(d), B_g = U/sqrt(r).

    Seeds: W_q = seed, W_o = seed+3, W_k = seed+1, W_v = seed+2 (the reference
    test convention, tests/test_attention.py:40-53); K group g factors use
    seeds seed+1000+2g / +1, V group g factors seed+2000+2g / +1.
    """
    sq = 1.0 / math.sqrt(d)
    wq = random_matrix(d, d, seed) * sq
    wo = random_matrix(d, d, seed + 3) * sq
    gk, gv = n_heads // s_k, n_heads // s_v
    ranks_k = [ranks_k] * gk if isinstance(ranks_k, int) else list(ranks_k)
    ranks_v = [ranks_v] * gv if isinstance(ranks_v, int) else list(ranks_v)
    ak, bk, av, bv = [], [], [], []
    for g, r in enumerate(ranks_k):
        a = random_matrix(d, r, seed + 1000 + 2 * g) * sq
        b = random_matrix(r, s_k * head_dim, seed + 1001 + 2 * g) / math.sqrt(r)
        if hadamard_fused:
            a, b = fuse_hadamard(a, b)
        ak.append(a)
        bk.append(b)
    for g, r in enumerate(ranks_v):
        a = random_matrix(d, r, seed + 2000 + 2 * g) * sq
        b = random_matrix(r, s_v * head_dim, seed + 2001 + 2 * g) / math.sqrt(r)
        if hadamard_fused:
            a, b = fuse_hadamard(a, b)
        av.append(a)
        bv.append(b)
    wk = random_matrix(d, d, seed + 1) * sq if with_kv else None
    wv = random_matrix(d, d, seed + 2) * sq if with_kv else None
    return OracleLayer(wq=wq, wo=wo, ak=ak, bk=bk, av=av, bv=bv, s_k=s_k, s_v=s_v, wk=wk, wv=wv)


# --------------------------------------------------------------------------
# GQA (BASELINE configs[3], Mistral-7B: 32 query heads, 8 KV heads).  The
# reference has no GQA (AttentionConfig forces d = n d_h, attention.py:44-47);
# the MHA-equivalent layer replicates each KV head's factors across the
# query heads that share it, so the unchanged reference
# computes exact GQA semantics.  gqa_decode_step_rope is an independent
# KV-head restatement used to check that equivalence.
# --------------------------------------------------------------------------
def synth_gqa_layer(d: int, n_q: int, n_kv: int, head_dim: int, rank_k: int, rank_v: int,
                    seed: int, hadamard_fused: bool = False) -> OracleLayer:
    """Replicated-B layer: group j = the n_q / n_kv query heads of KV head j,
    A_j = U(d x r)/sqrt(d), B_j = [B_kv B_kv ...] with B_kv = U(r x d_h)/sqrt(r)."""
    s = n_q // n_kv
    sq = 1.0 / math.sqrt(d)
    wq = random_matrix(d, d, seed) * sq
    wo = random_matrix(d, d, seed + 3) * sq
    ak, bk, av, bv = [], [], [], []
    for g in range(n_kv):
        for r, dst_a, dst_b, off in ((rank_k, ak, bk, 1000), (rank_v, av, bv, 2000)):
            a = random_matrix(d, r, seed + off + 2 * g) * sq
            b = np.tile(random_matrix(r, head_dim, seed + off + 1 + 2 * g) / math.sqrt(r), (1, s))
            if hadamard_fused:
                a, b = fuse_hadamard(a, b)
            dst_a.append(a)
            dst_b.append(b)
    return OracleLayer(wq=wq, wo=wo, ak=ak, bk=bk, av=av, bv=bv, s_k=s, s_v=s)


def gqa_decode_step_rope(layer: OracleLayer, hk: np.ndarray, hv: np.ndarray, x_t, n_q: int,
                         n_kv: int, head_dim: int, rope_base: float, t: int) -> np.ndarray:
    """One GQA decode step over KV heads (not via the MHA-equivalent path):
    keys of KV head j = rope(H_k,j B_kv,j), query head i attends to KV head
    i // (n_q / n_kv); H_k / H_v hold rows 0..t (the newest token's included)."""
    s, dh = n_q // n_kv, head_dim
    x = np.asarray(x_t, dtype=np.float64)
    off_k = np.concatenate([[0], np.cumsum([a.shape[1] for a in layer.ak])])
    off_v = np.concatenate([[0], np.cumsum([a.shape[1] for a in layer.av])])
    pos = np.arange(t + 1, dtype=np.float64)
    out = np.zeros(n_q * dh)
    for j in range(n_kv):
        keys = rope_rows(hk[:, off_k[j]:off_k[j + 1]] @ layer.bk[j][:, :dh], pos, rope_base)
        vals = hv[:, off_v[j]:off_v[j + 1]] @ layer.bv[j][:, :dh]
        for i in range(j * s, (j + 1) * s):
            q = rope_rows((x @ layer.wq[:, i * dh:(i + 1) * dh])[None, :], np.array([float(t)]),
                          rope_base)[0]
            p = softmax(keys @ q / math.sqrt(dh))
            out += (p @ vals) @ layer.wo[i * dh:(i + 1) * dh, :]
    return out

