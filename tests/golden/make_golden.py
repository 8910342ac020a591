"""Generate golden fixtures by running the UNMODIFIED reference (read-only import).

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It writes small ``.npz`` files next to this script.  They pin the CPU oracle
(``oracle/palu_oracle.py``) and, through it, the CUDA path.  Nothing at test or
bench time reads /root/reference; only this generator does.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)

from palu.attention import (  # noqa: E402
    AttentionConfig,
    LatentKVCache,
    LayerKV,
    LayerWeights,
    ModelWeights,
    build_fused,
    palu_decode,
    palu_decode_step_rope,
    reference_decode,
)
from palu.core import Matrix, random_matrix  # noqa: E402
from palu.decompose import DecomposedLayer, Granularity, GroupFactors, decompose  # noqa: E402
from palu.quant import QuantParams, fuse_hadamard, pack_codes, quantize_rows  # noqa: E402
from oracles import naive_decode_latent  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


# ----------------------------------------------------------------------------
def gen_rng():
    shapes = [(3, 5, 0), (7, 11, 42), (16, 16, 12345), (1, 64, 2**40 + 7), (33, 9, 2**63 - 1)]
    out = {}
    for i, (r, c, s) in enumerate(shapes):
        out[f"m{i}"] = random_matrix(r, c, seed=s).data
        out[f"m{i}_shape_seed"] = np.array([r, c, s], dtype=np.uint64)
    big = random_matrix(512, 4096, seed=777).data
    out["big_sha256"] = np.frombuffer(hashlib.sha256(big.tobytes()).digest(), dtype=np.uint8)
    out["big_row_301"] = big[301]
    _save("rng.npz", **out)


# ----------------------------------------------------------------------------
def gen_quant():
    rows = [
        np.array([0.0, 1.0, 2.0, 3.0, 0.0, 1.0, 2.0, 3.0]),  # lattice aligned (test_quant.py:22-26)
        np.array([-1.0, 0.0, 1.0, -1.0, 0.0, 1.0, 0.5, -0.5]),  # clamp bites (test_quant.py:34-42)
        np.full(8, 5.0),  # constant row -> range floor
        np.full(8, -2.5),
        np.linspace(0.1, 9.0, 8),  # all positive -> negative zero point
        np.linspace(-9.0, -0.1, 8),  # all negative
        np.array([1e-9, -1e-9, 0.0, 1e-9, 0.0, 0.0, -1e-9, 0.0]),  # below the range floor
        np.array([0.5, 1.5, 2.5, -0.5, -1.5, 3.5, 4.5, -2.5]),  # half-way ties
    ]
    x_edge = np.stack(rows)
    x_rand = random_matrix(256, 64, seed=9).data * 3.0
    x_big = random_matrix(64, 256, seed=901).data * 5.0 + random_matrix(64, 1, seed=902).data * 4.0
    out = {"x_edge": x_edge, "x_rand": x_rand, "x_big": x_big}
    for bits in (2, 3, 4, 8):
        for name, x in (("edge", x_edge), ("rand", x_rand), ("big", x_big)):
            q = quantize_rows(x, QuantParams(bits))
            out[f"{name}_b{bits}_codes"] = q.codes
            out[f"{name}_b{bits}_scales"] = q.scales
            out[f"{name}_b{bits}_zps"] = q.zero_points
            out[f"{name}_b{bits}_packed"] = np.frombuffer(pack_codes(q.codes, bits), dtype=np.uint8)
    _save("quant.npz", **out)


# ----------------------------------------------------------------------------
def _weights(d, layers, seed, scale=1.0):
    out = []
    for li in range(layers):
        base = seed + 101 * li
        out.append(LayerWeights(
            wq=Matrix(random_matrix(d, d, seed=base).data * scale),
            wk=Matrix(random_matrix(d, d, seed=base + 1).data * scale),
            wv=Matrix(random_matrix(d, d, seed=base + 2).data * scale),
            wo=Matrix(random_matrix(d, d, seed=base + 3).data * scale),
        ))
    return ModelWeights(layers=tuple(out))


SMALL_CASES = [
    # name, rope, layers, gran_k, rank_k, gran_v, rank_v, bits, tile_len, hadamard, T
    ("rope_joint_full", True, 2, ("joint", 4), 16, None, None, 16, None, False, 8),
    ("rope_group2_r5", True, 2, ("group", 2), 5, None, None, 16, 3, False, 9),
    ("rope_multi_r2", True, 2, ("multi", 1), 2, None, None, 16, 3, False, 8),
    ("rope_mixed", True, 1, ("multi", 1), 2, ("joint", 4), 9, 16, None, False, 6),
    ("rope_b4_multi_r3", True, 2, ("multi", 1), 3, None, None, 4, 2, False, 7),
    ("rope_b16_4_group2", True, 2, ("group", 2), 4, None, None, (16, 4), 2, False, 6),
    ("rope_b8_joint", True, 1, ("joint", 4), 16, None, None, 8, None, False, 8),
    ("rope_b3_group2", True, 1, ("group", 2), 7, None, None, 3, 4, False, 10),
    ("rope_b2_group2_had", True, 1, ("group", 2), 6, None, None, 2, None, True, 12),
    ("rope_b4_had_mixed", True, 2, ("group", 2), 8, ("multi", 1), 3, 4, 5, True, 9),
    ("norope_group2_r5", False, 2, ("group", 2), 5, None, None, 16, None, False, 8),
    ("norope_b4_multi", False, 1, ("multi", 1), 3, None, None, 4, None, False, 7),
    ("rope_base_1e6", True, 1, ("group", 2), 6, None, None, 16, None, False, 10),
]


def _gran(spec, n):
    kind, s = spec
    if kind == "joint":
        return Granularity.joint_head(n)
    if kind == "multi":
        return Granularity.multi_head()
    return Granularity.group_head(s)


def gen_small():
    n, dh = 4, 4
    d = n * dh
    out = {}
    names = []
    for ci, (name, rope, layers, gk, rk, gv, rv, bits, tile, had, T) in enumerate(SMALL_CASES):
        base = 1e6 if name == "rope_base_1e6" else 10000.0
        config = AttentionConfig(d, n, dh, layers=layers, rope=rope, rope_base=base)
        weights = _weights(d, layers, seed=300 + 17 * ci)
        gran_k = _gran(gk, n)
        gran_v = _gran(gv, n) if gv else gran_k
        rv = rk if rv is None else rv
        decomposed = []
        for lw in weights.layers:
            key = decompose(lw.wk, n, dh, gran_k, rk)
            value = decompose(lw.wv, n, dh, gran_v, rv)
            if had:
                key = fuse_hadamard(key).layer
                value = fuse_hadamard(value).layer
            decomposed.append(LayerKV(key=key, value=value))
        toks = random_matrix(T, d, seed=900 + ci).data * 0.5
        got, cache = palu_decode(weights, decomposed, config, toks, bits=bits, tile_len=tile)
        p = f"c{ci}_"
        names.append(name)
        out[p + "meta"] = np.array([rope, layers, gran_k.group_size, gran_v.group_size,
                                    rk, rv, T, had, base], dtype=np.float64)
        out[p + "bits"] = np.array(bits if isinstance(bits, tuple) else (bits, bits))
        out[p + "tile"] = np.array([-1 if tile is None else tile])
        out[p + "tokens"] = toks
        out[p + "outputs"] = got
        for li, (lw, kv) in enumerate(zip(weights.layers, decomposed)):
            out[p + f"L{li}_wq"] = lw.wq.data
            out[p + f"L{li}_wo"] = lw.wo.data
            out[p + f"L{li}_wk"] = lw.wk.data
            out[p + f"L{li}_wv"] = lw.wv.data
            for g, gf in enumerate(kv.key.groups):
                out[p + f"L{li}_ak{g}"] = gf.a.data
                out[p + f"L{li}_bk{g}"] = gf.b.data
            for g, gf in enumerate(kv.value.groups):
                out[p + f"L{li}_av{g}"] = gf.a.data
                out[p + f"L{li}_bv{g}"] = gf.b.data
            # the cache exactly as the reference holds it after the stream
            if cache.k_bits == 16:
                out[p + f"L{li}_hk"] = cache.hk(li)
            else:
                for g, st in enumerate(cache.layers[li].k_groups):
                    q = st.quantized_latent()
                    out[p + f"L{li}_k{g}_codes"] = q.codes
                    out[p + f"L{li}_k{g}_scales"] = q.scales
                    out[p + f"L{li}_k{g}_zps"] = q.zero_points
            if cache.v_bits == 16:
                out[p + f"L{li}_hv"] = cache.hv(li)
        if not had and bits == 16:
            ref = reference_decode(weights, config, toks).outputs
            out[p + "reference_decode"] = ref
        if rope and not had:
            lwd = [{"wq": lw.wq.data, "wk": lw.wk.data, "wv": lw.wv.data, "wo": lw.wo.data}
                   for lw in weights.layers]
            lfd = [{"k": [(g.a.data, g.b.data) for g in kv.key.groups],
                    "v": [(g.a.data, g.b.data) for g in kv.value.groups]} for kv in decomposed]
            if bits == 16:
                out[p + "naive_latent"] = naive_decode_latent(lwd, lfd, n, dh, toks, rope=True,
                                                              rope_base=base)
    out["names"] = np.array(names)
    _save("small_decode.npz", **out)


# ----------------------------------------------------------------------------
def _synth_ref_layer(d, n, dh, s_k, ranks_k, s_v, ranks_v, seed, hadamard_fused=False):
    """Reference-typed twin of oracle.synth_layer (same seeds and scaling)."""
    sq = 1.0 / math.sqrt(d)
    lw = LayerWeights(
        wq=Matrix(random_matrix(d, d, seed=seed).data * sq),
        wk=Matrix(random_matrix(d, d, seed=seed + 1).data * sq),
        wv=Matrix(random_matrix(d, d, seed=seed + 2).data * sq),
        wo=Matrix(random_matrix(d, d, seed=seed + 3).data * sq),
    )
    kg, vg = [], []
    for g, r in enumerate(ranks_k):
        a = random_matrix(d, r, seed=seed + 1000 + 2 * g).data * sq
        b = random_matrix(r, s_k * dh, seed=seed + 1001 + 2 * g).data / math.sqrt(r)
        kg.append(GroupFactors(a=Matrix(a), b=Matrix(b), rank=r))
    for g, r in enumerate(ranks_v):
        a = random_matrix(d, r, seed=seed + 2000 + 2 * g).data * sq
        b = random_matrix(r, s_v * dh, seed=seed + 2001 + 2 * g).data / math.sqrt(r)
        vg.append(GroupFactors(a=Matrix(a), b=Matrix(b), rank=r))

    def gran(s):
        if s == 1:
            return Granularity.multi_head()
        if s == n:
            return Granularity.joint_head(n)
        return Granularity.group_head(s)

    key = DecomposedLayer(gran(s_k), tuple(kg), d, dh, n)
    value = DecomposedLayer(gran(s_v), tuple(vg), d, dh, n)
    if hadamard_fused:
        key = fuse_hadamard(key).layer
        value = fuse_hadamard(value).layer
    return lw, LayerKV(key=key, value=value)


def _direct_fill(cache, kv, li, x_rows):
    """O(T) fill through the reference's own _GroupStore.append (attention.py:248-255)."""
    for g, st in zip(kv.key.groups, cache.layers[li].k_groups):
        h = x_rows @ g.a.data
        for row in h:
            st.append(row)
    for g, st in zip(kv.value.groups, cache.layers[li].v_groups):
        h = x_rows @ g.a.data
        for row in h:
            st.append(row)


MEDIUM_CASES = [
    # name, d, n, dh, s_k, ranks_k, s_v, ranks_v, T, bits, base, x_scale, hadamard
    ("med_g2_nonuniform", 512, 4, 128, 2, [64, 40], 2, [48, 64], 300, 16, 10000.0, 2.0, False),
    ("med_g4_r256", 512, 4, 128, 4, [256], 4, [256], 257, 16, 10000.0, 2.0, False),
    ("med_g2_b4_had", 512, 4, 128, 2, [64, 64], 2, [64, 64], 300, 4, 10000.0, 2.0, True),
    ("med_g2_b2_had", 512, 4, 128, 2, [64, 32], 2, [32, 64], 200, 2, 10000.0, 2.0, True),
    ("med_g2_b16_4", 512, 4, 128, 2, [64, 64], 2, [96, 64], 250, (16, 4), 1e6, 2.0, True),
    ("med_mixed_gran", 512, 4, 128, 1, [32, 16, 24, 8], 4, [128], 130, 16, 10000.0, 2.0, False),
    ("med_b8_b3", 256, 2, 128, 2, [48], 1, [40, 24], 140, (8, 3), 10000.0, 2.0, True),
    # the paper's Palu-50% latency preset: kept K 25% / V 75%
    ("med_preset_k128_v384", 512, 4, 128, 4, [128], 4, [384], 300, 16, 10000.0, 2.0, False),
    ("med_preset_b4v", 512, 4, 128, 4, [128], 4, [384], 260, (16, 4), 10000.0, 2.0, True),
]


def gen_medium():
    out = {}
    names = []
    for ci, (name, d, n, dh, s_k, rk, s_v, rv, T, bits, base, xs, had) in enumerate(MEDIUM_CASES):
        seed = 5000 + 100 * ci
        config = AttentionConfig(d, n, dh, layers=1, rope=True, rope_base=base)
        lw, kv = _synth_ref_layer(d, n, dh, s_k, rk, s_v, rv, seed, had)
        weights = ModelWeights(layers=(lw,))
        fused = build_fused(weights, [kv], config)
        cache = LatentKVCache([kv], config, bits=bits)
        x_rows = random_matrix(T, d, seed=seed + 77).data * xs
        _direct_fill(cache, kv, 0, x_rows)
        cache.t = T
        x_t = random_matrix(1, d, seed=seed + 78).data[0] * xs
        y = palu_decode_step_rope(weights, fused, cache, x_t)
        y2 = palu_decode_step_rope(weights, fused, cache, y)  # a second step, fed back
        p = f"c{ci}_"
        names.append(name)
        out[p + "meta"] = np.array([d, n, dh, s_k, s_v, T, base, xs, seed, had], dtype=np.float64)
        out[p + "ranks_k"] = np.array(rk)
        out[p + "ranks_v"] = np.array(rv)
        out[p + "bits"] = np.array(bits if isinstance(bits, tuple) else (bits, bits))
        out[p + "out1"] = y
        out[p + "out2"] = y2
    out["names"] = np.array(names)
    _save("medium_step.npz", **out)


def gen_c1():
    """BASELINE config C1: one Llama-2-7B-shaped layer, gs 4, r 256, T=2048."""
    d, n, dh, s, r, T = 4096, 32, 128, 4, 256, 2048
    out = {}
    for tag, bits, had in (("b16", 16, False), ("b4had", 4, True)):
        seed = 7000
        t0 = time.time()
        config = AttentionConfig(d, n, dh, layers=1, rope=True, rope_base=10000.0)
        lw, kv = _synth_ref_layer(d, n, dh, s, [r] * 8, s, [r] * 8, seed, had)
        weights = ModelWeights(layers=(lw,))
        fused = build_fused(weights, [kv], config)
        cache = LatentKVCache([kv], config, bits=bits)
        x_rows = random_matrix(T, d, seed=seed + 77).data
        _direct_fill(cache, kv, 0, x_rows)
        cache.t = T
        x_t = random_matrix(1, d, seed=seed + 78).data[0]
        y = palu_decode_step_rope(weights, fused, cache, x_t)
        out[f"{tag}_out1"] = y
        print(f"c1 {tag}: {time.time() - t0:.1f}s")
    out["meta"] = np.array([d, n, dh, s, r, T, 10000.0, 1.0, 7000], dtype=np.float64)
    _save("c1_step.npz", **out)


GQA_CASES = [
    # name, d, n_q, n_kv, dh, rank_k, rank_v, T, bits, hadamard, base
    ("gqa_q8_kv2_r64", 1024, 8, 2, 128, 64, 64, 300, 16, False, 1e6),
    ("gqa_q8_kv2_r64_k16v4_had", 1024, 8, 2, 128, 64, 64, 260, (16, 4), True, 1e6),
    ("gqa_q8_kv2_r32_b4_had", 1024, 8, 2, 128, 32, 64, 200, 4, True, 1e6),
]


def gen_gqa():
    """BASELINE configs[3] semantics (Mistral-7B GQA), scaled down: the
    MHA-equivalent replicated-B layer decoded by the
    UNMODIFIED reference, checked against an independent KV-head restatement
    (oracle.gqa_decode_step_rope) before it is stored."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from oracle import palu_oracle as po
    out, names = {}, []
    for ci, (name, d, nq, nkv, dh, rk, rv, T, bits, had, base) in enumerate(GQA_CASES):
        seed = 8100 + 100 * ci
        L = po.synth_gqa_layer(d, nq, nkv, dh, rk, rv, seed, hadamard_fused=had)
        s = nq // nkv
        config = AttentionConfig(d, nq, dh, layers=1, rope=True, rope_base=base)
        z = Matrix(np.zeros((d, d)))
        lw = LayerWeights(wq=Matrix(L.wq), wk=z, wv=z, wo=Matrix(L.wo))
        gran = Granularity.group_head(s)
        key = DecomposedLayer(gran, tuple(GroupFactors(Matrix(a), Matrix(b), a.shape[1])
                                          for a, b in zip(L.ak, L.bk)), d, dh, nq)
        value = DecomposedLayer(gran, tuple(GroupFactors(Matrix(a), Matrix(b), a.shape[1])
                                            for a, b in zip(L.av, L.bv)), d, dh, nq)
        kv = LayerKV(key=key, value=value)
        weights = ModelWeights(layers=(lw,))
        fused = build_fused(weights, [kv], config)
        cache = LatentKVCache([kv], config, bits=bits)
        x_rows = random_matrix(T, d, seed=seed + 77).data
        _direct_fill(cache, kv, 0, x_rows)
        cache.t = T
        x_t = random_matrix(1, d, seed=seed + 78).data[0]
        y = palu_decode_step_rope(weights, fused, cache, x_t)
        indep = po.gqa_decode_step_rope(L, cache.hk(0), cache.hv(0), x_t, nq, nkv, dh, base, T)
        err = float(np.linalg.norm(indep - y) / np.linalg.norm(y))
        assert err < 1e-12, (name, err)
        p = f"c{ci}_"
        names.append(name)
        out[p + "meta"] = np.array([d, nq, nkv, dh, rk, rv, T, had, base, seed], dtype=np.float64)
        out[p + "bits"] = np.array(bits if isinstance(bits, tuple) else (bits, bits))
        out[p + "out1"] = y
        out[p + "indep_rel_err"] = np.array([err])
        print(f"gqa {name}: reference vs independent GQA restatement rel-L2 {err:.2e}")
    out["names"] = np.array(names)
    _save("gqa_step.npz", **out)


def gen_plan():
    """a layer- and group-varying (r_k, r_v) plan from the
    reference's own ranks.allocate (K budget 25 %, V 75 %: the paper's
    K-light / V-heavy split) on deterministic synthetic Fisher scores, and a
    two-layer Llama-2-7B-shaped decode step of the unmodified reference with
    those ranks."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2407_21118_b200 import rank_plan as RP
    from palu.ranks import FisherScore, allocate
    d, n, dh, s, layers, T, G = 4096, 32, 128, 4, 2, 1024, 8
    out = {}
    plans = {}
    for side, rate in (("k", 0.25), ("v", 0.75)):
        mine = RP.synthetic_fisher_scores(layers, G, side)
        ref = allocate([FisherScore(x.target_id, x.score) for x in mine], [s * dh] * layers * G, d, rate,
                       min_rank=8)
        plans[side] = [[ref.rank_for(RP.target_id(li, side, g)) for g in range(G)] for li in range(layers)]
        out[f"scores_{side}"] = np.array([x.score for x in mine])
        out[f"ranks_{side}"] = np.array(plans[side])
    config = AttentionConfig(d, n, dh, layers=layers, rope=True, rope_base=10000.0)
    lws, kvs = [], []
    for li in range(layers):
        lw, kv = _synth_ref_layer(d, n, dh, s, plans["k"][li], s, plans["v"][li], 9100 + 101 * li)
        lws.append(lw)
        kvs.append(kv)
    weights = ModelWeights(layers=tuple(lws))
    fused = build_fused(weights, kvs, config)
    cache = LatentKVCache(kvs, config, bits=16)
    for li in range(layers):
        _direct_fill(cache, kvs[li], li, random_matrix(T, d, seed=9100 + 101 * li + 77).data)
    cache.t = T
    x_t = random_matrix(1, d, seed=9178).data[0]
    t0 = time.time()
    out["out1"] = palu_decode_step_rope(weights, fused, cache, x_t)
    out["meta"] = np.array([d, n, dh, s, layers, T, 9100], dtype=np.float64)
    print(f"plan: K ranks {plans['k']} V ranks {plans['v']} ({time.time() - t0:.1f}s)")
    _save("plan_step.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "quant", "small", "medium", "c1", "gqa", "plan"]
    for w in which:
        globals()[f"gen_{w}"]()
