"""Rebuild oracle inputs from the committed golden fixtures (test helper)."""

from __future__ import annotations

import math

import numpy as np

from oracle import palu_oracle as po


def small_case(g, ci):
    """Layers, tokens and expected outputs of SMALL_CASES[ci] (make_golden.py)."""
    p = f"c{ci}_"
    rope, layers, s_k, s_v, rk, rv, T, had, base = g[p + "meta"]
    layers, s_k, s_v, T = int(layers), int(s_k), int(s_v), int(T)
    n, dh = 4, 4
    out = []
    for li in range(layers):
        gk, gv = n // s_k, n // s_v
        L = po.OracleLayer(
            wq=g[p + f"L{li}_wq"], wo=g[p + f"L{li}_wo"],
            ak=[g[p + f"L{li}_ak{j}"] for j in range(gk)],
            bk=[g[p + f"L{li}_bk{j}"] for j in range(gk)],
            av=[g[p + f"L{li}_av{j}"] for j in range(gv)],
            bv=[g[p + f"L{li}_bv{j}"] for j in range(gv)],
            s_k=s_k, s_v=s_v, wk=g[p + f"L{li}_wk"], wv=g[p + f"L{li}_wv"])
        out.append(L)
    bits = tuple(int(b) for b in g[p + "bits"])
    tile = int(g[p + "tile"][0])
    return dict(layers=out, tokens=g[p + "tokens"], outputs=g[p + "outputs"], rope=bool(rope),
                bits=bits, tile=None if tile < 0 else tile, n=n, dh=dh, base=float(base),
                T=T, had=bool(had))


def medium_case(g, ci):
    p = f"c{ci}_"
    d, n, dh, s_k, s_v, T, base, xs, seed, had = g[p + "meta"]
    d, n, dh, s_k, s_v, T, seed = (int(v) for v in (d, n, dh, s_k, s_v, T, seed))
    rk = [int(r) for r in g[p + "ranks_k"]]
    rv = [int(r) for r in g[p + "ranks_v"]]
    L = po.synth_layer(d, n, dh, s_k, rk, s_v, rv, seed, hadamard_fused=bool(had))
    x_rows = po.random_matrix(T, d, seed + 77) * xs
    x_t = po.random_matrix(1, d, seed + 78)[0] * xs
    bits = tuple(int(b) for b in g[p + "bits"])
    return dict(layer=L, x_rows=x_rows, x_t=x_t, bits=bits, base=float(base), n=n, dh=dh, d=d,
                T=T, out1=g[p + "out1"], out2=g[p + "out2"])


def c1_case(g, tag):
    d, n, dh, s, r, T, base, xs, seed = g["meta"]
    d, n, dh, s, r, T, seed = (int(v) for v in (d, n, dh, s, r, T, seed))
    had = tag == "b4had"
    L = po.synth_layer(d, n, dh, s, r, s, r, seed, hadamard_fused=had)
    x_rows = po.random_matrix(T, d, seed + 77)
    x_t = po.random_matrix(1, d, seed + 78)[0]
    bits = (4, 4) if tag == "b4had" else (16, 16)
    return dict(layer=L, x_rows=x_rows, x_t=x_t, bits=bits, base=float(base), n=n, dh=dh, d=d,
                T=T, out1=g[f"{tag}_out1"])


def oracle_step_from_fill(case, steps=1):
    """Direct-filled oracle cache, then ``steps`` decode steps (fed back)."""
    L = case["layer"]
    cache = po.OracleCache([L], bits=case["bits"])
    cache.fill_direct(0, case["x_rows"])
    cache.t = case["T"]
    wo_f = [po.build_wo_fused(L, case["n"], case["dh"])]
    x = case["x_t"]
    outs = []
    for _ in range(steps):
        x = po.decode_step_rope([L], wo_f, cache, x, case["n"], case["dh"], case["base"])
        outs.append(x)
    return outs, cache


def gqa_case(g, ci):
    """GQA_CASES[ci] (make_golden.py): the replicated-B layer from its seed."""
    p = f"c{ci}_"
    d, nq, nkv, dh, rk, rv, T, had, base, seed = g[p + "meta"]
    d, nq, nkv, dh, rk, rv, T, seed = (int(v) for v in (d, nq, nkv, dh, rk, rv, T, seed))
    L = po.synth_gqa_layer(d, nq, nkv, dh, rk, rv, seed, hadamard_fused=bool(had))
    x_rows = po.random_matrix(T, d, seed + 77)
    x_t = po.random_matrix(1, d, seed + 78)[0]
    bits = tuple(int(b) for b in g[p + "bits"])
    return dict(layer=L, x_rows=x_rows, x_t=x_t, bits=bits, base=float(base), n=nq, n_kv=nkv,
                dh=dh, d=d, T=T, out1=g[p + "out1"])


def plan_case(g):
    """gen_plan (make_golden.py): two layers with the reference plan's ranks."""
    d, n, dh, s, layers, T, seed = (int(v) for v in g["meta"])
    rk, rv = g["ranks_k"], g["ranks_v"]
    Ls = [po.synth_layer(d, n, dh, s, [int(r) for r in rk[li]], s, [int(r) for r in rv[li]],
                         seed + 101 * li) for li in range(layers)]
    x_rows = [po.random_matrix(T, d, seed + 101 * li + 77) for li in range(layers)]
    x_t = po.random_matrix(1, d, 9178)[0]
    return dict(layers=Ls, x_rows=x_rows, x_t=x_t, n=n, dh=dh, d=d, T=T, out1=g["out1"],
                ranks_k=rk, ranks_v=rv)

