"""Long-context parity harness: the GPU decode step at the benchmarked shape
(Llama-2-7B layers, gs 4, 16K-128K cached tokens) against the fp64 oracle.

TEST INFRASTRUCTURE ONLY (imports the oracle).  Both sides see the same
inputs: seeded weights/factors (random_matrix, core.py:331-356, generated on
the GPU bit-exactly), cache rows H = X @ A_g computed ONCE in fp64 and
handed to both the GPU cache (stored as bf16 or quantised by the device
quantiser) and the oracle's group stores (kept in fp64, or quantised by the
oracle's own restatement of quant.py:87-99 -- the codes then agree exactly,
which the harness checks).  The newest token's latents come from each side's
own append (GPU: bf16 weights, fp32 GEMV).
"""

from __future__ import annotations

import json
import math
import os
import time

import numpy as np

from oracle import palu_oracle as po


def log_result(rec: dict) -> None:
    """Append one measured error record (PALU_PARITY_LOG=<path>, jsonl)."""
    path = os.environ.get("PALU_PARITY_LOG")
    if path:
        os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def make_layers(n_layers, d=4096, n=32, dh=128, s=4, rk=256, rv=256, hadamard=False, seed=500,
                gqa_kv=0):
    """OracleLayer list with po.synth_layer's seeds/scales, via the GPU generator.
    gqa_kv > 0: po.synth_gqa_layer's replicated-B layers (n_kv = gqa_kv)."""
    from paper_2407_21118_b200.harness import random_matrix_gpu
    if gqa_kv:
        return [po.synth_gqa_layer(d, n, gqa_kv, dh, rk, rv, seed + 101 * li, hadamard_fused=hadamard)
                for li in range(n_layers)]

    def rm(r, c, sd):
        return random_matrix_gpu(r, c, sd).cpu().numpy()

    sq = 1.0 / math.sqrt(d)
    G = n // s
    rks = [rk] * G if isinstance(rk, int) else list(rk)
    rvs = [rv] * G if isinstance(rv, int) else list(rv)
    layers = []
    for li in range(n_layers):
        sd = seed + 101 * li
        ak, bk, av, bv = [], [], [], []
        for g, r in enumerate(rks):
            a, b = rm(d, r, sd + 1000 + 2 * g) * sq, rm(r, s * dh, sd + 1001 + 2 * g) / math.sqrt(r)
            if hadamard:
                a, b = po.fuse_hadamard(a, b)
            ak.append(a)
            bk.append(b)
        for g, r in enumerate(rvs):
            a, b = rm(d, r, sd + 2000 + 2 * g) * sq, rm(r, s * dh, sd + 2001 + 2 * g) / math.sqrt(r)
            if hadamard:
                a, b = po.fuse_hadamard(a, b)
            av.append(a)
            bv.append(b)
        layers.append(po.OracleLayer(wq=rm(d, d, sd) * sq, wo=rm(d, d, sd + 3) * sq,
                                     ak=ak, bk=bk, av=av, bv=bv, s_k=s, s_v=s))
    return layers


def to_package(layers, n, dh, rope, base):
    from paper_2407_21118_b200 import model as M
    d = n * dh
    z = np.broadcast_to(np.float64(0.0), (d, d))
    wl, dl = [], []
    for L in layers:
        wl.append(M.LayerWeights(wq=L.wq, wk=z, wv=z, wo=L.wo))
        key = M.DecomposedLayer(M.Granularity.group_head(L.s_k),
                                tuple(M.GroupFactors(a, b, a.shape[1]) for a, b in zip(L.ak, L.bk)),
                                d, dh, n)
        val = M.DecomposedLayer(M.Granularity.group_head(L.s_v),
                                tuple(M.GroupFactors(a, b, a.shape[1]) for a, b in zip(L.av, L.bv)),
                                d, dh, n)
        dl.append(M.LayerKV(key=key, value=val))
    cfg = M.AttentionConfig(d, n, dh, layers=len(layers), rope=rope, rope_base=base)
    return M.ModelWeights(layers=tuple(wl)), dl, cfg


def fill_both(cache, oc, layers, T, seed=900, chunk=8192):
    """H = X @ A_g (fp64, on the GPU) into the GPU cache and the oracle stores.

    Returns the number of (row, column) code mismatches between the GPU's
    stored codes and the oracle's (quantised sides; must be 0)."""
    import torch
    from paper_2407_21118_b200.harness import _fill_side, random_matrix_gpu
    dev = cache.device
    mism = 0
    for li, L in enumerate(layers):
        K, V = cache._stores[li]
        a_k = [torch.from_numpy(a).to(dev) for a in L.ak]
        a_v = [torch.from_numpy(a).to(dev) for a in L.av]
        for c0 in range(0, T, chunk):
            rows = min(chunk, T - c0)
            X = random_matrix_gpu(rows, L.wq.shape[0], seed + 17 * li, row0=c0, device=dev)
            for side, A, stores in ((K, a_k, oc.k_stores[li]), (V, a_v, oc.v_stores[li])):
                for g, a in enumerate(A):
                    h = X @ a
                    _fill_side(side, g, 0, c0, h)
                    stores[g].extend(h.cpu().numpy())
        torch.cuda.synchronize()
        # quantised sides: the device quantiser and the oracle agree bit for bit
        for side, stores in ((K, oc.k_stores[li]), (V, oc.v_stores[li])):
            if side.bits == po.FP_BITS:
                continue
            for g in (0, side.G - 1):
                q = side.quantized(0, g, T)
                mism += int(np.count_nonzero(q.codes != stores[g].codes[:T]))
                mism += int(np.count_nonzero(q.zero_points != stores[g].zps[:T]))
                mism += int(np.count_nonzero(q.scales != stores[g].scales[:T]))
    return mism


def run_case(P, *, T, n_layers=2, rk=256, rv=256, bits=16, hadamard=False, rope=True,
             base=10000.0, seed=500, steps=1, name="", gqa_kv=0):
    """One (or more) GPU decode steps vs the oracle; returns a record dict."""
    from paper_2407_21118_b200.harness import set_cache_t
    n, dh, s = 32, 128, 4
    layers = make_layers(n_layers, rk=rk, rv=rv, hadamard=hadamard, seed=seed, gqa_kv=gqa_kv)
    w, dec, cfg = to_package(layers, n, dh, rope, base)
    fused = P.build_fused(w, dec, cfg, dtype="bfloat16")
    cache = P.LatentKVCache(dec, cfg, bits, dtype="bfloat16", capacity=T + 8 * steps)
    oc = po.OracleCache(layers, bits=bits)
    mism = fill_both(cache, oc, layers, T, seed=seed + 400)
    set_cache_t(cache, T)
    oc.t = T
    wo = [po.build_wo_fused(L, n, dh) for L in layers]
    wq = None if rope else [po.build_wq_fused(L, n, dh) for L in layers]
    from paper_2407_21118_b200.harness import random_matrix_gpu
    x = random_matrix_gpu(1, n * dh, seed + 77).cpu().numpy()[0]
    xg, xo, errs, t_or = x, x, [], 0.0
    for _ in range(steps):
        if rope:
            yg = P.palu_decode_step_rope(w, fused, cache, xg)
            t0 = time.perf_counter()
            yo = po.decode_step_rope(layers, wo, oc, xo, n, dh, base)
        else:
            yg = P.palu_decode_step_norope(w, fused, cache, xg)
            t0 = time.perf_counter()
            yo = po.decode_step_norope(layers, wq, wo, oc, xo, n, dh)
        t_or += time.perf_counter() - t0
        errs.append(float(np.linalg.norm(yg - yo) / np.linalg.norm(yo)))
        xg, xo = yg, yo
    sess = cache._session
    rec = dict(case=name, T=T, layers=n_layers, rank_k=rk, rank_v=rv, kv_heads=gqa_kv or None,
               bits=list(bits) if isinstance(bits, tuple) else bits, hadamard=hadamard, rope=rope,
               rope_base=base, rel_l2=errs, code_mismatches=mism,
               score_kernel=("tcgen05_rep" if any(x is not None for x in getattr(sess, "rep_bkt", [])) else
                             "tcgen05" if any(sess.tc_layers) else
                             "latent_score_tc" if any(sess.ls_tc_layers) else "simt"),
               value_kernel="tcgen05" if any(sess.value_tc_layers) else "simt",
               oracle_s_per_step=round(t_or / steps, 2))
    del cache, fused, oc
    return rec
