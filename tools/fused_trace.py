"""Diagnostics: per-CTA timeline of one fused score+softmax+value launch.

    PALU_FUSED_TRACE=1 python tools/fused_trace.py [--context 65536] [--rank-k 256 --rank-v 256]

Prints role start/end spread, score-item throughput and, per value CTA, how
long it waited for readiness versus how long it streamed.  Not a bench.
"""

import argparse
import ctypes as C
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PALU_FUSED_TRACE", "1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--rank-k", type=int, default=256)
    ap.add_argument("--rank-v", type=int, default=256)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--score-kernel", default="fused", help="fused | tcgen05 (standalone value kernel)")
    ap.add_argument("--bits", default="16")
    a = ap.parse_args()
    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    _lib.load()
    bl = [int(x) for x in a.bits.split(",")]
    w, f, c = synthetic_engine(layers=1, batch=a.batch, context=a.context, extra=64,
                               rank_k=a.rank_k, rank_v=a.rank_v,
                               bits=bl[0] if len(bl) == 1 else tuple(bl))
    s = _session(f, c, score_kernel=a.score_kernel)
    s.x.normal_(0, 0.5)
    for _ in range(3):
        s.launch_step()
        torch.cuda.synchronize()
    prof = s.profile_step()
    print({k: [round(x * 1e3, 1) for x in v] for k, v in prof.items()}, "us")
    print("max co-resident 2-CTA clusters:", _lib.call("palu_fused_max_clusters", 230000))
    buf = np.zeros((1024, 512), dtype=np.uint64)
    n = _lib.call("palu_fused_trace", buf.ctypes.data_as(C.c_void_p), 1024)
    tr = buf[:n].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    score = [i for i in range(n) if 0 < tr[i, 3] < 1000000]
    value = [i for i in range(n) if tr[i, 3] >= 1000000]
    us = lambda x: (x - t0) / 1e3
    print(f"CTAs {n}: score {len(score)} value {len(value)}")
    for name, ids in (("score", score), ("value", value)):
        if not ids:
            continue
        st = [us(tr[i, 0]) for i in ids]
        en = [us(tr[i, 1]) for i in ids]
        print(f"{name}: start {min(st):.1f}..{max(st):.1f} us, end {min(en):.1f}.."
              f"{max(en):.1f} (median {statistics.median(en):.1f})")
    if score:
        i = score[0]
        cnt = int(tr[i, 3])
        ev = [us(x) for x in tr[i, 4:4 + cnt]]
        print(f"score CTA {i} (sm {tr[i, 2]}): {cnt} items, done at", [round(x, 1) for x in ev[:8]],
              "...", [round(x, 1) for x in ev[-3:]])
    if value:
        ph = np.array([[us(tr[i, c]) for c in (495, 496, 497, 498)] for i in value])
        print("value setup done / first TMA / first stage landed / ring wrapped (median us):",
              np.median(ph, axis=0).round(2), "vs end", round(float(np.median([us(tr[i, 1]) for i in value])), 1))
        ev = np.array([us(tr[i, 1]) for i in value])
        sm = np.array([tr[i, 2] for i in value])
        print("end by SM parity: even", np.median(ev[sm % 2 == 0]).round(1), "odd", np.median(ev[sm % 2 == 1]).round(1))
    merges = [(us(tr[i, 500]), us(tr[i, 501])) for i in value if tr[i, 500] > 0]
    print("merges (start, end) us:", [(round(a_, 1), round(b_, 1)) for a_, b_ in merges])
    for i in value[:6] + value[-2:]:
        k = int((tr[i, 4::5][:59] > 0).sum())
        if k == 0:
            continue
        rd = [us(tr[i, 4 + 5 * j]) for j in range(k)]
        dn = [us(tr[i, 5 + 5 * j]) for j in range(k)]
        ph = np.array([[tr[i, 6 + 5 * j] - tr[i, 4 + 5 * j], tr[i, 5 + 5 * j] - tr[i, 6 + 5 * j],
                        (tr[i, 4 + 5 * (j + 1)] - tr[i, 5 + 5 * j]) if j + 1 < k else 0]
                       for j in range(k)]) / 1e3
        print(f"  group A phases (max, P, gap to next) median us: {np.median(ph, axis=0).round(2)}")
        stream = sum(dn[j] - max(rd[j], dn[j - 1] if j else us(tr[i, 0])) for j in range(k))
        if tr[i, 500] > 0:
            print(f"  merge {us(tr[i, 500]):.1f} -> {us(tr[i, 501]):.1f} us")
        print(f"value CTA {i} (sm {tr[i, 2]}): {k} chunks, start {us(tr[i, 0]):.1f} end "
              f"{us(tr[i, 1]):.1f}; busy {stream:.1f} us; first ready {rd[0]:.1f}, "
              f"per-chunk (ready->done):", [(round(r, 1), round(d, 1)) for r, d in zip(rd[:6], dn[:6])])



    conv = [i for i in value if tr[i, 300] > 0]
    if conv:
        i = conv[0]
        k = int((tr[i, 300:500:3] > 0).sum())
        st = tr[i, 300:300 + 3 * k].reshape(k, 3)
        w_raw = (st[:, 1] - st[:, 0]) / 1e3
        w_empty = (st[:, 2] - st[:, 1]) / 1e3
        conv_t = (st[1:, 0] - st[:-1, 2]) / 1e3
        print(f"converter CTA {i}: {k} stages; wait raw-ring p50 {np.median(w_raw):.2f} us, "
              f"wait empty stage p50 {np.median(w_empty):.2f} us, convert p50 {np.median(conv_t):.2f} us")


if __name__ == "__main__":
    main()
