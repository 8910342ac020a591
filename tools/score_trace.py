"""Diagnostics: per-head-pair timeline of the tcgen05 score kernel.

    PALU_SCORE_TRACE=1 python tools/score_trace.py [--rank-k 256]

For leader CTAs: MMA start (after the TMEM slot is free), MMA issue end
(commit), epilogue wake (tfull) and slot release, per head-pair unit.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PALU_SCORE_TRACE", "1")


SU = 8  # trace marks per unit (palu_tc.cu)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--rank-k", type=int, default=256)
    ap.add_argument("--rank-v", type=int, default=256)
    ap.add_argument("--zero-keys", action="store_true", help="zero the key latents (data-power test)")
    ap.add_argument("--bits", type=int, default=16)
    ap.add_argument("--kv-heads", type=int, default=0, help="GQA replicated-B layer (Mistral: 8)")
    a = ap.parse_args()
    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    _lib.load()
    w, f, c = synthetic_engine(layers=1, batch=1, context=a.context, extra=64, rank_k=a.rank_k,
                               rank_v=a.rank_v, bits=a.bits, kv_heads=a.kv_heads,
                               rope_base=1e6 if a.kv_heads else 10000.0)
    if a.zero_keys:
        for K, _ in c._stores:
            K.rows.zero_()
    s = _session(f, c, score_kernel="tcgen05")
    s.x.normal_(0, 0.5)
    for _ in range(3):
        s.launch_step()
    torch.cuda.synchronize()
    prof = s.profile_step()  # the value kernel must not trace: PALU_FUSED_TRACE unset
    print({k: [round(x * 1e3, 1) for x in v] for k, v in prof.items()}, "us")
    buf = np.zeros((1024, 512), dtype=np.uint64)
    n = _lib.call("palu_fused_trace", buf.ctypes.data_as(C.c_void_p), 1024)
    tr = buf[:n].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()  # earliest CTA entry
    ent, setup, end = (tr[:, 0] - t0) / 1e3, (tr[:, 2] - t0) / 1e3, (tr[:, 1] - t0) / 1e3
    pc = lambda x: np.percentile(x, [0, 50, 100]).round(2)
    print(f"CTA entry us min/med/max {pc(ent)}; setup done {pc(setup)}; exit {pc(end)}")

    ld = [i for i in range(0, n, 2) if tr[i, 509] > 0]
    clk = np.array([tr[i, 508] for i in ld], dtype=float)
    ns = np.array([tr[i, 509] for i in ld], dtype=float)
    mm = np.array([tr[i, 510] for i in ld], dtype=float)
    print(f"MMA loop: SM clock {np.median(clk / ns):.3f} GHz, {np.median(clk / mm):.0f} clk and "
          f"{np.median(ns / mm):.1f} ns per pair-MMA (ideal 128 clk)")
    ghz = float(np.median(clk / ns)) if len(ld) else 1.9
    rows = []
    for cta in range(0, n, 2):  # leaders
        u = 0
        while 4 + SU * u + 7 < 508 and tr[cta, 4 + SU * u] > 0:
            ms, me, ew, er, ex, eb, ia, ib = tr[cta, 4 + SU * u:12 + SU * u]
            rows.append((cta, u, ms, me, ew, er, ex, eb, ia, ib))
            u += 1
    r = np.array(rows, dtype=np.int64)
    if not len(r):
        print("no trace")
        return
    # per-unit marks are SM clock64 values (cycles); convert with the measured clock
    mma_issue = (r[:, 3] - r[:, 2]) / ghz / 1e3
    for par in (0, 1):
        sel = r[:, 1] % 2 == par
        print(f"  unit parity {par} (half h={par}): issue span p50 {np.median(mma_issue[sel]):.3f} us")
    epi_lat = (r[:, 4] - r[:, 3]) / ghz / 1e3   # commit -> epilogue wake (other SM's clock: approx.)
    epi_dur = (r[:, 5] - r[:, 4]) / ghz / 1e3   # epilogue work on the slot
    gaps = []
    for cta in np.unique(r[:, 0]):
        rr = r[r[:, 0] == cta]
        gaps += list((rr[1:, 2] - rr[:-1, 3]) / ghz / 1e3)  # MMA idle between units (slot/data)
    pct = lambda x: np.percentile(x, [10, 50, 90]).round(3)
    print(f"units {len(r)}: MMA issue span us p10/50/90 {pct(mma_issue)}")
    print(f"  commit->epilogue wake {pct(epi_lat)}; epilogue on slot {pct(epi_dur)}")
    print(f"  MMA idle between units {pct(np.array(gaps))}")
    xch = (r[:, 6] - r[:, 5]) / ghz / 1e3        # math end -> cross-warp exchange done (jh 0 warp)
    ready = (r[:, 4] - r[:, 7]) / ghz / 1e3      # epilogue ready for the unit -> accumulator complete
    print(f"  exchange wait {pct(xch)}; epilogue waiting for the accumulator {pct(ready)}")
    cta = r[0, 0]
    c0 = tr[cta, 511]
    rr = r[r[:, 0] == cta][:12]
    us = lambda v: round((v - c0) / ghz / 1e3, 2)
    for x in rr:
        print("  unit", x[1], "mma", us(x[2]), "->", us(x[3]), "epi ready", us(x[7]), "wake", us(x[4]),
              "math end", us(x[5]), "exchanged", us(x[6]),
              *(("item start", us(x[8]), "staged", us(x[9])) if x[8] else ()))


if __name__ == "__main__":
    main()
