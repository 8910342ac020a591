"""Diagnostics: per-CTA timeline of one packed-V value launch (value_q_kernel).

    PALU_FUSED_TRACE=1 python tools/vq_trace.py [--rank-k 128 --rank-v 384 --bits 16,4]

Prints, for a few CTAs, the per-block TMA issue / conversion times and the
per-sub-block group A / MMA / group B times relative to kernel entry (us).
Not a bench.
"""

import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PALU_FUSED_TRACE", "1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--rank-k", type=int, default=128)
    ap.add_argument("--rank-v", type=int, default=384)
    ap.add_argument("--bits", default="16,4")
    ap.add_argument("--ctas", default="0,1,73,147")
    a = ap.parse_args()
    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    _lib.load()
    bl = [int(x) for x in a.bits.split(",")]
    w, f, c = synthetic_engine(layers=1, context=a.context, extra=64, rank_k=a.rank_k,
                               rank_v=a.rank_v, bits=bl[0] if len(bl) == 1 else tuple(bl))
    s = _session(f, c)
    s.x.normal_(0, 0.5)
    for _ in range(3):
        s.launch_step()
        torch.cuda.synchronize()
    prof = s.profile_step()
    print({k: [round(x * 1e3, 1) for x in v] for k, v in prof.items()}, "us")
    buf = np.zeros((1024, 512), dtype=np.uint64)
    n = _lib.call("palu_fused_trace", buf.ctypes.data_as(C.c_void_p), 1024)
    tr = buf[:n].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    ends = (tr[:, 1] - t0) / 1e3
    starts = (tr[:, 0] - t0) / 1e3
    print(f"CTAs {n}: start spread {starts.min():.1f}..{starts.max():.1f} us, "
          f"end spread {ends.min():.1f}..{ends.max():.1f} us")
    busy = ends[tr[:, 3] > 2000000]
    print("  CTA end us p10/p50/p90/max", np.percentile(busy, [10, 50, 90, 100]).round(1),
          " even-SM CTAs median", np.median(ends[0::2]).round(1), "odd", np.median(ends[1::2]).round(1))

    GHZ = 1.9  # slots >= 3 hold SM clock64 values; slot 2 = clock64 at entry

    def row(c, lo, cnt):
        v = tr[c, lo:lo + cnt]
        return [round((x - tr[c, 2]) / GHZ / 1e3, 2) for x in v if x > 0]

    for c in [int(x) for x in a.ctas.split(",") if int(x) < n]:
        print(f"--- CTA {c}: {(tr[c, 1] - tr[c, 0]) / 1e3:.1f} us")
        print("  TMA issue  ", row(c, 8, 48))
        print("  conv start ", row(c, 56, 48))
        print("  conv done  ", row(c, 104, 48))
        print("  A start    ", row(c, 184, 16))
        print("  A pre-bar  ", row(c, 300, 16))
        print("  A post-bar ", row(c, 316, 16))
        print("  A dempty ok", row(c, 216, 16))
        print("  A digits ok", row(c, 332, 16))
        print("  A pfull    ", row(c, 200, 16))
        print("  MMA start  ", row(c, 152, 16))
        print("  MMA commit ", row(c, 168, 16))
        print("  B dfull    ", row(c, 232, 16))



if __name__ == "__main__":
    main()
