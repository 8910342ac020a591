"""Diagnostics: per-CTA timeline of one rope-off int8-pipe latent-score launch
(latent_score_q_kernel).  Needs the diagnostic build:

    python -m paper_2407_21118_b200.build --out abtmp/diag -DPALU_DIAG -DPALU_TRACE
    PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_LSQ_TRACE=1 python tools/lsq_trace.py [--bits 4]

Prints per tile (µs from CTA entry, SM clock): producer issue, converter
start/done, MMA issue, epilogue wake/done.  Not a bench.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PALU_LSQ_TRACE", "1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--rank-k", type=int, default=256)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--ctas", default="0,73")
    ap.add_argument("--ghz", type=float, default=1.9)
    a = ap.parse_args()
    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    _lib.load()
    w, f, c = synthetic_engine(layers=1, context=a.context, extra=64, rank_k=a.rank_k, rank_v=a.rank_k,
                               bits=a.bits, rope=False)
    s = _session(f, c)
    s.x.normal_(0, 0.5)
    for _ in range(3):
        s.launch_step()
        torch.cuda.synchronize()
    os.environ["PALU_VALUE_MERGE"] = "kernel"
    prof = s.profile_step()
    print({k: [round(x * 1e3, 1) for x in v] for k, v in prof.items()}, "us")
    buf = np.zeros((1024, 512), dtype=np.uint64)
    n = _lib.call("palu_fused_trace", buf.ctypes.data_as(C.c_void_p), 1024)
    tr = buf[:n].astype(np.int64)
    t0 = tr[:, 4][tr[:, 4] > 0].min()
    ent = (tr[:, 4] - t0) / 1e3
    dep = (tr[:, 5] - t0) / 1e3
    print(f"kernel entry (min/max) {ent.min():.1f}/{ent.max():.1f} us, after griddepcontrol.wait {dep.min():.1f}/{dep.max():.1f}, setup done 0..{((tr[:, 0] - t0) / 1e3).max():.1f}")
    print(f"CTAs {n}: end spread {((tr[:, 1] - t0) / 1e3).min():.1f}..{((tr[:, 1] - t0) / 1e3).max():.1f} us")
    for cta in [int(x) for x in a.ctas.split(",")]:
        k = int(tr[cta, 3])
        rel = lambda base: [round(float(tr[cta, base + i] - tr[cta, 2]) / a.ghz / 1e3, 2) for i in range(min(k, 60))]
        print(f"--- CTA {cta}: {k} tiles, {(tr[cta, 1] - tr[cta, 0]) / 1e3:.1f} us")
        for name, base in (("produce", 8), ("conv start", 68), ("conv done", 128), ("MMA issue", 188),
                           ("epi wake", 248), ("epi done", 308)):
            print(f"  {name:10s}", rel(base)[:30])


if __name__ == "__main__":
    main()
