"""Diagnostics: per-launch device time of each step kernel when the same
launch repeats back to back (CUDA events around N launches; no host gaps, no
profiler).  Compare with ncu's gpu__time_duration and the bench's per-kernel
profile.  Not a bench.

    python tools/kernel_loop.py [--rope off] [--bits 4] [--rank-k 256 --rank-v 256]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--rank-k", type=int, default=256)
    ap.add_argument("--rank-v", type=int, default=256)
    ap.add_argument("--bits", default="16")
    ap.add_argument("--rope", default="on")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    _lib.load()
    bl = [int(x) for x in a.bits.split(",")]
    w, f, c = synthetic_engine(layers=1, context=a.context, extra=64, rank_k=a.rank_k, rank_v=a.rank_v,
                               bits=bl[0] if len(bl) == 1 else tuple(bl), rope=a.rope == "on")
    s = _session(f, c)
    s.x.normal_(0, 0.5)
    for _ in range(3):
        s.launch_step()
    torch.cuda.synchronize()
    calls = []
    orig = _lib.call

    def rec(name, *args):
        calls.append((name, args))
        return orig(name, *args)

    _lib.call = rec
    try:
        s.launch_step()
    finally:
        _lib.call = orig
    torch.cuda.synchronize()
    seen = {}
    for name, args in calls:
        if name == "palu_advance":
            continue
        k = seen.setdefault(name, 0)
        seen[name] = k + 1
        for _ in range(3):
            orig(name, *args)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(a.reps):
            orig(name, *args)
        ev1.record()
        torch.cuda.synchronize()
        print(f"{name}[{k}]: {ev0.elapsed_time(ev1) * 1e3 / a.reps:.1f} us per back-to-back launch")


if __name__ == "__main__":
    main()
