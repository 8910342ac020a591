import ctypes as C, os, sys, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["PALU_FUSED_TRACE"] = "1"
import torch
from paper_2407_21118_b200 import _lib
from paper_2407_21118_b200.attention import _session
from paper_2407_21118_b200.harness import synthetic_engine
_lib.load()
w, f, c = synthetic_engine(layers=1, context=65536, extra=64)
s = _session(f, c, score_kernel="tcgen05")
s.x.normal_(0, 0.5)
for _ in range(3):
    s.launch_step(); torch.cuda.synchronize()
for rep in range(2):
    s.profile_step()
    buf = np.zeros((1024, 512), dtype=np.uint64)
    n = _lib.call("palu_fused_trace", buf.ctypes.data_as(C.c_void_p), 1024)
    tr = buf[:n].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    end = (tr[:, 1] - t0) / 1e3
    sm = tr[:, 2]
    # count of units per CTA: group A trace slots 4 + 5k (unit starts)
    units = np.array([int((tr[i, 4::5][:59] > 0).sum()) for i in range(n)])
    order = np.argsort(end)
    print("rep", rep, "end p0/p10/p50/p90/max", np.percentile(end, [0, 10, 50, 90, 100]).round(1))
    print(" slowest 12 (cta, sm, units, end):", [(int(i), int(sm[i]), int(units[i]), round(float(end[i]), 1)) for i in order[-12:]])
    print(" fastest 6:", [(int(i), int(sm[i]), int(units[i]), round(float(end[i]), 1)) for i in order[:6]])
    for u in sorted(set(units.tolist())):
        print("  units", u, "count", int((units == u).sum()), "median end", round(float(np.median(end[units == u])), 1))
    # by SM id halves (die?)
    print("  sm<74 median", round(float(np.median(end[sm < 74])), 1), "sm>=74", round(float(np.median(end[sm >= 74])), 1))
