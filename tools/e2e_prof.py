import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch, cProfile, pstats, io
import paper_2407_21118_b200 as P
from paper_2407_21118_b200.harness import synthetic_engine
w, f, c = synthetic_engine(layers=32, batch=1, context=4096, extra=400)
x = np.random.default_rng(0).standard_normal(4096) * 0.5
for _ in range(3): P.palu_decode_step_rope(w, f, c, x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50): P.palu_decode_step_rope(w, f, c, x)
e2e = (time.perf_counter() - t0) / 50 * 1e6
from paper_2407_21118_b200.attention import _session
s = _session(f, c)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(50):
    s.step_device()
torch.cuda.synchronize()
dev = (time.perf_counter() - t0) / 50 * 1e6
print(f"e2e {e2e:.1f} us/step, graph-only {dev:.1f} us/step, host overhead {e2e - dev:.1f} us")
pr = cProfile.Profile(); pr.enable()
for _ in range(20): P.palu_decode_step_rope(w, f, c, x)
pr.disable(); st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(12); print(st.getvalue()[:3000])
