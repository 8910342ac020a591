import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2407_21118_b200 as P
from golden_cases import small_case
import test_gpu_parity as T
g = np.load("tests/golden/small_decode.npz", allow_pickle=True)
ci = list(g["names"]).index("rope_b4_multi_r3")
case = small_case(g, ci)
w, dec, cfg = T._to_types(P, case["layers"], case["n"], case["dh"], True, case["base"])
_, cache = P.palu_decode(w, dec, cfg, case["tokens"], bits=4)
for li in range(len(case["layers"])):
    for side in ("k", "v"):
        grp = cache.layers[li].k_groups if side == "k" else cache.layers[li].v_groups
        for gi, gr in enumerate(grp):
            key = f"c{ci}_L{li}_{side}{gi}_codes"
            if key not in g.files: continue
            q = gr.quantized_latent()
            print(key, q.codes.shape, "mismatch frac", float(np.mean(q.codes != g[key])), "max diff", int(np.max(np.abs(q.codes.astype(int) - g[key].astype(int)))))
