"""Golden `.palu` latent containers from the UNMODIFIED reference (read-only import).

    python tests/golden/make_container_golden.py

For each bit width it quantises fixed fp32-representable latents with the
reference's quantize_rows (quant.py:87-99), packs them with pack_codes
(quant.py:156-169) and writes them with write_container (container.py:92-124)
using the tensor naming of the pipeline's latent export (pipeline.py:513-531).
The latents and the exact container bytes go to container.npz; the GPU test
appends the same latents through the CUDA quantiser and exports the cache
with paper_2407_21118_b200.container.export_latents, which must reproduce the
bytes.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from palu.container import PackedTensor, write_container  # noqa: E402
from palu.quant import QuantParams, pack_codes, quantize_rows  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
T = 45
RANKS = {"k": (24, 17), "v": (31, 8)}  # per group, two groups per side
LAYERS = 2
META = {"model": {"name": "golden", "layers": LAYERS}, "seed": 0}


def main():
    rng = np.random.default_rng(2407)
    out = {}
    lat = {}
    for li in range(LAYERS):
        for proj in ("k", "v"):
            for g, r in enumerate(RANKS[proj]):
                x = (rng.standard_normal((T, r)) * (0.5 + g)).astype(np.float32)
                x[3] = x[3, 0]  # a constant row (range floor)
                lat[f"layer{li}.{proj}.g{g}"] = x
                out[f"lat.layer{li}.{proj}.g{g}"] = x
    for bits in (2, 3, 4, 8):
        tensors = {}
        for name, x in lat.items():
            q = quantize_rows(x.astype(np.float64), QuantParams(bits))
            tensors[f"{name}.codes"] = PackedTensor(data=pack_codes(q.codes, q.bits),
                                                    shape=q.codes.shape, bits=q.bits)
            tensors[f"{name}.scales"] = q.scales
            tensors[f"{name}.zero_points"] = q.zero_points.astype(np.float64)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "latents.palu")
            write_container(path, tensors, meta=dict(META, bits=bits))
            blob = open(path, "rb").read()
        out[f"palu_b{bits}"] = np.frombuffer(blob, dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "container.npz"), **out)
    print("wrote", os.path.join(HERE, "container.npz"), {k: v.shape for k, v in out.items() if k.startswith("palu")})


if __name__ == "__main__":
    main()
