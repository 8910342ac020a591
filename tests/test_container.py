"""`.palu` latent export against containers written by the
unmodified reference (tests/golden/make_container_golden.py)."""

import json
import os

import numpy as np
import pytest

from paper_2407_21118_b200 import container as PC

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "container.npz"))
RANKS = {"k": (24, 17), "v": (31, 8)}
LAYERS, T = 2, 45


def _parse(blob: bytes):
    """Minimal reader (test helper): header dict and raw data section."""
    assert blob[:4] == b"PALU" and blob[4] == 1
    n = int.from_bytes(blob[5:9], "little")
    return json.loads(blob[9:9 + n].decode()), blob[9 + n:]


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_writer_reproduces_reference_bytes(bits):
    """Re-encoding the tensors of a reference container gives the same bytes."""
    blob = GOLDEN[f"palu_b{bits}"].tobytes()
    head, data = _parse(blob)
    tensors = {}
    for e in head["tensors"]:
        raw = data[e["offset"]:e["offset"] + e["byte_len"]]
        if e["dtype"] == "u8-packed":
            tensors[e["name"]] = PC.Packed(raw, e["shape"], e["bits"])
        else:
            tensors[e["name"]] = np.frombuffer(raw, dtype="<f8").reshape(e["shape"])
    assert PC.encode(tensors, head["meta"]) == blob


def test_writer_validation():
    with pytest.raises(Exception):
        PC.Packed(b"\x00", (3, 3), 4)
    with pytest.raises(Exception):
        PC.encode({"x": np.float64(1.0)})


def _cache(bits):
    import torch

    from paper_2407_21118_b200 import model as M
    from paper_2407_21118_b200.attention import LatentKVCache
    n, s, dh = 4, 2, 16
    d = n * dh
    rng = np.random.default_rng(0)
    gran = M.Granularity.group_head(s)
    side = lambda rs: M.DecomposedLayer(gran, tuple(
        M.GroupFactors(rng.standard_normal((d, r)), rng.standard_normal((r, s * dh)), r) for r in rs),
        d, dh, n)
    dec = [M.LayerKV(key=side(RANKS["k"]), value=side(RANKS["v"])) for _ in range(LAYERS)]
    cfg = M.AttentionConfig(d, n, dh, layers=LAYERS)
    return LatentKVCache(dec, cfg, bits, batch=1, capacity=T + 8, device=torch.device("cuda"))


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_gpu_export_matches_reference_container(bits):
    """Latents appended through the CUDA quantiser and exported from the cache
    (codes re-packed on the GPU) reproduce the reference container bytes."""
    import torch

    from paper_2407_21118_b200 import _lib
    _lib.load()
    cache = _cache(bits)
    t_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    for li in range(LAYERS):
        for si, proj in enumerate(("k", "v")):
            st = cache._stores[li][si]
            rk = RANKS[proj]
            lat = np.concatenate([GOLDEN[f"lat.layer{li}.{proj}.g{g}"] for g in range(len(rk))], 1)
            lat_d = torch.from_numpy(np.ascontiguousarray(lat)).cuda()
            ranks = torch.tensor(rk, dtype=torch.int32, device="cuda")
            offs = torch.tensor(np.concatenate([[0], np.cumsum(rk)[:-1]]), dtype=torch.int32,
                                device="cuda")
            for t in range(T):
                t_dev.fill_(t)
                rc = _lib.call("palu_latent_append", 0, bits, lat_d[t].data_ptr(), 1, lat.shape[1],
                               len(rk), ranks.data_ptr(), offs.data_ptr(), st.rows.data_ptr(),
                               st.scales.data_ptr(), st.zps.data_ptr(), st.scales64.data_ptr(),
                               st.zps64.data_ptr(), st.r_pad, st.cap, t_dev.data_ptr(), None)
                assert rc == 0
    torch.cuda.synchronize()
    cache.t = T
    meta = {"model": {"name": "golden", "layers": LAYERS}, "seed": 0, "bits": bits}
    blob = PC.encode(PC.latent_tensors(cache), meta)
    ref = GOLDEN[f"palu_b{bits}"].tobytes()
    assert blob == ref
