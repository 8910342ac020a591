"""`.palu` latent export: the quantised latent cache written
in the reference's container format, byte for byte.

Format (restated from container.py:1-14 and write_container :92-124): the
4-byte magic ``PALU``, version byte 1, uint32-LE header length, a compact
UTF-8 JSON header ``{"meta": ..., "tensors": [...]}`` with sorted keys, then
the payloads in tensor-name order, each at an 8-byte aligned offset relative
to the data section (zero padding between them).  A tensor entry holds
``name``, ``dtype`` (``f64`` little-endian row-major, or ``u8-packed`` with
``bits``), ``shape``, ``offset`` and ``byte_len``.

``export_latents`` mirrors the pipeline's latent export (pipeline.py:513-531):
per layer, side (``k``/``v``) and group, ``layer{l}.{k|v}.g{g}.codes`` (the
T x rank codes packed as one bitstream, quant.py:156-169), ``.scales`` and
``.zero_points`` (fp64).  The codes are re-packed on the GPU from the cache's
padded rows (``palu_pack_code_stream``); scales and zero points come from the
fp64 copies the device quantiser keeps next to the fp32 ones.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ValidationError

MAGIC = b"PALU"
VERSION = 1
ALIGN = 8


class Packed:
    """A ``u8-packed`` payload: the bitstream and its logical code shape."""

    def __init__(self, data: bytes, shape, bits: int):
        if bits not in (2, 3, 4, 8):
            raise ValidationError(f"packed bits must be 2/3/4/8, got {bits}")
        n = int(np.prod(shape)) if len(shape) else 0
        if len(data) != (n * bits + 7) // 8:
            raise ValidationError(f"packed payload is {len(data)} bytes for shape {tuple(shape)}")
        self.data, self.shape, self.bits = bytes(data), tuple(int(s) for s in shape), bits


def encode(tensors: dict, meta: dict | None = None) -> bytes:
    """The container bytes of ``tensors`` (name -> fp64 array or Packed)."""
    entries, chunks, pos = [], [], 0
    for name in sorted(tensors):
        v = tensors[name]
        if isinstance(v, Packed):
            body = v.data
            ent = {"name": name, "dtype": "u8-packed", "shape": list(v.shape), "bits": v.bits}
        else:
            a = np.asarray(v, dtype=np.float64)
            if a.ndim == 0:
                raise ValidationError("scalar tensors are not supported; use shape (1,)")
            body = np.ascontiguousarray(a, dtype="<f8").tobytes()
            ent = {"name": name, "dtype": "f64", "shape": list(a.shape)}
        ent["offset"], ent["byte_len"] = pos, len(body)
        entries.append(ent)
        pad = (-(pos + len(body))) % ALIGN
        chunks.append(body + bytes(pad))
        pos += len(body) + pad
    head = json.dumps({"tensors": entries, "meta": meta or {}}, sort_keys=True,
                      separators=(",", ":")).encode("utf-8")
    return MAGIC + bytes([VERSION]) + len(head).to_bytes(4, "little") + head + b"".join(chunks)


def write(path, tensors: dict, meta: dict | None = None) -> None:
    Path(path).write_bytes(encode(tensors, meta))


def _pack_group(side, b: int, g: int, t: int) -> bytes:
    import torch

    r = side.ranks[g]
    nbytes = (t * r * side.bits + 7) // 8
    out = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=side.rows.device)
    row_bytes = side.rows.shape[-1]
    base = side.rows[b, g].data_ptr()
    _lib.call("palu_pack_code_stream", side.bits, base, row_bytes, r, t, out.data_ptr(), nbytes,
              torch.cuda.current_stream().cuda_stream)
    return out[:nbytes].cpu().numpy().tobytes()


def latent_tensors(cache, b: int = 0) -> dict:
    """Export tensors of sequence ``b`` of a quantised LatentKVCache
    (pipeline.py:517-525 naming); raw (bits 16) sides have nothing to export."""
    if not 0 <= b < cache.batch:
        raise ValidationError(f"sequence {b} outside batch {cache.batch}")
    t = cache.t
    out = {}
    for li, (ks, vs) in enumerate(cache._stores):
        for proj, side in (("k", ks), ("v", vs)):
            if side.bits == 16:
                continue
            for g, r in enumerate(side.ranks):
                name = f"layer{li}.{proj}.g{g}"
                out[f"{name}.codes"] = Packed(_pack_group(side, b, g, t), (t, r), side.bits)
                out[f"{name}.scales"] = side.scales64[b, g, :t].cpu().numpy()
                out[f"{name}.zero_points"] = side.zps64[b, g, :t].cpu().numpy().astype(np.float64)
    if not out:
        raise ValidationError("cache holds raw latents (bits 16); nothing to export")
    return out


def export_latents(cache, path, meta: dict | None = None, b: int = 0) -> None:
    """Write sequence ``b``'s quantised latents as a ``.palu`` container."""
    write(path, latent_tensors(cache, b), meta)
