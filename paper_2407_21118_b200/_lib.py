"""ctypes binding of libpalu_b200.so (the C ABI in include/palu_b200.h).

There is no fallback: if the library is missing or the device is not
sm_100, every call raises.  This is the binding INTEGRATION.md documents.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PALU_LIB_PATH: load another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("PALU_LIB_PATH") or os.path.join(_HERE, "libpalu_b200.so")

PALU_OK = 0
PALU_EVALIDATION = -1
PALU_ECUDA = -2
PALU_EUNSUPPORTED = -3

DTYPE_F32 = 0
DTYPE_BF16 = 1

i32, i64, f32, p, sz = C.c_int, C.c_int64, C.c_float, C.c_void_p, C.c_size_t

# name -> (restype, argtypes); mirrors include/palu_b200.h one to one
SIGNATURES = {
    "palu_version": (C.c_char_p, []),
    "palu_last_error": (C.c_char_p, []),
    "palu_device_check": (i32, [i32]),
    "palu_gemv": (i32, [i32, p, i32, i32, p, i32, i32, p, i32, i32, p]),
    "palu_latent_append": (i32, [i32, i32, p, i32, i32, i32, p, p, p, p, p, p, p, i32, i32, p, p]),
    "palu_latent_append_kv": (i32, [i32, i32, i32, p, p, i32, i32, i32, i32, p, p, p, p,
                                    p, p, p, p, p, p, p, p, p, p, i32, i32, i32, p, p]),
    "palu_pack_code_stream": (i32, [i32, p, i32, i32, i32, p, i64, p]),
    "palu_quantize_rows": (i32, [p, i32, i32, i32, p, p, p, p]),
    "palu_pack_rows": (i32, [p, i32, i32, i32, p, p]),
    "palu_query_absorb": (i32, [i32, p, i32, i32, i32, i32, i32, p, i32, i32, p, f32, p, p, i32, p]),
    "palu_append_absorb": (i32, [i32, i32, i32, p, p, i32, i32, i32, i32, p, p, p, p,
                                 p, p, p, p, p, p, p, p, p, p, i32, i32, i32,
                                 p, i32, i32, i32, i32, p, i32, p, f32, p, i32, p, p]),
    "palu_rope_score": (i32, [i32, i32, p, p, p, i32, i32, i32, i32, i32, i32, i32, p, p, p, p,
                              i32, p]),
    "palu_rope_score_tc_splits": (i32, [i32, i32]),
    "palu_rope_score_tc": (i32, [i32, p, p, p, i32, i32, i32, i32, i32, i32, p, p, p, p, i32, p]),
    "palu_rope_score_tc_pf": (i32, [i32, p, p, p, i32, i32, i32, i32, i32, i32, p, p, p, p, i32, p, i64, p]),
    "palu_rope_score_tc_rep": (i32, [p, i32, i32, i32, i32, i32, p, p, p, p, p, i32, p]),
    "palu_rope_attend_workspace": (sz, [i32, i32, i32, i32, i32]),
    "palu_rope_attend_tc": (i32, [p, p, i32, i32, i32, i32, i32, i32, i32, p, p, p, p, i32, p, p, p,
                                  i32, p, i32, p]),
    "palu_value_tc": (i32, [i32, p, p, p, i32, i32, i32, i32, i32, i32, p, i32, p, p, p, p, i32, p,
                            p]),
    "palu_latent_score": (i32, [i32, i32, p, p, p, i32, i32, i32, i32, i32, i32, p, i32, p, p, f32,
                                p, p, i32, p]),
    "palu_latent_score_tc": (i32, [i32, p, p, p, i32, i32, i32, i32, i32, i32, p, i32, p, p, f32, p,
                                   p, i32, p]),
    "palu_fused_trace": (i32, [p, sz]),
    "palu_fused_max_clusters": (i32, [i32]),
    "palu_rope_table": (i32, [p, i32, i32, p, p]),
    "palu_rope_table_floats": (sz, [i32, i32]),
    "palu_softmax_value_workspace": (sz, [i32, i32, i32, i32]),
    "palu_softmax_value": (i32, [i32, i32, p, p, p, i32, i32, i32, i32, i32, p, p, i32, p, i32, i32,
                                 sz, p, i32, p, p, i32, p]),
    "palu_advance": (i32, [p, p]),
    "palu_dense_decode": (i32, [i32, p, i32, i32, i32, p, p, i32, p, p, i32, p, p, p]),
    "palu_dense_workspace": (sz, [i32, i32, i32, i32]),
    "palu_dense_append_paged": (i32, [p, i32, i32, i32, i32, p, i32, i32, p, p, p, p]),
    "palu_cast_bf16_f32": (i32, [p, p, i32, p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the library once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2407_21118_b200.build` "
            "(there is no CPU fallback for the Palu B200 path)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:  # an older build loaded through PALU_LIB_PATH (A/B timing)
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols(path: str = LIB_PATH) -> list[str]:
    lib = C.CDLL(path)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(status: int, what: str) -> None:
    if status >= PALU_OK:
        return
    msg = (_lib.palu_last_error() or b"").decode(errors="replace")
    if status == PALU_EVALIDATION:
        raise ValidationError(f"{what}: {msg}")
    if status == PALU_EUNSUPPORTED:
        raise ValidationError(f"{what}: unsupported configuration: {msg}")
    raise RuntimeError(f"{what} failed (CUDA): {msg}")


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    if SIGNATURES[name][0] is i32:
        check(rc, name)
    return rc
