"""Reconstruct-once score for replicated-B key groups (GQA as its MHA-equivalent
layer, BASELINE configs[3]), host side and algebra, CPU only.

* replicated_key_operand must recognise groups whose query-head blocks of B_k
  are all equal and return the K-major B operand [G][d_h][R_pad];
* the kernel's epilogue formula -- rotate each (j, j + d_h/2) pair of
  K = H B_kv by the token's angle, dot with scale x RoPE(q) -- must equal the
  oracle's logits rope(K_t, t) . rope(q, pos) / sqrt(d_h) (attention.py:433-444
  via oracle.rope_rows).
"""

import math

import numpy as np
import torch

from oracle import palu_oracle as po
from paper_2407_21118_b200.attention import replicated_key_operand


def _bk(G=3, rows=8, s=4, dh=16, replicated=True, seed=0):
    g = torch.Generator().manual_seed(seed)
    if replicated:
        blk = torch.randn(G, rows, dh, generator=g)
        return blk.repeat(1, 1, s), blk
    return torch.randn(G, rows, s * dh, generator=g), None


def test_replicated_groups_give_the_kv_head_operand():
    bk, blk = _bk()
    r_pad = 6
    op = replicated_key_operand(bk, r_pad, 4, 16)
    assert op is not None and op.shape == (3, 16, r_pad)
    assert torch.equal(op, blk[:, :r_pad].transpose(1, 2))
    assert op.is_contiguous()


def test_distinct_head_blocks_are_not_replicated():
    bk, _ = _bk(replicated=False)
    assert replicated_key_operand(bk, 8, 4, 16) is None
    # one group differing in one head block is enough to refuse
    bk, _ = _bk()
    bk[1, 0, 2 * 16] += 1.0
    assert replicated_key_operand(bk, 8, 4, 16) is None
    # a width that is not s_k x d_h is refused, not reshaped
    assert replicated_key_operand(bk, 8, 3, 16) is None


def test_epilogue_formula_matches_rope_logits():
    rng = np.random.default_rng(7)
    dh, r, T, s, base, pos = 16, 6, 40, 4, 1e6, 39
    H = rng.standard_normal((T, r))
    B = rng.standard_normal((r, dh))
    q = rng.standard_normal((s, dh))
    scale = 1.0 / math.sqrt(dh)
    t = np.arange(T, dtype=np.float64)
    # oracle: rope(H B, t) . rope(q, pos) / sqrt(d_h)
    want = po.rope_rows(H @ B, t, base) @ po.rope_rows(q, np.full(s, float(pos)), base).T * scale
    # kernel: accumulator columns j (dim j) and j + h (dim j + h) of K = H B
    # (the B operand rows of replicated_key_operand), pair rotation, dot with
    # the rotated, scaled queries (absorb layout 4)
    op = replicated_key_operand(torch.from_numpy(np.tile(B, (1, s)))[None], r, s, dh)[0].numpy()
    acc = H @ op.T
    h = dh // 2
    theta = base ** (-2.0 * np.arange(h) / dh)
    c, sn = np.cos(t[:, None] * theta), np.sin(t[:, None] * theta)
    lo, hi = acc[:, :h], acc[:, h:]
    klo, khi = c * lo - sn * hi, sn * lo + c * hi
    qr = scale * po.rope_rows(q, np.full(s, float(pos)), base)
    got = klo @ qr[:, :h].T + khi @ qr[:, h:].T
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
