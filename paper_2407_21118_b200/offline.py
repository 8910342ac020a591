"""Offline preparation on the GPU: factor decomposition, the
Hadamard fusion and the fused output/query weights, in fp64 on the device.

The reference runs these once per model on the CPU: decompose.py:142-199
(one-sided Jacobi SVD per head-group slab, core.py:159-257: ~80 s per
4096 x 512 slab), quant.py:127-153 (fuse_hadamard) and attention.py:194-232
(build_fused).  Here every head-group slab of a layer is one batched fp64
SVD / GEMM on the GPU (cuSOLVER / cuBLAS through torch -- library calls, not
the decode hot path), with the reference's conventions restated so that the
factors agree with the reference's to fp64 round-off:

  * descending singular values, truncated to the group rank;
  * sign: the largest-magnitude entry of every left singular vector is made
    non-negative, flipping the matching right vector (core.py:247-254);
  * A = U_r sqrt(S_r), B = sqrt(S_r) V_r^T (decompose.py:186-197); whitened
    mode decomposes L^T W_g for the Cholesky factor of X^T X + jitter I and
    un-whitens A (decompose.py:171-196).
"""

from __future__ import annotations

import numpy as np

from .errors import ValidationError
from .model import DecomposedLayer, GroupFactors, Matrix, RotatedLayer, as_array, hadamard

_WHITEN_JITTER_REL = 1e-6  # decompose.py:27


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("offline GPU preparation needs a CUDA device")
    return torch


def _rank_list(ranks, n_groups: int, max_rank: int) -> list:
    """decompose.py:128-139."""
    rl = [int(ranks)] * n_groups if isinstance(ranks, (int, np.integer)) else [int(r) for r in ranks]
    if len(rl) != n_groups:
        raise ValidationError(f"expected {n_groups} ranks, got {len(rl)}")
    for r in rl:
        if not (1 <= r <= max_rank):
            raise ValidationError(f"rank {r} outside [1, {max_rank}]")
    return rl


def decompose_gpu(w, n_heads: int, head_dim: int, granularity, ranks, mode: str = "plain",
                  calib=None, device=None) -> DecomposedLayer:
    """decompose.py:142-199 on the GPU: all groups' slabs in one batched SVD."""
    torch = _torch()
    dev = device or torch.device("cuda")
    wa = as_array(w)
    if wa.shape[1] != head_dim * n_heads:
        raise ValidationError(
            f"weight has {wa.shape[1]} columns, expected head_dim*n_heads = {head_dim * n_heads}")
    if hasattr(granularity, "validate_for"):
        granularity.validate_for(n_heads)
    if mode not in ("plain", "whitened"):
        raise ValidationError(f"unknown decomposition mode {mode!r}")
    d = wa.shape[0]
    s = granularity.group_size
    width, G = head_dim * s, n_heads // s
    rank_list = _rank_list(ranks, G, min(d, width))
    W = torch.from_numpy(np.ascontiguousarray(wa)).to(dev, torch.float64)
    slabs = W.reshape(d, G, width).permute(1, 0, 2)  # [G, d, width]
    lt = None
    if mode == "whitened":
        if calib is None:
            raise ValidationError("whitened mode requires a CalibrationSet")
        x = torch.from_numpy(np.ascontiguousarray(as_array(calib.x))).to(dev, torch.float64)
        if x.shape[1] != d:
            raise ValidationError(f"calibration width {x.shape[1]} != d_model {d}")
        if x.shape[0] < d:
            raise ValidationError(f"whitening needs at least d_model={d} samples, got {x.shape[0]}")
        gram = x.T @ x
        jitter = _WHITEN_JITTER_REL * float(torch.trace(gram)) / d
        low = torch.linalg.cholesky(gram + jitter * torch.eye(d, dtype=torch.float64, device=dev))
        lt = low.T
        slabs = lt.unsqueeze(0) @ slabs
    u, sv, vt = torch.linalg.svd(slabs, full_matrices=False)  # descending singular values
    # core.py:247-254: the largest-|entry| of each left vector is non-negative
    idx = u.abs().argmax(dim=1, keepdim=True)
    sign = torch.where(torch.gather(u, 1, idx) < 0, -1.0, 1.0)  # [G, 1, k]
    u = u * sign
    vt = vt * sign.transpose(1, 2)
    groups = []
    for j, r in enumerate(rank_list):
        root = sv[j, :r].sqrt()
        a = u[j, :, :r] * root
        if lt is not None:
            a = torch.linalg.solve_triangular(lt, a, upper=True)
        b = root[:, None] * vt[j, :r, :]
        groups.append(GroupFactors(Matrix.wrap(a.cpu().numpy()), Matrix.wrap(b.cpu().numpy()), r))
    return DecomposedLayer(granularity, tuple(groups), d, head_dim, n_heads)


def fuse_hadamard_gpu(layer, device=None) -> RotatedLayer:
    """quant.py:127-153 on the GPU: (A, B) -> (A H, H^T B) per group."""
    torch = _torch()
    dev = device or torch.device("cuda")
    groups, dims = [], []
    for g in layer.groups:
        h = torch.tensor(np.asarray(hadamard(g.rank).data), device=dev)  # copy: the Matrix view is read-only
        a = torch.from_numpy(np.ascontiguousarray(as_array(g.a))).to(dev, torch.float64)
        b = torch.from_numpy(np.ascontiguousarray(as_array(g.b))).to(dev, torch.float64)
        groups.append(GroupFactors(Matrix.wrap((a @ h).cpu().numpy()), Matrix.wrap((h.T @ b).cpu().numpy()),
                                   g.rank))
        dims.append(g.rank)
    rotated = DecomposedLayer(granularity=layer.granularity, groups=tuple(groups),
                              d_model=layer.d_model, head_dim=layer.head_dim, n_heads=layer.n_heads)
    return RotatedLayer(layer=rotated, rotation_dims=tuple(dims))


def fused_blocks_gpu(wq, wo, bk, bv, n_heads: int, head_dim: int, s_k: int, s_v: int, rope: bool,
                     device=None):
    """attention.py:214-221 on the GPU: wo_fused block i = B_v[g][:, i-in-g]
    @ W_o[rows i] (and wq_fused block i = W_q[:, i] @ B_k[g][:, i-in-g]^T when
    rope is off) as one batched fp64 GEMM over heads.  Returns numpy arrays."""
    torch = _torch()
    dev = device or torch.device("cuda")
    dh = head_dim
    t = lambda m: torch.from_numpy(np.ascontiguousarray(m)).to(dev, torch.float64)
    W_o = t(wo).reshape(n_heads, dh, -1)                                # [n, dh, d]
    bvh = [t(b) for b in bv]
    o_blocks = [bvh[i // s_v][:, (i % s_v) * dh:(i % s_v + 1) * dh] @ W_o[i] for i in range(n_heads)]
    wo_fused = torch.cat(o_blocks, dim=0).cpu().numpy()
    wq_fused = None
    if not rope:
        W_q = t(wq)
        bkh = [t(b) for b in bk]
        q_blocks = [W_q[:, i * dh:(i + 1) * dh] @ bkh[i // s_k][:, (i % s_k) * dh:(i % s_k + 1) * dh].T
                    for i in range(n_heads)]
        wq_fused = torch.cat(q_blocks, dim=1).cpu().numpy()
    return wo_fused, wq_fused
