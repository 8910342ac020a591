"""Model / factor types of the reference API, same names and validation.

Mirrors palu.attention's AttentionConfig / LayerWeights / ModelWeights /
LayerKV (attention.py:34-90) and palu.decompose's Granularity /
GroupFactors / DecomposedLayer (decompose.py:30-118).  Matrices may be the
reference's own immutable ``Matrix`` objects (anything with ``.data``) or
plain arrays, so objects built with the reference package drop in unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError

MULTI_HEAD = "multi_head"
GROUP_HEAD = "group_head"
JOINT_HEAD = "joint_head"


def as_array(m) -> np.ndarray:
    """Read-only float64 view of a reference ``Matrix`` (core.py:21-43) or array."""
    data = m.data if hasattr(m, "data") and not isinstance(m, np.ndarray) else m
    arr = np.asarray(data, dtype=np.float64)
    if arr.ndim != 2:
        raise ValidationError(f"Matrix requires a 2-D payload, got ndim={arr.ndim}")
    return arr


def _shape(m):
    return tuple(m.shape) if hasattr(m, "shape") else as_array(m).shape


@dataclass(frozen=True)
class AttentionConfig:
    """attention.py:34-54."""

    d_model: int
    n_heads: int
    head_dim: int
    layers: int
    rope: bool = False
    rope_base: float = 10000.0

    def __post_init__(self):
        if self.d_model != self.n_heads * self.head_dim:
            raise ValidationError(
                f"d_model {self.d_model} != n_heads*head_dim {self.n_heads * self.head_dim}")
        if self.layers < 1:
            raise ValidationError(f"layers must be >= 1, got {self.layers}")
        if self.rope:
            if self.rope_base <= 1.0:
                raise ValidationError(f"rope base must exceed 1, got {self.rope_base}")
            if self.head_dim % 2 != 0:
                raise ValidationError("rotary embedding requires an even head_dim")


@dataclass(frozen=True)
class LayerWeights:
    """attention.py:57-65: wq/wk/wv column blocks per head, wo row blocks."""

    wq: object
    wk: object
    wv: object
    wo: object


@dataclass(frozen=True)
class ModelWeights:
    """attention.py:68-82."""

    layers: tuple

    def validate_for(self, config) -> None:
        if len(self.layers) != config.layers:
            raise ValidationError(f"{len(self.layers)} weight layers for a {config.layers}-layer config")
        d = config.d_model
        for i, lw in enumerate(self.layers):
            for name in ("wq", "wk", "wv", "wo"):
                shp = _shape(getattr(lw, name))
                if shp != (d, d):
                    raise ValidationError(f"layer {i} {name} has shape {shp}, expected ({d}, {d})")


def validate_weights(weights, config) -> None:
    """ModelWeights.validate_for for ours or the reference's object."""
    ModelWeights.validate_for(weights, config)


@dataclass(frozen=True)
class Granularity:
    """decompose.py:30-72."""

    kind: str
    group_size: int

    def __post_init__(self):
        if self.kind not in (MULTI_HEAD, GROUP_HEAD, JOINT_HEAD):
            raise ValidationError(f"unknown granularity kind {self.kind!r}")
        if self.group_size < 1:
            raise ValidationError(f"group_size must be positive, got {self.group_size}")
        if self.kind == MULTI_HEAD and self.group_size != 1:
            raise ValidationError("multi_head granularity requires group_size 1")

    @classmethod
    def multi_head(cls):
        return cls(MULTI_HEAD, 1)

    @classmethod
    def group_head(cls, group_size: int):
        return cls(GROUP_HEAD, group_size)

    @classmethod
    def joint_head(cls, n_heads: int):
        return cls(JOINT_HEAD, n_heads)

    def validate_for(self, n_heads: int) -> None:
        if n_heads % self.group_size != 0:
            raise ValidationError(f"group_size {self.group_size} does not divide n_heads {n_heads}")
        if self.kind == JOINT_HEAD and self.group_size != n_heads:
            raise ValidationError(
                f"joint_head granularity requires group_size == n_heads ({self.group_size} != {n_heads})")
        if self.kind == GROUP_HEAD and self.group_size == 1:
            raise ValidationError("group_head with group_size 1 is multi_head")

    def n_groups(self, n_heads: int) -> int:
        self.validate_for(n_heads)
        return n_heads // self.group_size


@dataclass(frozen=True)
class GroupFactors:
    """decompose.py:75-87: a (d x rank) down- and b (rank x width) up-projection."""

    a: object
    b: object
    rank: int

    def __post_init__(self):
        sa, sb = _shape(self.a), _shape(self.b)
        if sa[1] != self.rank or sb[0] != self.rank:
            raise ValidationError(f"factor shapes {sa} / {sb} disagree with rank {self.rank}")


@dataclass(frozen=True)
class DecomposedLayer:
    """decompose.py:90-118."""

    granularity: Granularity
    groups: tuple
    d_model: int
    head_dim: int
    n_heads: int

    def __post_init__(self):
        expect = self.granularity.n_groups(self.n_heads)
        if len(self.groups) != expect:
            raise ValidationError(f"expected {expect} groups, got {len(self.groups)}")
        width = self.head_dim * self.granularity.group_size
        for g in self.groups:
            sa, sb = _shape(g.a), _shape(g.b)
            if sa[0] != self.d_model or sb[1] != width:
                raise ValidationError(
                    f"group factors {sa} x {sb} do not match d_model {self.d_model} and group width {width}")
            if g.rank > min(self.d_model, width):
                raise ValidationError(
                    f"rank {g.rank} exceeds min(d, group width) {min(self.d_model, width)}")

    @property
    def group_width(self) -> int:
        return self.head_dim * self.granularity.group_size

    @property
    def ranks(self) -> tuple:
        return tuple(g.rank for g in self.groups)


@dataclass(frozen=True)
class LayerKV:
    """attention.py:85-90."""

    key: object
    value: object


class Matrix:
    """Read-only 2-D float64 matrix with the reference's surface (core.py:21-66):
    ``.data`` (non-writable ndarray), ``.rows``, ``.cols``, ``.shape``, ``wrap``,
    ``t()`` and ``@``.  Returned by the offline helpers so callers written
    against the reference (``hadamard(r).data``) run unchanged."""

    __slots__ = ("data",)

    def __init__(self, data, *, _own: bool = False):
        arr = np.asarray(data, dtype=np.float64)
        arr = np.ascontiguousarray(arr) if _own else np.array(arr, dtype=np.float64, order="C", copy=True)
        if arr.ndim != 2:
            raise ValidationError(f"Matrix requires a 2-D payload, got ndim={arr.ndim}")
        if arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValidationError(f"Matrix dimensions must be positive, got {arr.shape}")
        if not np.all(np.isfinite(arr)):
            raise ValidationError("Matrix entries must be finite (found NaN or Inf)")
        arr.setflags(write=False)
        object.__setattr__(self, "data", arr)

    def __setattr__(self, name, value):
        raise AttributeError("Matrix is immutable")

    @classmethod
    def wrap(cls, arr) -> "Matrix":
        return cls(arr, _own=True)

    @property
    def rows(self) -> int:
        return self.data.shape[0]

    @property
    def cols(self) -> int:
        return self.data.shape[1]

    @property
    def shape(self) -> tuple:
        return self.data.shape

    def t(self) -> "Matrix":
        return Matrix.wrap(self.data.T.copy())

    def __matmul__(self, other) -> "Matrix":
        return Matrix.wrap(self.data @ as_array(other))

    def __array__(self, dtype=None, copy=None):
        return self.data if dtype is None else self.data.astype(dtype)


@dataclass(frozen=True)
class RotatedLayer:
    """quant.py:119-124: a DecomposedLayer whose factors carry a fused
    Hadamard rotation, plus the per-group rotation sizes."""

    layer: DecomposedLayer
    rotation_dims: tuple


def hadamard(dim: int) -> Matrix:
    """Offline prep (core.py:282-313): Sylvester blocks over the binary decomposition."""
    if dim <= 0:
        raise ValidationError(f"hadamard dimension must be positive, got {dim}")
    out = np.zeros((dim, dim))
    at, remaining = 0, dim
    while remaining:
        p = 1 << (remaining.bit_length() - 1)
        h = np.array([[1.0]])
        while h.shape[0] < p:
            h = np.block([[h, h], [h, -h]])
        out[at:at + p, at:at + p] = h / np.sqrt(p)
        at += p
        remaining -= p
    return Matrix.wrap(out)


def fuse_hadamard(layer: DecomposedLayer) -> RotatedLayer:
    """Offline prep (quant.py:127-153): (A, B) -> (A H, H^T B) per group;
    returns RotatedLayer(layer, rotation_dims) like the reference."""
    groups, dims = [], []
    for g in layer.groups:
        h = hadamard(g.rank).data
        groups.append(GroupFactors(a=Matrix.wrap(as_array(g.a) @ h), b=Matrix.wrap(h.T @ as_array(g.b)),
                                   rank=g.rank))
        dims.append(g.rank)
    rotated = DecomposedLayer(granularity=layer.granularity, groups=tuple(groups),
                              d_model=layer.d_model, head_dim=layer.head_dim, n_heads=layer.n_heads)
    return RotatedLayer(layer=rotated, rotation_dims=tuple(dims))
