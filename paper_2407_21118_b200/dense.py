"""Uncompressed GPU baseline: reference_decode (attention.py:133-168) on B200.

Standard cached multi-head attention over a post-RoPE key cache: per layer
one fused q|k|v GEMV, palu_dense_decode (RoPE + append row t + split-T
softmax(K q / sqrt(d_h)) V), and the W_o GEMV.  This is the comparator the
Palu path must beat (BASELINE.json: "beating uncompressed GPU attention");
bench.py also times flashinfer's trtllm-gen decode kernel at the same shape.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .attention import _dt, _ptr, _round_up, _stream, _torch, theta_table
from .errors import ValidationError
from .model import as_array, validate_weights


@dataclass
class DecodeResult:
    """attention.py:127-130."""

    outputs: np.ndarray
    cache: object


class DenseModel:
    """Device weights + K/V cache [B][n][T_cap][d_h] for the uncompressed path."""

    def __init__(self, config, wqkv: list, wo_t: list, dtype: str = "float32", batch: int = 1,
                 capacity: int = 256):
        torch = _torch()
        self.config, self.dtype, self.batch, self.cap = config, dtype, batch, capacity
        code, tdt = _dt(dtype)
        self.code = code
        dev = torch.device("cuda", torch.cuda.current_device())
        d, n, dh = config.d_model, config.n_heads, config.head_dim
        self.wqkv = [w.to(dev, tdt).contiguous() for w in wqkv]  # [3d, d] rows: q | k | v columns
        self.wo_t = [w.to(dev, tdt).contiguous() for w in wo_t]  # [d, d] = W_o^T
        L = len(self.wqkv)
        self.kc = torch.zeros(L, batch, n, capacity, dh, dtype=tdt, device=dev)
        self.vc = torch.zeros_like(self.kc)
        self.t = 0
        self.t_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        th = theta_table(dh, config.rope_base) if config.rope else np.zeros(dh // 2)
        self.theta = torch.from_numpy(th).to(dev)
        self.x = torch.zeros(batch, d, dtype=torch.float32, device=dev)
        self.qkv = torch.zeros(batch, 3 * d, dtype=torch.float32, device=dev)
        self.attn = torch.zeros(batch, d, dtype=torch.float32, device=dev)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.n_chunks = max(-(-2 * sms // (n * batch)), -(-capacity // 4096), 1)
        ws = _lib.call("palu_dense_workspace", batch, n, dh, self.n_chunks)
        self.ws = torch.zeros(ws // 4 + 1, dtype=torch.float32, device=dev)
        self.graph = None

    @classmethod
    def from_weights(cls, weights, config, dtype="float32", batch=1, capacity=256):
        torch = _torch()
        validate_weights(weights, config)
        wqkv, wo_t = [], []
        for lw in weights.layers:
            w = np.concatenate([as_array(lw.wq).T, as_array(lw.wk).T, as_array(lw.wv).T], axis=0)
            wqkv.append(torch.from_numpy(np.ascontiguousarray(w)))
            wo_t.append(torch.from_numpy(np.ascontiguousarray(as_array(lw.wo).T)))
        return cls(config, wqkv, wo_t, dtype, batch, capacity)

    def launch_step(self):
        if not self.config.rope:
            raise ValidationError("the B200 uncompressed baseline implements the rope-on path")
        st = _stream()
        d, n, dh = self.config.d_model, self.config.n_heads, self.config.head_dim
        B = self.batch
        for li in range(len(self.wqkv)):
            _lib.call("palu_gemv", self.code, _ptr(self.wqkv[li]), 3 * d, d, _ptr(self.x), B, d,
                      _ptr(self.qkv), 3 * d, 0, st)
            _lib.call("palu_dense_decode", self.code, _ptr(self.qkv), B, n, dh, _ptr(self.kc[li]),
                      _ptr(self.vc[li]), self.cap, _ptr(self.theta), _ptr(self.t_dev),
                      self.n_chunks, _ptr(self.ws), _ptr(self.attn), st)
            _lib.call("palu_gemv", self.code, _ptr(self.wo_t[li]), d, d, _ptr(self.attn), B, d,
                      _ptr(self.x), d, 0, st)
        _lib.call("palu_advance", _ptr(self.t_dev), st)

    def step_device(self, use_graph=True):
        torch = _torch()
        if not use_graph:
            self.launch_step()
            return
        if self.graph is None:
            import gc

            self.launch_step()  # warm (lazy module load) outside capture
            gc.collect()  # no dead graph may be destroyed while the capture is open
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self.launch_step()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = g
            return
        self.graph.replay()


def reference_decode(weights, config, token_stream, *, dtype: str = "float32") -> DecodeResult:
    """attention.py:133-168 on the GPU: standard cached MHA over a stream."""
    tokens = np.asarray(token_stream, dtype=np.float64)
    if tokens.ndim != 2 or tokens.shape[1] != config.d_model:
        raise ValidationError(f"token stream must be (T, {config.d_model})")
    torch = _torch()
    m = DenseModel.from_weights(weights, config, dtype=dtype, capacity=max(tokens.shape[0], 8))
    outputs = np.zeros_like(tokens)
    for t in range(tokens.shape[0]):
        m.x.copy_(torch.from_numpy(tokens[t:t + 1].astype(np.float32)))
        m.step_device(use_graph=False)
        m.t += 1
        outputs[t] = m.x[0].double().cpu().numpy()
    return DecodeResult(outputs=outputs, cache=m)
