"""B200-native (sm_100a) Palu latent-KV RoPE decode attention.

Drop-in for the decode path of the reference package ``palu``
(pkg/src/palu/attention.py): same public names, argument meaning and error
behaviour, with the numpy stages replaced by hand-written CUDA kernels in
``libpalu_b200.so`` (C ABI: include/palu_b200.h).
"""

from .attention import (
    FP_BITS,
    FusedWeights,
    LatentKVCache,
    LayerFused,
    QuantizedLatent,
    build_fused,
    palu_decode,
    palu_decode_step_norope,
    palu_decode_step_quantized,
    palu_decode_step_rope,
    palu_prefill,
    rope_apply,
)
from . import container, offline, rank_plan
from .offline import decompose_gpu, fuse_hadamard_gpu
from .container import export_latents
from .dense import DecodeResult, DenseModel, reference_decode
from .errors import GoldenMismatchError, NumericalError, PaluError, ValidationError
from .model import (
    AttentionConfig,
    DecomposedLayer,
    Granularity,
    GroupFactors,
    LayerKV,
    LayerWeights,
    Matrix,
    ModelWeights,
    RotatedLayer,
    fuse_hadamard,
    hadamard,
)

__version__ = "0.1.0"
