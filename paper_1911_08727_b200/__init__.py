"""B200-native LAGS-SGD sparsify -> exchange -> decode -> update path (arXiv 1911.08727).

Drop-in for the reference package ``lagsgd`` on its hot path: same names,
argument meaning and errors (``top_k``, ``decompress``, ``lags_step``,
``CompressionPolicy``, ``SparseChunk``, ``StepSizeSchedule``), backed by the
hand-written sm_100a kernels of ``liblagsb200.so`` (C ABI: include/lags_b200.h).
Importing the package fails loudly when the library has not been built.
"""

from . import _native  # noqa: F401  (raises ImportError when liblagsb200.so is missing)
from .engine import Bucket
from .errors import DivergenceError, StructureError
from .layered import LayeredVector, LayerShape, concat
from .sparsify import (
    CompressionPolicy, FusionBuffer, FusionMessage, SparseChunk, decode_chunk, decode_message, decompress, encode_chunk,
    encode_message, fusion_flush, top_k, top_k_device,
)
from .training import StepSizeSchedule, lags_step, slgs_step
from .analysis import topk_aggregation_ratio

__all__ = [
    "Bucket", "CompressionPolicy", "DivergenceError", "FusionBuffer", "FusionMessage", "LayeredVector", "LayerShape",
    "SparseChunk", "StepSizeSchedule", "StructureError", "concat", "decode_chunk", "decode_message", "decompress",
    "encode_chunk", "encode_message", "fusion_flush", "lags_step", "slgs_step", "top_k", "top_k_device",
    "topk_aggregation_ratio",
]
__version__ = "0.1.0"
