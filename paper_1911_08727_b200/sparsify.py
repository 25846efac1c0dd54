"""Compression operators of the drop-in surface (R: sparsify.py).

``top_k`` and ``decompress`` run on the B200 through liblagsb200.so; there is
no CPU path.  ``SparseChunk`` and ``CompressionPolicy`` are host-side records
with the reference's invariants and error behaviour.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import StructureError

INDEX_BYTES = 4
VALUE_BYTES_F64 = 8
CHUNK_HEADER_BYTES = 8


@dataclass(frozen=True)
class SparseChunk:
    """Selected entries of one layer (R: sparsify.py:26-60): strictly increasing int64 indices."""

    layer_id: int
    dim: int
    indices: np.ndarray
    values: np.ndarray
    k_target: int

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64)
        vals = np.asarray(self.values)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", vals)
        if idx.ndim != 1 or idx.shape != vals.shape:
            raise StructureError("indices and values must be 1-D arrays of equal length")
        if idx.size > self.k_target:
            raise StructureError(f"{idx.size} entries exceed k_target={self.k_target}")
        if idx.size:
            if idx[0] < 0 or idx[-1] >= self.dim:
                raise StructureError("indices out of range for layer dim")
            if np.any(idx[1:] <= idx[:-1]):
                raise StructureError("indices must be strictly increasing")

    def __len__(self) -> int:
        return int(self.indices.size)

    def nbytes(self, value_width: int = VALUE_BYTES_F64) -> int:
        return CHUNK_HEADER_BYTES + len(self) * (INDEX_BYTES + value_width)


@dataclass(frozen=True)
class CompressionPolicy:
    """Per-layer compression ratio c_l = 1/rho_l plus the cap (R: sparsify.py:151-193)."""

    per_layer_ratio: Mapping[int, float]
    ratio_cap: float

    def __post_init__(self):
        ratios = {int(k): float(v) for k, v in dict(self.per_layer_ratio).items()}
        object.__setattr__(self, "per_layer_ratio", ratios)
        if self.ratio_cap < 1:
            raise ValueError(f"ratio_cap must be >= 1, got {self.ratio_cap}")
        for lid, c in ratios.items():
            if c < 1:
                raise ValueError(f"layer {lid}: ratio {c} < 1")
            if c > self.ratio_cap:
                raise ValueError(f"layer {lid}: ratio {c} exceeds cap {self.ratio_cap}")

    @classmethod
    def uniform(cls, ratio: float, shape, cap: float | None = None) -> "CompressionPolicy":
        return cls({ls.layer_id: float(ratio) for ls in shape}, float(cap) if cap is not None else float(ratio))

    @classmethod
    def from_density(cls, rho: float, shape, cap: float | None = None) -> "CompressionPolicy":
        """rho_l = 1/c_l (north_star vocabulary); 1/0.001 == 1000.0 exactly."""
        return cls.uniform(1.0 / rho, shape, cap)

    def ratio_for(self, layer_id: int) -> float:
        return self.per_layer_ratio[layer_id]

    def k_for(self, layer) -> int:
        # R: sparsify.py:182-184 -- min(d, max(1, floor(d / c))), floor on floats as numpy does
        return min(layer.dim, max(1, int(layer.dim // self.ratio_for(layer.layer_id))))

    def selection_counts(self, shape) -> dict[int, int]:
        return {ls.layer_id: self.k_for(ls) for ls in shape}

    def effective_max_ratio(self, shape) -> float:
        return max(ls.dim / self.k_for(ls) for ls in shape)

    def is_lossless(self, shape) -> bool:
        return all(self.k_for(ls) == ls.dim for ls in shape)


def _mode_of(dtype) -> int:
    if dtype in (np.float32, torch.float32):
        return N.F32
    if dtype in (np.float64, torch.float64):
        return N.F64
    raise TypeError(f"unsupported dtype {dtype}; the B200 path handles float32 and float64")


def top_k_device(x: torch.Tensor, k: int, stream=None):
    """Device top-k: returns (idx int32 [count], val [count]) CUDA tensors (one host sync for count)."""
    if x.dim() != 1 or x.numel() == 0:
        raise ValueError("input must be a non-empty 1-D array")
    d = x.numel()
    if not 1 <= k <= d:
        raise ValueError(f"k={k} outside 1..{d}")
    mode = _mode_of(x.dtype)
    x = x.contiguous()
    idx = torch.empty(k, dtype=torch.int32, device=x.device)
    val = torch.empty(k, dtype=x.dtype, device=x.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=x.device)
    ws = torch.empty(N.lags_top_k_workspace_bytes(mode, d), dtype=torch.uint8, device=x.device)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    N.check(N.lags_top_k(mode, x.data_ptr(), d, int(k), idx.data_ptr(), val.data_ptr(), cnt.data_ptr(),
                         ws.data_ptr(), ws.numel(), s.cuda_stream), "lags_top_k")
    n = int(cnt.item())
    return idx[:n], val[:n]


def top_k(x, k: int, layer_id: int = 0) -> SparseChunk:
    """Exact magnitude top-k on the GPU; same contract as R: sparsify.py:71-90.

    Accepts a numpy array (copied to the device) or a CUDA tensor.
    """
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
    else:
        arr = np.asarray(x)
        if arr.ndim != 1 or arr.size == 0:
            raise ValueError("input must be a non-empty 1-D array")
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    idx, val = top_k_device(t, int(k))
    return SparseChunk(layer_id, t.numel(), idx.cpu().numpy().astype(np.int64), val.cpu().numpy(), k_target=int(k))


def decompress(chunk: SparseChunk) -> np.ndarray:
    """Dense array with the chunk's values at its indices (R: sparsify.py:63-68), built on the GPU."""
    dtype = chunk.values.dtype if len(chunk) else np.dtype(np.float64)
    mode = _mode_of(dtype.type)
    tdt = torch.float32 if mode == N.F32 else torch.float64
    out = torch.empty(chunk.dim, dtype=tdt, device="cuda")
    n = len(chunk)
    idx = torch.from_numpy(chunk.indices.astype(np.int32)).cuda() if n else torch.zeros(1, dtype=torch.int32, device="cuda")
    val = torch.from_numpy(np.ascontiguousarray(chunk.values)).cuda() if n else torch.zeros(1, dtype=tdt, device="cuda")
    cnt = torch.tensor([n], dtype=torch.int32, device="cuda")
    N.check(N.lags_decompress(mode, idx.data_ptr(), val.data_ptr(), cnt.data_ptr(), chunk.dim, out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream), "lags_decompress")
    return out.cpu().numpy()
