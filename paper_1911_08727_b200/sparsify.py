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


# --- tensor fusion (R: sparsify.py:199-257) --------------------------------------------------


@dataclass(frozen=True)
class FusionMessage:
    """Chunks merged into one network message, per-layer identity retained (R: sparsify.py:199-206)."""

    chunks: tuple

    def nbytes(self, value_width: int = VALUE_BYTES_F64) -> int:
        return sum(c.nbytes(value_width) for c in self.chunks)


def fusion_flush(buffer: Sequence[SparseChunk], capacity_bytes: int, first_layer_done: bool,
                 value_width: int = VALUE_BYTES_F64) -> FusionMessage | None:
    """Flush rule of R: sparsify.py:209-238: send the buffered chunks when their accounting bytes
    reach the capacity or the backward pass has produced its final (first) layer; never split or
    reorder.  The same rule sizes LagsSGD's device buckets (optim.plan_buckets)."""
    if capacity_bytes <= 0:
        raise ValueError("capacity_bytes must be positive")
    chunks = tuple(buffer)
    seen: set[int] = set()
    for c in chunks:
        if c.layer_id in seen:
            raise StructureError(f"duplicate layer {c.layer_id} in fusion buffer")
        seen.add(c.layer_id)
        if c.nbytes(value_width) >= capacity_bytes:
            raise ValueError(f"capacity {capacity_bytes} does not exceed chunk of {c.nbytes(value_width)} bytes")
    if not chunks:
        return None
    if sum(c.nbytes(value_width) for c in chunks) >= capacity_bytes or first_layer_done:
        return FusionMessage(chunks)
    return None


class FusionBuffer:
    """Stateful wrapper around ``fusion_flush`` for streaming use (R: sparsify.py:241-257)."""

    def __init__(self, capacity_bytes: int, value_width: int = VALUE_BYTES_F64):
        self.capacity_bytes = capacity_bytes
        self.value_width = value_width
        self._pending: list[SparseChunk] = []

    def push(self, chunk: SparseChunk, first_layer_done: bool = False) -> FusionMessage | None:
        self._pending.append(chunk)
        msg = fusion_flush(self._pending, self.capacity_bytes, first_layer_done, self.value_width)
        if msg is not None:
            self._pending.clear()
        return msg

    def pending_bytes(self) -> int:
        return sum(c.nbytes(self.value_width) for c in self._pending)


# --- wire format (R: sparsify.py:260-310), encoded / decoded by the device kernels -------------


def _table(chunks: Sequence[SparseChunk]):
    from . import wire as W

    for c in chunks:
        if c.dim > 0x7FFFFFFF:
            raise ValueError(f"layer {c.layer_id}: dim {c.dim} exceeds the device index range (2^31 - 1)")
    counts = [len(c) for c in chunks]
    first = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64) if chunks else np.zeros(1, np.int64)
    n = max(sum(counts), 1)
    idx = np.zeros(n, dtype=np.int32)
    val = np.zeros(n, dtype=np.float64)
    for c, f in zip(chunks, first):
        idx[f:f + len(c)] = c.indices
        val[f:f + len(c)] = c.values  # f32 -> f64 is exact (R: sparsify.py:274)
    dev = torch.device("cuda")
    return (W._u32([c.layer_id for c in chunks] or [0], dev), W._u32([c.dim for c in chunks] or [0], dev),
            torch.tensor(counts or [0], dtype=torch.int32, device=dev), torch.from_numpy(first).to(dev),
            torch.from_numpy(idx).to(dev), torch.from_numpy(val).to(dev), counts)


def _encode(chunks: Sequence[SparseChunk], mode: int) -> bytes:
    from . import wire as W

    lids, dims, cnts, first, idx, val, counts = _table(chunks)
    cap = W.wire_bytes(counts, with_header=mode == W.MESSAGE)
    buf, wlen, err = W.encode_table(lids[:len(chunks)], dims[:len(chunks)], cnts[:len(chunks)], first, idx, val,
                                    mode=mode, capacity=cap)
    W.raise_for(W.error_word(err))
    return buf[: int(wlen.item())].cpu().numpy().tobytes()


def encode_chunk(chunk: SparseChunk) -> bytes:
    """R: sparsify.py:269-274 -- 12-byte header + count x (u32 index, f64 value)."""
    from . import wire as W

    return _encode([chunk], W.CHUNK)


def encode_message(message: FusionMessage) -> bytes:
    """R: sparsify.py:291-295 -- u32 chunk count + the chunks."""
    from . import wire as W

    return _encode(list(message.chunks), W.MESSAGE)


def _decode(buf: bytes, offset: int, mode: int):
    from . import wire as W

    raw = bytes(buf)
    t = torch.frombuffer(bytearray(raw), dtype=torch.uint8) if raw else torch.zeros(1, dtype=torch.uint8)
    out = W.decode_table(t.cuda(), len(raw), offset=offset, mode=mode)
    W.raise_for(W.error_word(out["error"]), int(out["end"].item()), len(raw))
    n = int(out["nchunks"].item())
    counts = out["counts"][:n].cpu().tolist()
    lids, dims = W._as_u32(out["layer_ids"][:n]), W._as_u32(out["dims"][:n])
    idx = out["idx"].cpu().numpy().astype(np.int64)
    val = out["val"].cpu().numpy()
    chunks, f = [], 0
    for lid, dim, c in zip(lids, dims, counts):
        chunks.append(SparseChunk(lid, dim, idx[f:f + c].copy(), val[f:f + c].copy(), k_target=c))
        f += c
    return chunks, int(out["end"].item())


def decode_chunk(buf: bytes, offset: int = 0) -> tuple[SparseChunk, int]:
    """R: sparsify.py:277-288 -- one chunk at ``offset``; returns (chunk, next offset)."""
    from . import wire as W

    chunks, end = _decode(buf, offset, W.CHUNK)
    return chunks[0], end


def decode_message(buf: bytes) -> FusionMessage:
    """R: sparsify.py:298-310 -- the whole buffer must be consumed."""
    from . import wire as W

    chunks, _ = _decode(buf, 0, W.MESSAGE)
    return FusionMessage(tuple(chunks))
