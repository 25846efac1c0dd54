"""Sparse wire format on the device (R: sparsify.py:260-310) through liblagsb200.so.

chunk = u32 layer_id, u32 dim, u32 count, count x (u32 index, f64 value), little-endian;
message = u32 chunk count + chunks.  ``encode_table`` / ``decode_table`` work on a chunk table of
device tensors (a bucket's message, or uploaded SparseChunks); the reference-named host functions
(``encode_chunk`` ... ``decode_message``) in ``sparsify`` are built on them.  Errors map to the
reference's ``StructureError`` messages, the first bad chunk in stream order winning.
"""

from __future__ import annotations

import torch

from . import _native as N
from .errors import StructureError

MESSAGE, CHUNK = N.WIRE_MESSAGE, N.WIRE_CHUNK


def _u32(values, device) -> torch.Tensor:
    """uint32 values as the bits of an int32 tensor (the kernels read u32)."""
    t = torch.as_tensor([int(v) & 0xFFFFFFFF for v in values], dtype=torch.int64)
    return torch.where(t >= 2**31, t - 2**32, t).to(torch.int32).to(device)


def _as_u32(t: torch.Tensor) -> list[int]:
    return [int(v) & 0xFFFFFFFF for v in t.cpu().tolist()]


def _val_mode(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return N.F32
    if dtype == torch.float64:
        return N.F64
    raise TypeError(f"wire values must be float32 or float64, got {dtype}")


def wire_bytes(counts, with_header: bool = True) -> int:
    """Encoded length: 12 + 12 * count per chunk (+ 4)."""
    return (4 if with_header else 0) + sum(12 + 12 * int(c) for c in counts)


def raise_for(code: int, end: int = 0, length: int = 0) -> None:
    """Raise the reference's exception for a device error word (no-op when OK)."""
    if code == N.WIRE_OK:
        return
    kind = code & 0xFF
    if kind == N.WIRE_ERR_TRUNCATED_MESSAGE:
        raise StructureError("truncated message header")
    if kind == N.WIRE_ERR_TRUNCATED_HEADER:
        raise StructureError("truncated chunk header")
    if kind == N.WIRE_ERR_TRUNCATED_PAYLOAD:
        raise StructureError("truncated chunk payload")
    if kind == N.WIRE_ERR_INDEX_RANGE:
        raise StructureError("indices out of range for layer dim")
    if kind == N.WIRE_ERR_INDEX_ORDER:
        raise StructureError("indices must be strictly increasing")
    if kind == N.WIRE_ERR_TRAILING:
        raise StructureError(f"{length - end} trailing bytes after message payload")
    if kind == N.WIRE_ERR_CAPACITY:
        raise ValueError(f"wire buffer or chunk table too small (chunk {code >> 8})")
    raise RuntimeError(f"unknown wire error word {code:#x}")


def encode_table(layer_ids: torch.Tensor, dims: torch.Tensor, counts: torch.Tensor, first: torch.Tensor,
                 idx: torch.Tensor, val: torch.Tensor, mode: int = MESSAGE, capacity: int | None = None,
                 stream=None):
    """Encode a device chunk table.  Returns (wire uint8 [capacity], wire_len int64 [1], error int64 [1]),
    all on the device; nothing is synchronised."""
    dev = idx.device
    n = int(counts.numel())
    if capacity is None:
        raise ValueError("capacity (bytes) is required: the counts live on the device")
    wire = torch.empty(max(int(capacity), 4), dtype=torch.uint8, device=dev)
    wlen = torch.zeros(1, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int64, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    N.check(N.lags_wire_encode(mode, n, layer_ids.data_ptr(), dims.data_ptr(), counts.data_ptr(), first.data_ptr(),
                               idx.data_ptr(), val.data_ptr(), _val_mode(val.dtype), wire.data_ptr(), int(capacity),
                               wlen.data_ptr(), err.data_ptr(), s.cuda_stream), "lags_wire_encode")
    return wire, wlen, err


def decode_table(wire: torch.Tensor, length: int, offset: int = 0, mode: int = MESSAGE, max_chunks: int | None = None,
                 first: torch.Tensor | None = None, caps: torch.Tensor | None = None,
                 entry_capacity: int | None = None, val_dtype: torch.dtype = torch.float64,
                 idx: torch.Tensor | None = None, val: torch.Tensor | None = None, stream=None) -> dict:
    """Decode wire[offset:length] on the device into a chunk table (tensors in the returned dict:
    layer_ids, dims, counts, idx, val, nchunks, end, error).  idx / val may be given (e.g. a bucket
    message's views with ``first`` = its slot offsets); else packed outputs are allocated."""
    dev = wire.device
    if max_chunks is None:
        max_chunks = 1 if mode == CHUNK else max(1, min(N.WIRE_MAX_CHUNKS, (int(length) - int(offset) - 4) // 12))
    if entry_capacity is None:
        entry_capacity = max(1, (int(length) - int(offset)) // 12)
    if idx is None:
        idx = torch.empty(entry_capacity, dtype=torch.int32, device=dev)
    if val is None:
        val = torch.empty(entry_capacity, dtype=val_dtype, device=dev)
    out = dict(
        layer_ids=torch.zeros(max_chunks, dtype=torch.int32, device=dev),
        dims=torch.zeros(max_chunks, dtype=torch.int32, device=dev),
        counts=torch.zeros(max_chunks, dtype=torch.int32, device=dev),
        idx=idx, val=val,
        nchunks=torch.zeros(1, dtype=torch.int32, device=dev),
        end=torch.zeros(1, dtype=torch.int64, device=dev),
        error=torch.zeros(1, dtype=torch.int64, device=dev),
    )
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    N.check(N.lags_wire_decode(mode, wire.data_ptr(), int(length), int(offset), int(max_chunks),
                               first.data_ptr() if first is not None else None,
                               caps.data_ptr() if caps is not None else None, int(entry_capacity),
                               out["layer_ids"].data_ptr(), out["dims"].data_ptr(), out["counts"].data_ptr(),
                               idx.data_ptr(), val.data_ptr(), _val_mode(val.dtype), out["nchunks"].data_ptr(),
                               out["end"].data_ptr(), out["error"].data_ptr(), s.cuda_stream), "lags_wire_decode")
    return out


def error_word(t: torch.Tensor) -> int:
    return int(t.item()) & 0xFFFFFFFFFFFFFFFF
