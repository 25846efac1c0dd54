"""Host-side layered vector (the reference's flat-buffer-plus-offsets layout, R: layered.py:23-125).

Only what the drop-in step needs: a flat numpy array plus (layer_id, dim)
records with layer ids 1..L.  ``lags_step`` also accepts the reference's own
``LayeredVector`` objects (duck typing on ``.shape`` / ``.data``).  On the
device the same layout is one flat tensor per worker with the offsets kept in
the bucket's layer table (include/lags_b200.h, ``lags_layer_t``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import StructureError


@dataclass(frozen=True)
class LayerShape:
    """One layer's 1-based position and element count (R: layered.py:23-32)."""

    layer_id: int
    dim: int

    def __post_init__(self):
        if self.dim <= 0:
            raise StructureError(f"layer {self.layer_id}: dim must be positive, got {self.dim}")


def layout_of(vec) -> tuple[tuple[int, int], ...]:
    """(layer_id, dim) pairs of any layered vector (ours or the reference's)."""
    return tuple((int(ls.layer_id), int(ls.dim)) for ls in vec.shape)


def validate_layout(pairs: Sequence[tuple[int, int]]) -> None:
    """Layer ids must run 1..L (R: layered.py:35-43)."""
    if not pairs:
        raise StructureError("shape must contain at least one layer")
    for pos, (lid, _) in enumerate(pairs, start=1):
        if lid != pos:
            raise StructureError(f"layer ids must be consecutive from 1; position {pos} has id {lid}")


class LayeredVector:
    """Flat array + layer split; ``layer_slice`` returns writable views."""

    __slots__ = ("shape", "data", "_off")

    def __init__(self, shape: Sequence[LayerShape], data):
        shape = tuple(shape)
        validate_layout([(ls.layer_id, ls.dim) for ls in shape])
        data = np.asarray(data)
        if data.ndim != 1:
            raise StructureError(f"data must be 1-D, got ndim={data.ndim}")
        off = np.zeros(len(shape) + 1, dtype=np.int64)
        np.cumsum([ls.dim for ls in shape], out=off[1:])
        if data.shape[0] != off[-1]:
            raise StructureError(f"data length {data.shape[0]} does not match layer dims summing to {off[-1]}")
        self.shape = shape
        self.data = data
        self._off = off

    @classmethod
    def zeros(cls, shape, dtype=np.float64):
        shape = tuple(shape)
        return cls(shape, np.zeros(sum(ls.dim for ls in shape), dtype=dtype))

    @classmethod
    def zeros_like(cls, other):
        return cls(other.shape, np.zeros(other.data.shape[0], dtype=other.data.dtype))

    @property
    def dim(self) -> int:
        return int(self._off[-1])

    @property
    def num_layers(self) -> int:
        return len(self.shape)

    @property
    def dtype(self):
        return self.data.dtype

    def copy(self):
        return LayeredVector(self.shape, self.data.copy())

    def layer_slice(self, layer_id: int) -> np.ndarray:
        if not 1 <= layer_id <= len(self.shape):
            raise IndexError(f"layer_id {layer_id} outside 1..{len(self.shape)}")
        return self.data[self._off[layer_id - 1]:self._off[layer_id]]


def concat(parts, dtype=np.float64) -> LayeredVector:
    parts = [np.asarray(p, dtype=dtype) for p in parts]
    if not parts:
        raise StructureError("cannot concatenate an empty list of parts")
    return LayeredVector([LayerShape(i, p.size) for i, p in enumerate(parts, start=1)], np.concatenate(parts))
