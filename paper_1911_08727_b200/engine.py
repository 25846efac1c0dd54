"""Device-resident bucket engine: layer table, workspaces, message layout, C-ABI calls.

A *bucket* is a contiguous run of layers of the flat per-worker buffers (the
reference's LayeredVector layout, R: layered.py:46-107).  ``Bucket`` owns the
device copies of its layer table and workspaces and calls the CUDA library:

* ``compress``  -> lags_compress      (R: training.py:250-252 per worker, fused :174)
* ``decode``    -> lags_decode_update (R: training.py:248,253-254)

The sparse message of one worker for one bucket is a single byte buffer::

    [ counts int32[L] | pad | idx int32[sum k] | pad | val acc[sum k] | pad ]

so the exchange is one fixed-size all-gather of ``msg_bytes`` per rank.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _native as N


def _align(x: int, a: int = 16) -> int:
    return (x + a - 1) // a * a


def value_dtype(mode: int) -> torch.dtype:
    return torch.float32 if mode == N.F32 else torch.float64


def storage_dtype(mode: int) -> torch.dtype:
    return torch.float64 if mode == N.F64 else torch.float32


def _stream_handle(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Bucket:
    """One bucket of layers: dims/ks in flat order, a dtype mode and device workspaces."""

    def __init__(self, dims: Sequence[int], ks: Sequence[int], mode: int = N.F32, device=None,
                 world: int = 1, offsets: Sequence[int] | None = None):
        if len(dims) != len(ks) or not dims:
            raise ValueError("dims and ks must be non-empty and of equal length")
        for d, k in zip(dims, ks):
            if d < 1:
                raise ValueError(f"layer dim must be >= 1, got {d}")
            if not 1 <= k <= d:
                raise ValueError(f"k={k} outside 1..{d}")
            if d > 0x7FFFFFFF:
                raise ValueError("layer dim exceeds the int32 index range")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.mode = int(mode)
        self.dims = [int(d) for d in dims]
        self.ks = [int(k) for k in ks]
        self.nlayers = len(dims)
        off = np.zeros(self.nlayers + 1, dtype=np.int64)
        np.cumsum(self.dims, out=off[1:])
        self.offsets = off[:-1] if offsets is None else np.asarray(offsets, dtype=np.int64)
        self.n_total = int(off[-1]) if offsets is None else int(self.offsets[-1] + self.dims[-1])
        slots = np.zeros(self.nlayers + 1, dtype=np.int64)
        np.cumsum(self.ks, out=slots[1:])
        self.slots = slots[:-1]
        self.total_k = int(slots[-1])
        table = np.zeros(self.nlayers, dtype=N.LAYER_DTYPE)
        table["offset"], table["dim"], table["k"], table["slot"] = self.offsets, self.dims, self.ks, self.slots
        self.table = torch.from_numpy(table.view(np.uint8).copy()).to(self.device)
        # message layout
        self.val_size = 4 if self.mode == N.F32 else 8
        self.off_cnt = 0
        self.off_idx = _align(4 * self.nlayers)
        self.off_val = _align(self.off_idx + 4 * self.total_k)
        self.msg_bytes = _align(self.off_val + self.val_size * self.total_k)
        # workspaces
        cws = N.lags_compress_workspace_bytes(self.mode, self.nlayers, self.n_total, self.total_k)
        self.compress_ws = torch.empty(max(cws, 256), dtype=torch.uint8, device=self.device)
        self.state = torch.zeros(self.nlayers * N.STATE_BYTES, dtype=torch.uint8, device=self.device)
        self.world = int(world)
        self._decode_ws = None
        self._decode_P = 0

    # -- message views ---------------------------------------------------------------------
    def new_messages(self, count: int) -> torch.Tensor:
        return torch.zeros(count * self.msg_bytes, dtype=torch.uint8, device=self.device)

    def counts_view(self, msg: torch.Tensor) -> torch.Tensor:
        return msg[self.off_cnt:self.off_cnt + 4 * self.nlayers].view(torch.int32)

    def idx_view(self, msg: torch.Tensor) -> torch.Tensor:
        return msg[self.off_idx:self.off_idx + 4 * self.total_k].view(torch.int32)

    def val_view(self, msg: torch.Tensor) -> torch.Tensor:
        return msg[self.off_val:self.off_val + self.val_size * self.total_k].view(value_dtype(self.mode))

    # -- kernels -----------------------------------------------------------------------------
    def compress(self, g: torch.Tensor, r: torch.Tensor, alpha: float, msg: torch.Tensor,
                 status: torch.Tensor, stream=None, use_state: bool = True) -> None:
        """acc = r + alpha*g; select per layer; r <- acc with selected entries +0.0; msg <- pairs."""
        sd = storage_dtype(self.mode)
        if g.dtype != sd or r.dtype != sd:
            raise TypeError(f"bucket mode {self.mode} expects {sd} buffers")
        if g.numel() < self.n_total or r.numel() < self.n_total or msg.numel() < self.msg_bytes:
            raise ValueError("buffer smaller than the bucket")
        rc = N.lags_compress(
            self.mode, self.table.data_ptr(), self.nlayers, self.n_total, self.total_k,
            g.data_ptr(), r.data_ptr(), float(alpha),
            msg.data_ptr() + self.off_idx, msg.data_ptr() + self.off_val, msg.data_ptr() + self.off_cnt,
            status.data_ptr(), self.state.data_ptr() if use_state else None,
            self.compress_ws.data_ptr(), self.compress_ws.numel(), _stream_handle(stream))
        N.check(rc, "lags_compress")

    def decode_workspace(self, P: int) -> torch.Tensor:
        if self._decode_ws is None or self._decode_P < P:
            nbytes = N.lags_decode_workspace_bytes(self.mode, self.n_total, P)
            self._decode_ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
            self._decode_P = P
        return self._decode_ws

    def decode(self, msgs: torch.Tensor, P: int, v: torch.Tensor, momentum: torch.Tensor | None = None,
               mu: float = 0.0, stream=None) -> None:
        """Rank-ordered fp64 decode of P messages and v <- v - total/P (or momentum)."""
        if msgs.numel() < P * self.msg_bytes:
            raise ValueError("message buffer smaller than P messages")
        ws = self.decode_workspace(P)
        base = msgs.data_ptr()
        rc = N.lags_decode_update(
            self.mode, self.table.data_ptr(), self.nlayers, self.n_total, self.total_k,
            base + self.off_idx, base + self.off_val, base + self.off_cnt, self.msg_bytes, P,
            v.data_ptr(), momentum.data_ptr() if momentum is not None else None, float(mu),
            ws.data_ptr(), ws.numel(), _stream_handle(stream))
        N.check(rc, "lags_decode_update")

    # -- host helpers (tests / diagnostics) ----------------------------------------------------
    def unpack(self, msg: torch.Tensor):
        """[(idx int64 ndarray, val ndarray)] per layer from one message (copies to host)."""
        cnt = self.counts_view(msg).cpu().numpy()
        idx = self.idx_view(msg).cpu().numpy()
        val = self.val_view(msg).cpu().numpy()
        out = []
        for j in range(self.nlayers):
            s = int(self.slots[j])
            out.append((idx[s:s + cnt[j]].astype(np.int64), val[s:s + cnt[j]].copy()))
        return out
