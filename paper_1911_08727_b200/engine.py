"""Device-resident bucket engine: owns a bucket's device memory and calls the C ABI.

A *bucket* is a contiguous run of layers of the flat per-worker buffers (the
reference's LayeredVector layout, R: layered.py:46-107).  ``Bucket`` wraps the
library's ``lags_bucket_t`` handle:

* ``compress``  -> lags_bucket_compress      (R: training.py:250-252 per worker, fused :174)
* ``decode``    -> lags_bucket_decode_update (R: training.py:248,253-254)

One worker's sparse message for a bucket is a single byte buffer::

    [ counts int32[L] | pad | idx int32[sum k] | pad | val[sum k] | pad ]

so the exchange is one fixed-size all-gather of ``msg_bytes`` per rank.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .errors import StructureError


def value_dtype(mode: int) -> torch.dtype:
    return torch.float32 if mode == N.F32 else torch.float64


def storage_dtype(mode: int) -> torch.dtype:
    return torch.float64 if mode == N.F64 else torch.float32


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Bucket:
    """One bucket: layer dims/ks in flat order, a dtype mode, up to ``max_world`` exchanging ranks."""

    def __init__(self, dims: Sequence[int], ks: Sequence[int], mode: int = N.F32, device=None,
                 max_world: int = 1):
        if len(dims) != len(ks) or not len(dims):
            raise ValueError("dims and ks must be non-empty and of equal length")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.mode = int(mode)
        self.dims = [int(d) for d in dims]
        self.ks = [int(k) for k in ks]
        self.nlayers = len(self.dims)
        self.max_world = int(max_world)
        off = np.zeros(self.nlayers + 1, dtype=np.int64)
        np.cumsum(self.dims, out=off[1:])
        self.offsets = off[:-1]
        self.n_total = int(off[-1])
        slots = np.zeros(self.nlayers + 1, dtype=np.int64)
        np.cumsum(self.ks, out=slots[1:])
        self.slots = slots[:-1]
        self.total_k = int(slots[-1])
        for d, k in zip(self.dims, self.ks):
            if not 1 <= k <= d:  # R: sparsify.py:82-83
                raise ValueError(f"k={k} outside 1..{d}")
        d_arr = np.asarray(self.dims, dtype=np.int64)
        k_arr = np.asarray(self.ks, dtype=np.int32)
        nbytes = N.lags_bucket_device_bytes(self.mode, d_arr.ctypes.data, k_arr.ctypes.data, self.nlayers,
                                            self.max_world)
        if nbytes == 0:
            N.check(N.ERR_INVALID_ARG, "lags_bucket_device_bytes")
        with torch.cuda.device(self.device):
            self.memory = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            handle = C.c_void_p()
            N.check(N.lags_bucket_create(self.mode, d_arr.ctypes.data, k_arr.ctypes.data, self.nlayers,
                                         self.max_world, self.memory.data_ptr(), nbytes,
                                         stream_handle(torch.cuda.current_stream(self.device)), C.byref(handle)),
                    "lags_bucket_create")
        self._h = handle
        oc, oi, ov, mb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lags_bucket_message_layout(self._h, C.byref(oc), C.byref(oi), C.byref(ov), C.byref(mb)))
        self.off_cnt, self.off_idx, self.off_val, self.msg_bytes = oc.value, oi.value, ov.value, mb.value
        self.val_size = 4 if self.mode == N.F32 else 8

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = getattr(N, "lags_bucket_destroy", None)
        if h and destroy is not None:  # at interpreter shutdown the binding may already be gone
            destroy(h)
            self._h = None

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
                 status: torch.Tensor, stream=None, exact: bool = False, zero_grad: bool = False,
                 peer=None) -> None:
        """acc = r + alpha*g; per-layer top-k; r <- acc with selected entries +0.0; msg <- pairs.
        ``zero_grad`` clears g in the same pass (the optimizer's fused zero_grad).  ``peer`` (a
        p2p.PeerExchange): the selection also pushes every finished layer into every rank's
        receive area (fused exchange); follow it with ``peer.wait(stream)``."""
        self._check_buffers(g, r, None, msg)
        flags = (N.COMPRESS_EXACT if exact else 0) | (N.COMPRESS_ZERO_GRAD if zero_grad else 0)
        if peer is not None:
            N.check(N.lags_bucket_compress_push(self._h, g.data_ptr() if g is not None else None, r.data_ptr(),
                                                float(alpha), msg.data_ptr(), status.data_ptr(), flags,
                                                C.byref(peer.push_desc(self.msg_bytes)), stream_handle(stream)),
                    "lags_bucket_compress_push")
            return
        N.check(N.lags_bucket_compress(self._h, g.data_ptr() if g is not None else None, r.data_ptr(), float(alpha),
                                       msg.data_ptr(), status.data_ptr(), flags, stream_handle(stream)),
                "lags_bucket_compress")

    def step_local(self, g: torch.Tensor, r: torch.Tensor, alpha: float, v: torch.Tensor, msg: torch.Tensor,
                   status: torch.Tensor, stream=None, exact: bool = False, zero_grad: bool = False) -> None:
        """Single rank (P = 1): compress with v <- v - sent fused into the selection epilogue."""
        self._check_buffers(g, r, v, msg)
        flags = (N.COMPRESS_EXACT if exact else 0) | (N.COMPRESS_ZERO_GRAD if zero_grad else 0)
        N.check(N.lags_bucket_step_local(self._h, g.data_ptr() if g is not None else None, r.data_ptr(), float(alpha),
                                         v.data_ptr(), msg.data_ptr(), status.data_ptr(), flags,
                                         stream_handle(stream)), "lags_bucket_step_local")

    def _check_buffers(self, g, r, v, msg) -> None:
        sd = storage_dtype(self.mode)
        if g is None and getattr(self, "_grad_table", None) is None:
            raise ValueError("g is required unless a gradient table is set (set_grad_table)")
        for t in (g, r, v):
            if t is not None and (t.dtype != sd or t.numel() < self.n_total):
                raise TypeError(f"bucket mode {self.mode} expects {sd} buffers of >= {self.n_total} elements")
        if msg.numel() < self.msg_bytes:
            raise ValueError("message buffer smaller than the bucket's message")

    def set_grad_table(self, table: torch.Tensor | None) -> None:
        """Read gradients through a device int64 tensor of nlayers per-layer gradient pointers
        (lags_bucket_set_grad_table); compress / step_local then take g=None.  None: flat g again."""
        if table is not None and (table.dtype != torch.int64 or table.numel() < self.nlayers or not table.is_cuda):
            raise ValueError("the gradient table is a CUDA int64 tensor of nlayers pointers")
        N.check(N.lags_bucket_set_grad_table(self._h, table.data_ptr() if table is not None else None),
                "lags_bucket_set_grad_table")
        self._grad_table = table  # keep it alive while the library holds the pointer

    def decode(self, msgs: torch.Tensor, P: int, v: torch.Tensor, momentum: torch.Tensor | None = None,
               mu: float = 0.0, stream=None, msg_stride: int | None = None) -> None:
        """Rank-ordered fp64 decode of P messages and v <- v - total/P (or heavy-ball momentum).
        A float64 ``v`` with a float32 bucket keeps the unrounded fp64 result (LAGS_DECODE_V64)."""
        stride = self.msg_bytes if msg_stride is None else int(msg_stride)
        if msgs.numel() < (P - 1) * stride + self.msg_bytes:
            raise ValueError("message buffer smaller than P messages")
        v64 = v.dtype == torch.float64 and storage_dtype(self.mode) != torch.float64
        if (v.dtype != storage_dtype(self.mode) and not v64) or v.numel() < self.n_total:
            raise ValueError("parameter buffer does not match the bucket")
        N.check(N.lags_bucket_decode_update(self._h, msgs.data_ptr(), stride, int(P), v.data_ptr(),
                                            momentum.data_ptr() if momentum is not None else None, float(mu),
                                            N.DECODE_V64 if v64 else 0, stream_handle(stream)),
                "lags_bucket_decode_update")

    # -- diagnostics (R: analysis.py:24-56, training.py:320-337) ---------------------------------
    def reconstruct(self, msgs: torch.Tensor, P: int, r: torch.Tensor, acc: torch.Tensor, stream=None,
                    msg_stride: int | None = None, plane_stride: int | None = None) -> None:
        """acc_p = r_p with message p's pairs written back: the accumulated vectors of P workers
        (P planes of ``plane_stride`` elements, default n_total)."""
        stride = self.n_total if plane_stride is None else int(plane_stride)
        ms = self.msg_bytes if msg_stride is None else int(msg_stride)
        if r.dtype != storage_dtype(self.mode) or acc.dtype != r.dtype:
            raise TypeError("r / acc must have the bucket's storage dtype")
        if min(r.numel(), acc.numel()) < (P - 1) * stride + self.n_total or msgs.numel() < (P - 1) * ms + self.msg_bytes:
            raise ValueError("buffers smaller than P planes / messages")
        N.check(N.lags_bucket_reconstruct(self._h, msgs.data_ptr(), ms, int(P), r.data_ptr(), acc.data_ptr(), stride,
                                          stream_handle(stream)), "lags_bucket_reconstruct")

    def delta(self, acc: torch.Tensor, r: torch.Tensor, P: int, out: torch.Tensor | None = None, stream=None,
              plane_stride: int | None = None) -> torch.Tensor:
        """Per-layer aggregation-quality ratio delta^(l) of P workers (float64 device tensor, NaN
        where the reference returns None).  acc / r: P accumulated / residual planes."""
        stride = self.n_total if plane_stride is None else int(plane_stride)
        if r.dtype != storage_dtype(self.mode) or acc.dtype != r.dtype:
            raise TypeError("r / acc must have the bucket's storage dtype")
        if min(r.numel(), acc.numel()) < (P - 1) * stride + self.n_total:
            raise ValueError("buffers smaller than P planes")
        out = torch.empty(self.nlayers, dtype=torch.float64, device=self.device) if out is None else out
        N.check(N.lags_bucket_delta(self._h, acc.data_ptr(), r.data_ptr(), stride, int(P), out.data_ptr(),
                                    stream_handle(stream)), "lags_bucket_delta")
        return out

    # -- residual-identity monitor (R: training.py:197-200, 356-369) -----------------------------
    def shadow_step(self, g_sum: torch.Tensor, x: torch.Tensor, alpha: float, P: int, stream=None) -> None:
        """Dense shadow sequence: x -= (alpha * g_sum) / P in float64 (g_sum: the workers' summed
        gradient in the storage dtype)."""
        if x.dtype != torch.float64 or x.numel() < self.n_total or g_sum.dtype != storage_dtype(self.mode):
            raise TypeError("shadow_step: x float64 and g_sum in the bucket's storage dtype")
        N.check(N.lags_bucket_shadow_step(self._h, g_sum.data_ptr(), x.data_ptr(), float(alpha), int(P),
                                          stream_handle(stream)), "lags_bucket_shadow_step")

    def identity(self, v: torch.Tensor, x: torch.Tensor, r_sum: torch.Tensor, P: int, out: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
        """[||mean residual of layer j||^2 per layer, ||v - x||^2, max |(v - x) - r_sum / P|] (float64
        device tensor of nlayers + 2)."""
        out = torch.empty(self.nlayers + 2, dtype=torch.float64, device=self.device) if out is None else out
        N.check(N.lags_bucket_identity(self._h, v.data_ptr(), x.data_ptr(), r_sum.data_ptr(), int(P), out.data_ptr(),
                                       stream_handle(stream)), "lags_bucket_identity")
        return out

    # -- sparse wire format (R: sparsify.py:260-310) -------------------------------------------
    def _wire_tables(self, layer_ids):
        if getattr(self, "_wire", None) is None or self._wire[0] != tuple(layer_ids):
            from . import wire as W

            self._wire = (tuple(layer_ids), W._u32(layer_ids, self.device), W._u32(self.dims, self.device),
                          torch.tensor(self.slots, dtype=torch.int64, device=self.device),
                          torch.tensor(self.ks, dtype=torch.int32, device=self.device))
        return self._wire[1:]

    def wire_capacity(self) -> int:
        """Largest encoded message of this bucket (every layer at its full k)."""
        return 4 + sum(12 + 12 * k for k in self.ks)

    def encode_wire(self, msg: torch.Tensor, layer_ids=None, stream=None):
        """One message of this bucket in the reference's wire format, on the device (chunk j =
        layer j with id ``layer_ids[j]``, default 1..L).  Returns (wire uint8 [capacity],
        length int64 [1], error int64 [1]); stream-ordered, no host synchronisation."""
        from . import wire as W

        ids = list(layer_ids) if layer_ids is not None else list(range(1, self.nlayers + 1))
        lids, dims, first, _ = self._wire_tables(ids)
        return W.encode_table(lids, dims, self.counts_view(msg), first, self.idx_view(msg), self.val_view(msg),
                              W.MESSAGE, self.wire_capacity(), stream)

    def decode_wire(self, wire: torch.Tensor, length: int, layer_ids=None, msg: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
        """Inverse of encode_wire into a bucket message (synchronises to check the result).  The
        chunks must be this bucket's layers in order (ids, dims) with counts <= k."""
        from . import wire as W

        ids = list(layer_ids) if layer_ids is not None else list(range(1, self.nlayers + 1))
        lids, dims, first, caps = self._wire_tables(ids)
        msg = self.new_messages(1) if msg is None else msg
        out = W.decode_table(wire, int(length), mode=W.MESSAGE, max_chunks=self.nlayers, first=first, caps=caps,
                             entry_capacity=self.total_k, idx=self.idx_view(msg), val=self.val_view(msg),
                             stream=stream)
        W.raise_for(W.error_word(out["error"]), int(out["end"].item()), int(length))
        n = int(out["nchunks"].item())
        if n != self.nlayers or not torch.equal(out["layer_ids"], lids) or not torch.equal(out["dims"], dims):
            raise StructureError("wire message does not hold this bucket's layers in order")
        self.counts_view(msg).copy_(out["counts"])
        return msg

    # -- host helpers (tests / diagnostics) ----------------------------------------------------
    def set_probe_events(self, before, after) -> None:
        """Record these torch.cuda.Events around the streaming kernel K1 of every fp32 compress
        (None, None to stop)."""
        self._probes = (before, after)  # keep them alive while the library holds the handles
        N.check(N.lags_bucket_set_probe_events(self._h, before.cuda_event if before is not None else None,
                                               after.cuda_event if after is not None else None))

    def stats(self, stream=None) -> np.ndarray:
        """Per-layer [threshold key, fallbacks, last candidates, calls, cycles, path, phase cycles,
        t_start, t_end, t_launch (globaltimer ns, low 32 bits), 0] (synchronous)."""
        out = np.zeros((self.nlayers, 12), dtype=np.uint32)
        N.check(N.lags_bucket_stats(self._h, out.ctypes.data, stream_handle(stream)))
        return out

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
