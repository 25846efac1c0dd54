"""Drop-in ``lags_step`` (R: training.py:227-255) backed by the B200 kernels.

Same signature, semantics and errors as the reference: residuals are updated
in place, a new layered vector of ``type(v)`` is returned, ``StructureError``
on a layout mismatch and ``DivergenceError(iteration=t)`` on a non-finite
gradient (R: training.py:170-175).  It can be monkeypatched into the
reference's ``train()`` (R: training.py:348 looks ``lags_step`` up at call time).

Host numpy buffers are copied to the device, the P simulated workers are
compressed one after another into P sparse messages (the exchange), the
messages are decoded in rank order, and the results are copied back.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .engine import Bucket
from .errors import DivergenceError, StructureError
from .layered import layout_of

SCHEDULE_KINDS = ("constant", "inv-sqrt-T", "diminishing")


@dataclass(frozen=True)
class StepSizeSchedule:
    """alpha_t (R: training.py:41-69); inv-sqrt-T returns np.float64 exactly like the reference."""

    kind: str
    theta: float

    def __post_init__(self):
        if self.kind not in SCHEDULE_KINDS:
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if self.theta <= 0:
            raise ValueError("theta must be positive")

    def alpha(self, t: int, total: int):
        if self.kind == "constant":
            return self.theta
        if self.kind == "inv-sqrt-T":
            return self.theta / np.sqrt(total)
        return self.theta / (1.0 + t)


def mode_for(dtype, alpha) -> int:
    """numpy NEP 50 promotion of ``res + alpha * g`` (R: training.py:250) -> lags_dtype_t."""
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return N.F64
    if dtype == np.float32:
        if isinstance(alpha, np.floating) and np.dtype(type(alpha)).itemsize > 4:
            return N.F32_ACC64
        return N.F32
    raise TypeError(f"unsupported dtype {dtype}; the B200 path handles float32 and float64")


_BUCKETS: dict = {}


def _bucket_for(dims: tuple, ks: tuple, mode: int, world: int) -> Bucket:
    key = (dims, ks, mode, world, torch.cuda.current_device())
    b = _BUCKETS.get(key)
    if b is None:
        if len(_BUCKETS) > 16:
            _BUCKETS.clear()
        b = Bucket(dims, ks, mode, max_world=world)
        _BUCKETS[key] = b
    return b


def _to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=False)


class HostPinner:
    """DMA-friendly host buffers for the drop-in's numpy arguments.

    Arrays seen a second time (residuals updated in place, reused gradient buffers) are
    page-locked in place with cudaHostRegister (bounded LRU, the array is kept alive while
    registered); first-seen arrays go through pinned staging; results are returned in pinned
    memory so passing them back next step is a direct DMA.
    """

    def __init__(self, max_bytes: int = 16 << 30, max_entries: int = 64):
        self.max_bytes, self.max_entries = max_bytes, max_entries
        self.registered: "OrderedDict[tuple, np.ndarray]" = OrderedDict()
        self.seen: "OrderedDict[tuple, bool]" = OrderedDict()
        self.bytes = 0

    def pinned(self, arr: np.ndarray) -> bool:
        if not arr.flags.c_contiguous or arr.nbytes == 0:
            return False
        key = (arr.ctypes.data, arr.nbytes)
        if key in self.registered:
            self.registered.move_to_end(key)
            return True
        t = torch.from_numpy(arr)
        if t.is_pinned():
            return True
        if key not in self.seen:
            self.seen[key] = True
            if len(self.seen) > 4 * self.max_entries:
                self.seen.popitem(last=False)
            return False
        while self.registered and (self.bytes + arr.nbytes > self.max_bytes or len(self.registered) >= self.max_entries):
            (ptr, nb), _ = self.registered.popitem(last=False)
            torch._C._cudart.cudaHostUnregister(ptr)
            self.bytes -= nb
        if int(torch._C._cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)) != 0:
            return False
        self.registered[key] = arr
        self.bytes += arr.nbytes
        return True

    def h2d(self, arr: np.ndarray, device) -> torch.Tensor:
        arr = np.ascontiguousarray(arr)
        t = torch.from_numpy(arr)
        if not self.pinned(arr):
            st = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            st.copy_(t)
            t = st
        return t.to(device, non_blocking=True)

    def d2h_into(self, arr: np.ndarray, src: torch.Tensor):
        """Copy src into the numpy array; returns a finisher to call after synchronising."""
        if self.pinned(arr):
            torch.from_numpy(arr).copy_(src, non_blocking=True)
            return lambda: None
        st = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        st.copy_(src, non_blocking=True)
        return lambda: np.copyto(arr, st.numpy())


_PINNER = HostPinner()


def slgs_step(v, grads: Sequence, alpha, global_k: int, residuals: Sequence, t: int | None = None):
    """Single-layer (whole stacked vector) selection with error feedback -- R: training.py:203-224.

    The same kernels with one "layer" spanning the flat vector: R: training.py:216-217 checks k
    against the full dimension, selection and aggregation are then lags_step's with L = 1.
    """
    from .layered import LayerShape

    dim = int(v.data.shape[0])
    if not 1 <= global_k <= dim:
        raise ValueError(f"global_k={global_k} outside 1..{dim}")

    class _Flat:  # the stacked vector seen as one layer (views, no copies)
        def __init__(self, shape, data):
            self.shape = shape
            self.data = data

    one = (LayerShape(1, dim),)
    for p, g in enumerate(grads, start=1):  # layout check against the real layer split first
        if layout_of(g) != layout_of(v):
            return lags_step(v, grads, alpha, {ls.layer_id: 1 for ls in v.shape}, residuals, t)
    flat_res = [_Flat(one, r.data) for r in residuals]
    out = lags_step(_Flat(one, v.data), [_Flat(one, g.data) for g in grads], alpha, {1: int(global_k)}, flat_res, t,
                    _promote_v=True)
    return type(v)(v.shape, out.data)


def lags_step(v, grads: Sequence, alpha, counts: dict, residuals: Sequence, t: int | None = None, *,
              _promote_v: bool = False):
    """Per-layer selection with error feedback on the B200; R: training.py:227-255.

    (_promote_v: return float32 parameters as the unrounded float64 ``v - total / P``, which is
    what the reference's slgs_step does, R: training.py:224.)"""
    pairs = layout_of(v)
    P = len(grads)
    if P < 1 or len(residuals) != P:
        raise ValueError("need one residual per worker and at least one worker")
    dtype = v.data.dtype
    mode = mode_for(dtype, alpha)
    # R: training.py:171-175 -- worker by worker: layout, then finiteness.
    bad_layout = next((p for p, g in enumerate(grads, start=1) if layout_of(g) != pairs), None)
    status = torch.zeros(max(P, 1), dtype=torch.int32, device="cuda")
    if bad_layout is not None:
        for p in range(1, bad_layout):
            gd = _to_dev(grads[p - 1].data)
            N.check(N.lags_check_finite(N.F64 if gd.dtype == torch.float64 else N.F32, gd.data_ptr(), gd.numel(),
                                        status[p - 1:p].data_ptr(), torch.cuda.current_stream().cuda_stream))
        st = status.cpu().numpy()
        for p in range(1, bad_layout):
            if st[p - 1]:
                raise DivergenceError(f"worker {p} produced a non-finite gradient", iteration=t)
        raise StructureError(f"worker {bad_layout} gradient layout differs from params")
    for g, r in zip(grads, residuals):
        if g.data.dtype != dtype or r.data.dtype != dtype:
            raise TypeError("params, gradients and residuals must share one dtype")
        if layout_of(r) != pairs:
            raise StructureError("residual layout differs from params")
    dims = tuple(d for _, d in pairs)
    ks = []
    for lid, d in pairs:
        k = int(counts[lid])
        if not 1 <= k <= d:  # R: sparsify.py:82-83 (raised before any residual is touched)
            raise ValueError(f"k={k} outside 1..{d}")
        ks.append(k)
    bucket = _bucket_for(dims, tuple(ks), mode, P)

    dev = torch.device("cuda", torch.cuda.current_device())
    pin = _PINNER
    v_d = pin.h2d(v.data, dev)
    if _promote_v and v_d.dtype == torch.float32:
        v_d = v_d.double()
    msgs = bucket.new_messages(P)
    r_devs = []
    fused = P == 1 and mode == N.F32 and v_d.dtype == torch.float32
    for p in range(P):
        g_d = pin.h2d(grads[p].data, dev)
        r_d = pin.h2d(residuals[p].data, dev)
        msg_p = msgs[p * bucket.msg_bytes:(p + 1) * bucket.msg_bytes]
        if fused:  # one worker: the update is fused into the selection epilogue
            bucket.step_local(g_d, r_d, alpha, v_d, msg_p, status[p:p + 1])
        else:
            bucket.compress(g_d, r_d, alpha, msg_p, status[p:p + 1])
        r_devs.append(r_d)
    if not fused:
        bucket.decode(msgs, P, v_d)
    out = torch.empty(v_d.shape, dtype=v_d.dtype, pin_memory=True)
    out.copy_(v_d, non_blocking=True)
    st = status.cpu().numpy()  # synchronises: inputs copied, compress + decode done
    for p in range(P):
        if st[p] & N.STATUS_NONFINITE:  # residuals untouched on the host, as in the reference
            raise DivergenceError(f"worker {p + 1} produced a non-finite gradient", iteration=t)
    finish = [pin.d2h_into(res.data, r_d) for r_d, res in zip(r_devs, residuals)]
    torch.cuda.current_stream(dev).synchronize()
    for f in finish:
        f()
    return type(v)(v.shape, out.numpy())
