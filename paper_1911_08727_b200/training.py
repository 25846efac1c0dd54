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

import os
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
MAX_WORKERS = 32  # workers one decode combines (lags_bucket_create: max_world <= 32)


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
        if len(_BUCKETS) > 64:
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

    def source(self, arr: np.ndarray) -> torch.Tensor:
        """A pinned CPU tensor holding arr's data (arr itself when page-locked, else a staged copy)."""
        arr = np.ascontiguousarray(arr).reshape(-1)
        t = torch.from_numpy(arr)
        if self.pinned(arr):
            return t
        st = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        st.copy_(t)
        return st

    def dest(self, arr: np.ndarray, finish: list) -> torch.Tensor:
        """A pinned CPU tensor to copy results into for arr (arr itself when page-locked; else a
        staging buffer whose contents a finisher appended to ``finish`` copies into arr)."""
        flat = arr.reshape(-1)
        if arr.flags.c_contiguous and self.pinned(arr):
            return torch.from_numpy(flat)
        st = torch.empty(flat.shape, dtype=torch.from_numpy(flat[:0]).dtype, pin_memory=True)
        finish.append(lambda: np.copyto(flat, st.numpy()))
        return st

    def d2h_into(self, arr: np.ndarray, src: torch.Tensor):
        """Copy src into the numpy array; returns a finisher to call after synchronising."""
        if self.pinned(arr):
            torch.from_numpy(arr).copy_(src, non_blocking=True)
            return lambda: None
        st = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        st.copy_(src, non_blocking=True)
        return lambda: np.copyto(arr, st.numpy())


_PINNER = HostPinner()


_CHUNK_ELEMS = 4 << 20  # ~16 MB of fp32 per pipeline stage
_STREAMS: dict = {}


def _chunk_plan(dims: tuple) -> list:
    """Consecutive layer ranges of about _CHUNK_ELEMS elements: (lo, hi_exclusive, elem_lo, elem_hi)."""
    out, lo, acc, e0 = [], 0, 0, 0
    for j, d in enumerate(dims):
        acc += d
        if acc - e0 >= _CHUNK_ELEMS or j == len(dims) - 1:
            out.append((lo, j + 1, e0, acc))
            lo, e0 = j + 1, acc
    return out


def _streams(dev):
    key = dev.index
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(dev) for _ in range(3))  # h2d, compute, d2h
    return _STREAMS[key]


_COPY_POOL = None
_COPY_THREADS = 8  # host threads copying v into the pinned output of the drop-in step
# diagnostics: set to a list to collect (phase, time.perf_counter()) marks of _pipelined_step
PIPELINE_TRACE = None


def _mark(label: str) -> None:
    if PIPELINE_TRACE is not None:
        import time

        PIPELINE_TRACE.append((label, time.perf_counter()))


def _host_copy(dst: np.ndarray, src: np.ndarray, plan: list) -> list:
    """dst[:] = src (with dtype conversion) on host threads, chunk by chunk of ``plan`` in order;
    returns one joiner per chunk."""
    global _COPY_POOL
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=min(_COPY_THREADS, os.cpu_count() or 1))
    joins = []
    for (_, _, e0, e1) in plan:
        parts = max(1, min(4, (e1 - e0) // (1 << 20)))
        bounds = [e0 + (e1 - e0) * i // parts for i in range(parts + 1)]
        futs = [_COPY_POOL.submit(np.copyto, dst[a:b], src[a:b], "unsafe") for a, b in zip(bounds, bounds[1:])]
        joins.append(lambda futs=futs: [f.result() for f in futs])
    return joins


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """out = every rank's inp in rank order.  NCCL gathers the device tensors directly; other
    backends (gloo: e.g. several worker processes sharing one GPU) go through host copies."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    host = torch.empty(out.shape, dtype=out.dtype)
    dist.all_gather_into_tensor(host, inp.cpu(), group=group)
    out.copy_(host, non_blocking=False)


def _pipelined_step(v, grads, residuals, alpha, dims, ks, mode, t, promote_v, group=None):
    """The drop-in step with its host transfers overlapped, chunk by chunk of layers.

    PCIe carries only what must cross it: the gradients and residuals up, the new residuals down
    (R: training.py:252 updates them in place).  The new parameters differ from v only at the
    selected entries, so v never crosses the link: host threads copy v into the (pinned) output
    while the GPU works, and the decode then updates the selected entries of that output in place
    through its device mapping (pinned host memory is device-addressable under UVA).
    Order (R: training.py:174-175): every gradient goes up and is checked for finiteness before
    any residual is written back; residual chunks stream up behind the gradients, each chunk's
    compress runs as soon as it has arrived, and its new residual streams back on a third stream
    while later chunks still upload (the copy engines run both directions at once).

    With a process group this process is ONE worker (``grads``/``residuals`` hold its own): the
    finiteness flags of all workers are all-gathered before any residual is written back, and each
    chunk's fixed-size message is all-gathered over NCCL before the rank-ordered decode, so every
    rank computes the same new parameters as the single-process P-worker step."""
    _mark("start")
    P = len(grads)
    world, me = 1, 0
    if group is not None:
        import torch.distributed as dist

        world, me = dist.get_world_size(group), dist.get_rank(group)
        if P != 1:
            raise ValueError("with a process group each rank passes exactly its own gradient and residual")
    dev = torch.device("cuda", torch.cuda.current_device())
    s_up, s_cmp, s_down = _streams(dev)
    cur = torch.cuda.current_stream(dev)
    for s in (s_up, s_cmp, s_down):
        s.wait_stream(cur)
    pin = _PINNER
    plan = _chunk_plan(dims)
    out_dtype = np.float64 if promote_v else v.dtype
    out = torch.empty(v.shape, dtype=torch.from_numpy(np.empty(0, out_dtype)).dtype, pin_memory=True)
    join_copy = _host_copy(out.numpy(), v.reshape(-1), plan)  # per chunk; overlaps everything below
    g_src = [pin.source(g) for g in grads]
    r_src = [pin.source(r) for r in residuals]
    with torch.cuda.stream(s_up):
        g_dev = [[torch.empty(e1 - e0, dtype=g.dtype, device=dev) for (_, _, e0, e1) in plan] for g in g_src]
        for p in range(P):
            for (_, _, e0, e1), gd in zip(plan, g_dev[p]):
                gd.copy_(g_src[p][e0:e1], non_blocking=True)
        ev_g = torch.cuda.Event()
        ev_g.record(s_up)
        r_dev, ev_in = [], []
        for (_, _, e0, e1) in plan:
            r_dev.append([r_src[p][e0:e1].to(dev, non_blocking=True) for p in range(P)])
            e = torch.cuda.Event()
            e.record(s_up)
            ev_in.append(e)
    with torch.cuda.stream(s_cmp):
        s_cmp.wait_event(ev_g)
        pre = torch.zeros(P, dtype=torch.int32, device=dev)
        for p in range(P):
            for gd in g_dev[p]:
                N.check(N.lags_check_finite(N.F64 if gd.dtype == torch.float64 else N.F32, gd.data_ptr(), gd.numel(),
                                            pre[p:p + 1].data_ptr(), s_cmp.cuda_stream), "lags_check_finite")
        if world > 1:  # every worker's flags, in rank order (R: training.py:174-175 names the first)
            pre_all = torch.empty(world, dtype=torch.int32, device=dev)
            _all_gather(pre_all, pre, group)
            pre = pre_all
        pre_h = torch.empty(world * P, dtype=torch.int32, pin_memory=True)
        pre_h.copy_(pre, non_blocking=True)
        ev_pre = torch.cuda.Event()
        ev_pre.record(s_cmp)
        # every chunk's compress is queued now (it writes device buffers only), so it runs the
        # moment the chunk has arrived, whatever the host is doing
        status = torch.zeros(P, dtype=torch.int32, device=dev)
        staged = []
        for c, (lo, hi, e0, e1) in enumerate(plan):
            bucket = _bucket_for(dims[lo:hi], ks[lo:hi], mode, world * P)
            s_cmp.wait_event(ev_in[c])
            msgs = bucket.new_messages(P)
            for p in range(P):
                bucket.compress(g_dev[p][c], r_dev[c][p], alpha, msgs[p * bucket.msg_bytes:(p + 1) * bucket.msg_bytes],
                                status[p:p + 1], stream=s_cmp)
            done = torch.cuda.Event()
            done.record(s_cmp)
            staged.append((bucket, msgs, e0, e1, done))
    _mark("uploads and compress enqueued")
    ev_pre.synchronize()
    _mark("gradients checked")
    bad = [p for p in range(world * P) if pre_h[p] & N.STATUS_NONFINITE]
    if bad:  # R: training.py:174-175 -- raised before any residual is written back
        for j in join_copy:
            j()
        for s in (s_up, s_cmp, s_down):
            s.synchronize()
        raise DivergenceError(f"worker {bad[0] + 1} produced a non-finite gradient", iteration=t)
    finish = []
    r_dst = [pin.dest(r, finish) for r in residuals]
    with torch.cuda.stream(s_down):  # new residuals back, chunk by chunk as they are computed
        for c, (_, _, e0, e1, done) in enumerate(staged):
            s_down.wait_event(done)
            for p in range(P):
                r_dst[p][e0:e1].copy_(r_dev[c][p], non_blocking=True)
    with torch.cuda.stream(s_cmp):
        for c, (bucket, msgs, e0, e1, _) in enumerate(staged):
            if world > 1:  # every worker's message for this chunk, rank order
                allm = bucket.new_messages(world)
                _all_gather(allm, msgs, group)
                msgs = allm
            join_copy[c]()  # this chunk of the output holds v: update its selected entries in place
            bucket.decode(msgs, world * P, out[e0:e1], stream=s_cmp)
    _mark("chunks enqueued")
    s_cmp.synchronize()
    _mark("decode done")
    s_down.synchronize()
    _mark("residuals down")
    for f in finish:
        f()
    cur.wait_stream(s_down)
    return out


def slgs_step(v, grads: Sequence, alpha, global_k: int, residuals: Sequence, t: int | None = None, *,
              group=None):
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
            return lags_step(v, grads, alpha, {ls.layer_id: 1 for ls in v.shape}, residuals, t, group=group)
    flat_res = [_Flat(one, r.data) for r in residuals]
    out = lags_step(_Flat(one, v.data), [_Flat(one, g.data) for g in grads], alpha, {1: int(global_k)}, flat_res, t,
                    group=group, _promote_v=True)
    return type(v)(v.shape, out.data)


def lags_step(v, grads: Sequence, alpha, counts: dict, residuals: Sequence, t: int | None = None, *,
              group=None, _promote_v: bool = False):
    """Per-layer selection with error feedback on the B200; R: training.py:227-255.

    ``group`` (a torch.distributed process group; NCCL, or gloo for workers sharing a GPU): run as
    one worker of a multi-process job --
    ``grads``/``residuals`` hold this rank's own single gradient and residual, ``v`` the replica;
    the workers are the ranks in group order, and every rank returns the parameters the
    single-process step over all of their gradients would return (same bits).

    (_promote_v: return float32 parameters as the unrounded float64 ``v - total / P``, which is
    what the reference's slgs_step does, R: training.py:224.)"""
    pairs = layout_of(v)
    P = len(grads)
    if P < 1 or len(residuals) != P:
        raise ValueError("need one residual per worker and at least one worker")
    workers = P
    if group is not None:
        import torch.distributed as dist

        workers = P * dist.get_world_size(group)
    if workers > MAX_WORKERS:  # the decode's per-element rank bitmask is 32 bits
        raise ValueError(f"at most {MAX_WORKERS} workers per step, got {workers}")
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
    out = _pipelined_step(v.data, [g.data for g in grads], [r.data for r in residuals], alpha, dims, tuple(ks),
                          mode, t, _promote_v, group)
    return type(v)(v.shape, out.numpy())
