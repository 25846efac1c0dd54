"""LagsSGD: layer-wise adaptive gradient sparsification as a torch optimizer on real ranks.

The reference simulates P workers in one process (R: training.py:227-255) and only *models*
the overlap of communication with backprop (R: perf.py:173-195).  Here every rank is a GPU:

* parameters, gradients and the error-feedback residual live in flat per-rank buffers with the
  reference's layer layout (R: layered.py:46-107); ``p.data`` / ``p.grad`` are views into them;
* layers are grouped into fusion buckets in backprop order with the reference's flush rule
  (R: sparsify.py:209-238), using the fixed k_l-slot message of each layer as the chunk size;
* a ``post_accumulate_grad`` hook marks a parameter ready; when a bucket is complete its compress
  (residual add + per-layer exact top-k + residual zeroing + fused zero_grad) is launched on a
  compute-side stream, and its exchange of the fixed-size sparse messages (the peer-memory push over
  NVLink, or the NCCL all-gather) plus the rank-ordered fp64 decode + SGD (or momentum) update of
  the bucket's weights on a separate communication stream: the reference's two resources, compute
  (backprop + sparsify) and one serial network channel in release order (R: perf.py:173-195).
  Buckets launch in release order on every rank, so layer l's exchange overlaps the backprop of
  layers < l, and bucket l+1's compress never queues behind bucket l's exchange;
* ``step()`` launches buckets whose hooks never fired, then makes the compute stream wait for both
  streams (the next forward trails the last arrival, R: perf.py:194).

Numerics per layer and rank are exactly ``lags_step``'s (fp32 storage, lr absorbed into the
residual as in R: training.py:250): selection bit-exact, aggregation in fp64 in rank order.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

import torch
import torch.distributed as dist

from contextlib import nullcontext as _nullctx

from .errors import DivergenceError
from .sparsify import CompressionPolicy

CHUNK_HEADER_BYTES = 8  # R: sparsify.py:23 (accounting header of a chunk)
MAX_WORLD = 32  # ranks one decode can combine (lags_bucket_create: max_world <= 32)
INDEX_BYTES = 4


def selection_counts(dims: Sequence[int], ratios: Sequence[float]) -> list[int]:
    """k_l = min(d, max(1, floor(d / c_l))) -- R: sparsify.py:182-184."""
    return [min(d, max(1, int(d // c))) for d, c in zip(dims, ratios)]


def plan_buckets(dims: Sequence[int], ks: Sequence[int], capacity_bytes: int, value_width: int = 4):
    """Fusion buckets in backprop order (layer L first), by the reference's rule
    (R: sparsify.py:209-238): chunks accumulate until their accounted bytes reach the capacity or
    the first layer has been produced; chunks are never split or reordered.  A chunk that alone
    reaches the capacity travels alone (the reference's fusion_flush rejects it; a runtime must
    still ship it).  Chunk bytes = 8 + k_l * (4 + value_width) with the fixed k_l-slot message.
    Returns inclusive 0-based layer ranges (lo, hi) in release order."""
    if capacity_bytes <= 0:
        raise ValueError("capacity_bytes must be positive")
    out, pending, total = [], [], 0
    for l in range(len(dims) - 1, -1, -1):
        size = CHUNK_HEADER_BYTES + ks[l] * (INDEX_BYTES + value_width)
        if size >= capacity_bytes:
            if pending:
                out.append((min(pending), max(pending)))
                pending, total = [], 0
            out.append((l, l))
            continue
        pending.append(l)
        total += size
        if total >= capacity_bytes or l == 0:
            out.append((min(pending), max(pending)))
            pending, total = [], 0
    return out


@dataclass
class _BucketRT:
    lo: int
    hi: int
    offset: int
    numel: int
    engine: object
    msg_local: torch.Tensor
    msg_all: torch.Tensor | None
    gtab: torch.Tensor | None = None   # grads="tensors": device table of per-layer gradient pointers
    ring: list | None = None           # pinned host staging slots for the table, with their events
    slot: int = 0
    peer: object = None                # exchange="p2p": the bucket's PeerExchange
    ready: object = None               # event: the bucket's compress has been issued on the side stream


_RING = 4  # host staging slots per bucket (a slot is reused only after its copy has completed)


class LagsSGD(torch.optim.Optimizer):
    """Sparsified data-parallel SGD with per-layer density rho_l and error feedback.

    Args:
        params: parameters in layer order (layer ids 1..L, backprop visits L..1).
        lr: step size alpha (absorbed into the residual: acc = r + lr * g).
        rho: uniform density (c = 1/rho), or ``policy`` (a CompressionPolicy over layer ids 1..L).
        momentum: heavy-ball factor applied to the decoded update (0 = the reference's plain SGD).
        process_group: torch.distributed group (default: WORLD if initialised, else single rank).
        bucket_cap_bytes: fusion capacity of the reference's flush rule.
        engine_factory: builds a bucket engine (default: the CUDA ``Bucket``); tests inject stubs.
        check_every: read the non-finite flag back every this many steps (DivergenceError).
    """

    def __init__(self, params: Iterable[torch.nn.Parameter], lr: float, rho: float | None = None,
                 policy: CompressionPolicy | None = None, momentum: float = 0.0, process_group=None,
                 bucket_cap_bytes: int = 1 << 20, engine_factory: Callable | None = None, check_every: int = 1,
                 exchange: bool | str = True, delta_every: int = 0, grads: str = "auto", monitor_every: int = 0):
        params = [p for p in params]
        if not params:
            raise ValueError("no parameters")
        if (rho is None) == (policy is None):
            raise ValueError("give exactly one of rho or policy")
        super().__init__(params, dict(lr=lr, momentum=momentum))
        self.params = params
        self.device = params[0].device
        self.dims = [p.numel() for p in params]
        L = len(params)
        if policy is None:
            policy = CompressionPolicy({i + 1: 1.0 / rho for i in range(L)}, 1.0 / rho)
        self.policy = policy
        self.ratios = [policy.ratio_for(i + 1) for i in range(L)]
        self.ks = selection_counts(self.dims, self.ratios)
        self.group = process_group
        self.world = dist.get_world_size(process_group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(process_group) if self.world > 1 else 0
        if self.world > MAX_WORLD:
            raise ValueError(f"LagsSGD exchanges among at most {MAX_WORLD} ranks (the decode's rank bitmask is "
                             f"32 bits), got {self.world}")
        self.check_every = max(1, int(check_every))
        self.mu = float(momentum)
        # exchange: "nccl" (all-gather; True), "p2p" (peer-memory push over CUDA IPC / NVLink, one
        # receive area per bucket), or False: a local no-op (decode of the own message only) -- a
        # measurement mode for the exposed-communication time, not a training mode
        if exchange is True:
            exchange = "nccl"
        # "fused": the peer-memory exchange done by the selection itself (every finished layer is
        # stored into every rank's receive area by the CTA that selected it), then only the wait
        if exchange not in (False, "nccl", "p2p", "fused"):
            raise ValueError(f"exchange must be True, False, 'nccl', 'p2p' or 'fused', got {exchange!r}")
        self.exchange = exchange is not False
        self.exchange_mode = exchange if self.world > 1 and exchange else None
        # delta_every > 0: every that many steps, log the aggregation-quality ratio delta^(l) of
        # every layer on the device (R: training.py:320-337, delta_log_every); it all-gathers the
        # residuals once per logged step (dense traffic, diagnostics only)
        self.delta_every = int(delta_every)
        # monitor_every > 0: the residual-identity monitor of R: training.py:356-369 -- a dense fp64
        # shadow sequence x advanced every step with the workers' mean gradient (R: training.py:197-200;
        # a dense all-reduce of each bucket's gradient at N > 1: a diagnostic mode), and every that
        # many steps ||v - x||, max |(v - x) - mean residual| and the per-layer mean-residual norms
        self.monitor_every = int(monitor_every)
        self.shadow = None
        self._identity = None
        if engine_factory is None:
            from . import _native as N
            from .engine import Bucket

            def engine_factory(dims, ks, world, device):
                return Bucket(dims, ks, N.F32, device=device, max_world=world)

        # gradients: "flat" -- p.grad are views of one flat buffer that autograd accumulates into
        # and the compress clears; "tensors" -- autograd's own per-parameter tensors, read by the
        # compress through a device pointer table and released afterwards (no accumulate kernels,
        # no flat gradient buffer).  "auto" = tensors when the engine supports the table.
        if grads not in ("auto", "flat", "tensors"):
            raise ValueError(f"grads must be 'auto', 'flat' or 'tensors', got {grads!r}")
        if grads == "auto":
            probe = engine_factory([4], [1], 1, self.device)
            grads = "tensors" if hasattr(probe, "set_grad_table") and self.device.type == "cuda" else "flat"
            del probe
        self.grads_mode = grads
        # flat per-rank buffers with the reference's layer layout (R: layered.py:46-107) -- layers
        # back to back inside a fusion bucket, every bucket starting 16-byte aligned (so the
        # streaming pass takes its vector path); params (and flat grads) are views
        for p in params:
            if p.dtype != torch.float32:
                raise TypeError("LagsSGD keeps fp32 parameters")
        self.engine_factory = engine_factory
        self.bucket_cap_bytes = int(bucket_cap_bytes)
        self.flat_param = self.flat_grad = self.residual = self.momentum_buf = None
        self.offsets = None
        # high priority: a released bucket's compress (many short K1 CTAs) is scheduled ahead of the
        # remaining backprop kernels instead of interleaving with them for milliseconds
        self.side = (torch.cuda.Stream(self.device, priority=-1) if self.device.type == "cuda" else None)  # compress
        self.comm = (torch.cuda.Stream(self.device, priority=-1) if self.device.type == "cuda" else None)  # exchange + decode
        self.buckets = []
        self._relayout(plan_buckets(self.dims, self.ks, self.bucket_cap_bytes))
        if self.world > 1:  # identical starting point on every rank (no DDP: it would double-communicate)
            dist.broadcast(self.flat_param, group=process_group, group_src=0)
        if self.monitor_every > 0:
            self.shadow = self.flat_param.double()  # x_0 = v_0 (R: training.py:278)
        self._build_buckets()
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._status_host = torch.zeros(1, dtype=torch.int32, pin_memory=self.device.type == "cuda")
        self._status_event = None
        self._status_step = 0
        self._steps = 0
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in params]
        self._layer_of_param = {id(p): l for l, p in enumerate(params)}
        self.timing = None  # optional per-bucket CUDA events (see enable_timing)
        self._delta = torch.full((L,), float("nan"), dtype=torch.float64, device=self.device)
        self._delta_step = 0
        self._hook_events = None  # optional per-layer CUDA events at gradient readiness

    def _join(self) -> None:
        """The current stream waits for every launched compress, exchange and decode."""
        if self.side is not None:
            cur = torch.cuda.current_stream(self.device)
            cur.wait_stream(self.side)
            cur.wait_stream(self.comm)

    @staticmethod
    def _bucket_offsets(dims, ranges):
        """Layer offsets with every bucket's first layer at a multiple of 4 elements."""
        offsets, pos = [0] * len(dims), 0
        for lo, hi in sorted(ranges):
            pos = (pos + 3) // 4 * 4
            for l in range(lo, hi + 1):
                offsets[l] = pos
                pos += dims[l]
        return offsets, pos

    @torch.no_grad()
    def _relayout(self, ranges) -> None:
        """Place the flat buffers for these bucket ranges, carrying params, residual and momentum
        (and flat gradients) over layer by layer when the layout changes."""
        offsets, n = self._bucket_offsets(self.dims, ranges)
        if offsets == self.offsets and self.flat_param is not None and self.flat_param.numel() == n:
            return
        old = self.offsets

        def moved(buf, fill_params=False):
            new = torch.zeros(n, dtype=buf.dtype if buf is not None else torch.float32, device=self.device)
            for l, d in enumerate(self.dims):
                dst = new[offsets[l]:offsets[l] + d]
                if buf is not None:
                    dst.copy_(buf[old[l]:old[l] + d])
                elif fill_params:
                    dst.copy_(self.params[l].detach().reshape(-1))
            return new

        flat_mode = self.grads_mode == "flat"
        self.flat_param = moved(self.flat_param, fill_params=True)
        self.residual = moved(self.residual)
        self.momentum_buf = moved(self.momentum_buf) if self.mu else None
        self.flat_grad = moved(self.flat_grad) if flat_mode else None
        if getattr(self, "shadow", None) is not None:
            self.shadow = moved(self.shadow)
        self.offsets = offsets
        for l, (p, d) in enumerate(zip(self.params, self.dims)):
            off = offsets[l]
            p.data = self.flat_param[off:off + d].view_as(p)
            if flat_mode:
                p.grad = self.flat_grad[off:off + d].view_as(p)
            elif old is None:
                p.grad = None

    def _per_layer(self, buf) -> torch.Tensor:
        """The flat buffer without inter-bucket padding (the reference's layer layout)."""
        self._join()
        return torch.cat([buf[o:o + d] for o, d in zip(self.offsets, self.dims)])

    @property
    def ref_offsets(self) -> list[int]:
        """Layer offsets of the reference's LayeredVector layout (prefix sums of dims)."""
        out = [0]
        for d in self.dims[:-1]:
            out.append(out[-1] + d)
        return out

    def params_vector(self) -> torch.Tensor:
        """The parameters as the reference's flat LayeredVector data (a copy, no padding)."""
        return self._per_layer(self.flat_param)

    def residual_vector(self) -> torch.Tensor:
        """The error-feedback residual in the reference's layer layout (a copy, no padding)."""
        return self._per_layer(self.residual)

    def _build_buckets(self) -> None:
        """(Re)plan fusion buckets for the current ks; residual and momentum state are kept."""
        ranges = plan_buckets(self.dims, self.ks, self.bucket_cap_bytes)
        self._join()
        self._relayout(ranges)
        for old in self.buckets:  # collective (every rank re-plans in the same call)
            if old.peer is not None:
                old.peer.close()
        self.buckets: list[_BucketRT] = []
        self._bucket_of_param = {}
        for lo, hi in ranges:
            eng = self.engine_factory(self.dims[lo:hi + 1], self.ks[lo:hi + 1], self.world, self.device)
            msg_local = eng.new_messages(1)
            msg_all = eng.new_messages(self.world) if self.exchange_mode == "nccl" else None
            b = _BucketRT(lo, hi, self.offsets[lo], sum(self.dims[lo:hi + 1]), eng, msg_local, msg_all)
            if self.exchange_mode in ("p2p", "fused"):
                from .p2p import PeerExchange

                b.peer = PeerExchange(eng.msg_bytes, self.group)
            if self.device.type == "cuda":
                b.ready = torch.cuda.Event()
            if self.grads_mode == "tensors":
                nl = hi - lo + 1
                b.gtab = torch.zeros(nl, dtype=torch.int64, device=self.device)
                b.ring = [(torch.zeros(nl, dtype=torch.int64, pin_memory=True), torch.cuda.Event())
                          for _ in range(_RING)]
                eng.set_grad_table(b.gtab)
            for l in range(lo, hi + 1):
                self._bucket_of_param[id(self.params[l])] = len(self.buckets)
            self.buckets.append(b)
        self._size = [b.hi - b.lo + 1 for b in self.buckets]
        self._pending = list(self._size)
        self._next = 0  # next bucket to launch (release order)
        if getattr(self, "timing", None) is not None:
            self.enable_timing(True)

    def set_policy(self, policy: CompressionPolicy) -> None:
        """New per-layer ratios (e.g. from perf.select_ratios): recompute k_l, re-plan buckets.
        Call between steps.  The error-feedback residual carries over unchanged."""
        self.policy = policy
        self.ratios = [policy.ratio_for(i + 1) for i in range(len(self.params))]
        self.ks = selection_counts(self.dims, self.ratios)
        self._build_buckets()

    ADAPT_GRID = (25, 50, 100, 250, 500, 1000)

    def adapt(self, network, ratio_cap: float = 1000.0, ratio_grid=None, workers: int | None = None) -> CompressionPolicy:
        """Adaptive rho_l (R: perf.py:231-260) from this rank's device timings of the last step
        (enable_layer_timing + enable_timing before it): each layer gets the smallest grid ratio
        whose exchange + compress hides behind the next layer's backprop.  ``workers`` prices the
        exchange for that many workers (default: the process group's size).  Rank 0's choice is
        broadcast so every rank plans identical buckets and messages."""
        from . import perf

        # default grid keeps rho <= 4 %: the reference's selector prices sparsification as a
        # per-layer constant, while on the device selecting near-dense layers costs much more
        grid = self.ADAPT_GRID if ratio_grid is None else ratio_grid
        pol = perf.select_ratios(self.dims, self.layer_backward_times(), self.layer_spar_times(), network,
                                 self.world if workers is None else int(workers), ratio_cap, grid)
        ratios = torch.tensor([pol.ratio_for(i + 1) for i in range(len(self.params))], dtype=torch.float64,
                              device=self.device)
        if self.world > 1:
            dist.broadcast(ratios, group=self.group, group_src=0)
        pol = CompressionPolicy({i + 1: float(c) for i, c in enumerate(ratios.tolist())}, ratio_cap)
        self.set_policy(pol)
        return pol

    # -- measurement for the adaptive selector ------------------------------------------------
    def enable_layer_timing(self, on: bool = True) -> None:
        """Record a CUDA event on the compute stream when each layer's gradient is ready."""
        self._hook_events = ([torch.cuda.Event(enable_timing=True) for _ in self.params]
                             if on and self.device.type == "cuda" else None)

    def layer_backward_times(self, floor_s: float = 1e-6) -> list[float]:
        """Seconds of backprop attributed to each layer at the last step (layer ids 1..L order):
        the gap between consecutive gradient-ready events in backprop order (the first layer of
        backprop gets the next gap).  Synchronises."""
        ev = self._hook_events
        if ev is None:
            raise RuntimeError("enable_layer_timing() first")
        torch.cuda.synchronize(self.device)
        L = len(ev)
        t = [0.0] * L
        for l in range(L - 1, 0, -1):  # backprop order L..1
            t[l - 1] = max(ev[l].elapsed_time(ev[l - 1]) / 1e3, floor_s)
        t[L - 1] = t[L - 2] if L > 1 else floor_s
        return t

    def layer_spar_times(self) -> list[float]:
        """Compress time of each bucket (last step) spread over its layers by size.  Synchronises."""
        times = self.bucket_times_ms()
        if times is None:
            raise RuntimeError("enable_timing() first")
        out = [0.0] * len(self.params)
        for b, (comp, *_) in zip(self.buckets, times):
            for l in range(b.lo, b.hi + 1):
                out[l] = comp / 1e3 * self.dims[l] / b.numel
        return out

    # -- scheduling -------------------------------------------------------------------------
    def _on_grad(self, p: torch.Tensor) -> None:
        b = self._bucket_of_param.get(id(p))
        if b is None:
            return
        if self._pending[b] <= 0:
            # the bucket already launched this step: its gradients were consumed (and cleared) by
            # the compress, so a second backward before step() would be silently lost
            raise RuntimeError("LagsSGD consumes gradients during backward: call step() after every backward() "
                               "(gradient accumulation over several backward passes is not supported)")
        if self._hook_events is not None:
            self._hook_events[self._layer_of_param[id(p)]].record(torch.cuda.current_stream(self.device))
        self._pending[b] -= 1
        # launch every complete bucket in release order (identical collective order on all ranks)
        while self._next < len(self.buckets) and self._pending[self._next] <= 0:
            self._launch(self._next)
            self._next += 1

    def _launch(self, i: int) -> None:
        b = self.buckets[i]
        lr = self.param_groups[0]["lr"]
        r = self.residual[b.offset:b.offset + b.numel]
        v = self.flat_param[b.offset:b.offset + b.numel]
        m = self.momentum_buf[b.offset:b.offset + b.numel] if self.momentum_buf is not None else None
        if self.side is None:
            self._run_bucket(i, b, self.flat_grad[b.offset:b.offset + b.numel], r, v, m, lr, None)
            return
        cur = torch.cuda.current_stream(self.device)
        self.side.wait_stream(cur)  # the bucket's gradients are complete on the compute stream
        with torch.cuda.stream(self.side):
            if self.grads_mode == "tensors":
                held = self._stage_grad_table(b)
                if self.shadow is not None:
                    self._shadow_step(b, torch.cat([gt.reshape(-1) for _, gt in held]), lr)
                self._run_bucket(i, b, None, r, v, m, lr, self.side)
                for p, gt in held:  # released to autograd: the next backward hands over a fresh tensor
                    gt.record_stream(self.side)
                    p.grad = None
            else:
                g = self.flat_grad[b.offset:b.offset + b.numel]
                if self.shadow is not None:
                    self._shadow_step(b, g, lr)
                self._run_bucket(i, b, g, r, v, m, lr, self.side)

    def _shadow_step(self, b, g, lr) -> None:
        """x -= lr * (sum of the workers' gradients) / P for the bucket (before the compress clears g)."""
        gsum = g.clone()
        if self.world > 1:
            dist.all_reduce(gsum, group=self.group)
        b.engine.shadow_step(gsum, self.shadow[b.offset:b.offset + b.numel], lr, self.world, stream=self.side)

    def _log_identity(self) -> None:
        """The residual identity of every bucket after this step (R: training.py:356-369)."""
        outs = []
        for b in self.buckets:
            r = self.residual[b.offset:b.offset + b.numel]
            if self.world > 1:
                r = r.clone()
                dist.all_reduce(r, group=self.group)
            outs.append(b.engine.identity(self.flat_param[b.offset:b.offset + b.numel],
                                          self.shadow[b.offset:b.offset + b.numel], r, self.world))
        self._identity = (self._steps, outs)

    def last_identity(self):
        """(step, {"v_x_gap", "resid_dev", "residual_norms"}) of the last logged step, as the
        reference's IterationRecord fields (R: training.py:356-369); synchronises."""
        if self._identity is None:
            return None
        step, outs = self._identity
        norms, gsq, dev = [0.0] * len(self.params), 0.0, 0.0
        for b, o in zip(self.buckets, outs):  # buckets are in release order (layer L first)
            h = o.cpu().tolist()
            nl = b.hi - b.lo + 1
            norms[b.lo:b.hi + 1] = [x ** 0.5 for x in h[:nl]]
            gsq += h[nl]
            dev = max(dev, h[nl + 1])
        return step, {"v_x_gap": gsq ** 0.5, "resid_dev": dev, "residual_norms": norms}

    def _stage_grad_table(self, b):
        """Point the bucket's device table at its parameters' autograd gradient tensors (a pinned
        host slot, copied on the side stream); unused parameters get zeros."""
        host, ev = b.ring[b.slot]
        ev.synchronize()  # this slot's previous copy (_RING launches ago) has completed
        held = []
        ptrs = host.numpy()
        for q, l in enumerate(range(b.lo, b.hi + 1)):
            p = self.params[l]
            gt = p.grad
            if gt is None:
                gt = torch.zeros(self.dims[l], dtype=torch.float32, device=self.device)
            elif gt.dtype != torch.float32 or not gt.is_contiguous():
                gt = gt.float().contiguous()
            held.append((p, gt))
            ptrs[q] = gt.data_ptr()
        b.gtab.copy_(host, non_blocking=True)
        ev.record(self.side)
        b.slot = (b.slot + 1) % _RING
        return held

    def _run_bucket(self, i, b, g, r, v, m, lr, stream):
        t = self.timing[i] if self.timing is not None else None
        if t is not None:
            t[0].record(stream)
        local = self.world == 1 or not self.exchange
        zg = g is not None  # flat gradients are cleared by the compress (fused zero_grad)
        if local and m is None and hasattr(b.engine, "step_local"):  # P = 1: update fused into selection
            b.engine.step_local(g, r, lr, v, b.msg_local, self.status, stream=stream, zero_grad=zg)
            if t is not None:
                for e in t[1:]:
                    e.record(stream)
            if self._log_delta_now():
                self._log_delta(b, r, b.msg_local, 1, stream)
            return
        fused = self.exchange_mode == "fused"
        b.engine.compress(g, r, lr, b.msg_local, self.status, stream=stream, zero_grad=zg,
                          **({"peer": b.peer} if fused else {}))
        if t is not None:
            t[1].record(stream)
        comm = stream
        if stream is not None and self.comm is not None:  # exchange + decode on the serial network channel
            b.ready.record(stream)
            self.comm.wait_event(b.ready)
            comm = self.comm
        with torch.cuda.stream(comm) if comm is not None else _nullctx():
            if t is not None:
                t[2].record(comm)
            if self.exchange_mode == "nccl":
                dist.all_gather_into_tensor(b.msg_all, b.msg_local, group=self.group)
                msgs, P = b.msg_all, self.world
                if t is not None:
                    t[3].record(comm)
            elif self.exchange_mode == "p2p":
                msgs = b.peer.exchange(b.msg_local, stream=comm, mid_event=t[3] if t is not None else None)
                P = self.world
            elif fused:  # the transfer happened inside the compress: only the wait for the peers
                if t is not None:
                    t[3].record(comm)
                msgs, P = b.peer.wait(stream=comm), self.world
            else:
                msgs, P = b.msg_local, 1
                if t is not None:
                    t[3].record(comm)
            if t is not None:
                t[4].record(comm)
            b.engine.decode(msgs, P, v, momentum=m, mu=self.mu, stream=comm)
            if t is not None:
                t[5].record(comm)
            if self._log_delta_now():
                self._log_delta(b, r, msgs, P, comm)

    def _log_delta_now(self) -> bool:
        return self.delta_every > 0 and (self._steps + 1) % self.delta_every == 0

    def _log_delta(self, b, r, msgs, P, stream) -> None:
        """delta^(l) of the bucket's layers this step: acc_p = r_p + sent_p rebuilt from the
        gathered messages and all-gathered residuals (R: training.py:329-337)."""
        if P > 1:
            r_all = torch.empty(P * b.numel, dtype=r.dtype, device=r.device)
            dist.all_gather_into_tensor(r_all, r.contiguous(), group=self.group)
        else:
            r_all = r
        acc = torch.empty(P * b.numel, dtype=r.dtype, device=r.device)
        b.engine.reconstruct(msgs, P, r_all, acc, stream=stream)
        b.engine.delta(acc, r_all, P, out=self._delta[b.lo:b.hi + 1], stream=stream)
        self._delta_step = self._steps + 1

    def last_delta(self):
        """(step, [delta^(l) or None per layer]) of the last logged step (synchronises)."""
        self._join()
        vals = self._delta.cpu().tolist()
        return self._delta_step, [None if v != v else v for v in vals]

    def enable_timing(self, on: bool = True) -> None:
        """Record CUDA events around each bucket's compress, exchange and decode."""
        if on and self.device.type == "cuda":
            self.timing = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in self.buckets]
        else:
            self.timing = None

    def bucket_times_ms(self):
        """[(compress, exchange, decode, transfer, peer_wait)] per bucket of the last step, ms
        (synchronises).  compress on the side stream; on the communication stream: exchange = from
        the channel taking the bucket to its messages being available, transfer = the push (p2p)
        or all-gather (NCCL, which includes waiting for the slowest rank), peer_wait = waiting for
        the peers' pushes (p2p; 0 for NCCL), decode = the rank-ordered decode + update."""
        if self.timing is None:
            return None
        torch.cuda.synchronize(self.device)
        out = []
        for c0, c1, x0, x1, x2, d1 in self.timing:
            out.append((c0.elapsed_time(c1), x0.elapsed_time(x2), x2.elapsed_time(d1), x0.elapsed_time(x1),
                        x1.elapsed_time(x2)))
        return out

    # -- optimizer API ----------------------------------------------------------------------
    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        while self._next < len(self.buckets):  # hooks that never fired (unused params, no backward)
            self._launch(self._next)
            self._next += 1
        self._join()
        self._pending = list(self._size)
        self._next = 0
        self._steps += 1
        if self.shadow is not None and self._steps % self.monitor_every == 0:
            self._log_identity()
        self._poll_status()
        return loss

    def _poll_status(self) -> None:
        """Non-finite gradients (R: training.py:174-175) without stalling the host: the device flag
        is copied to pinned memory behind the step and inspected at a later step() once the copy
        has landed (so DivergenceError may surface a step late); check_divergence() waits."""
        if self.device.type != "cuda":
            if int(self.status.item()):
                raise DivergenceError("a worker produced a non-finite gradient", iteration=self._steps)
            return
        if self._status_event is not None and self._status_event.query():
            if int(self._status_host.item()):
                raise DivergenceError("a worker produced a non-finite gradient", iteration=self._status_step)
            self._status_event = None
        if self._status_event is None and self._steps % self.check_every == 0:
            self._status_host.copy_(self.status, non_blocking=True)
            self._status_event = torch.cuda.Event()
            self._status_event.record(torch.cuda.current_stream(self.device))
            self._status_step = self._steps

    def check_divergence(self) -> None:
        """Synchronous check of the non-finite flag (raises DivergenceError)."""
        if int(self.status.item()):
            raise DivergenceError("a worker produced a non-finite gradient", iteration=self._steps)

    def zero_grad(self, set_to_none: bool = False):
        """Gradients are cleared by the compress pass itself; the views must stay in place."""
        return None

    def state_dict(self):
        """Optimizer state plus the error-feedback residual and momentum in the reference's layer
        layout (R: layered.py:46-107, no padding) and the per-layer ratios: a true resume (the
        reference saves only final parameters, R: experiment.py:501-502)."""
        self._join()
        sd = super().state_dict()
        sd["lags"] = {"residual": self._per_layer(self.residual),
                      "momentum": None if self.momentum_buf is None else self._per_layer(self.momentum_buf),
                      "steps": self._steps, "ks": list(self.ks), "ratios": list(self.ratios)}
        return sd

    def load_state_dict(self, state_dict):
        lags = state_dict.pop("lags", None)
        super().load_state_dict(state_dict)
        if lags is not None:
            if "ratios" in lags and list(lags["ratios"]) != list(self.ratios):
                cap = max(self.policy.ratio_cap, max(lags["ratios"]))
                self.set_policy(CompressionPolicy({i + 1: float(c) for i, c in enumerate(lags["ratios"])}, cap))
            self._load_per_layer(self.residual, lags["residual"])
            if self.momentum_buf is not None and lags["momentum"] is not None:
                self._load_per_layer(self.momentum_buf, lags["momentum"])
            self._steps = int(lags["steps"])

    @torch.no_grad()
    def _load_per_layer(self, buf, src) -> None:
        src = src.to(buf.device, buf.dtype).reshape(-1)
        if src.numel() != sum(self.dims):
            raise ValueError("saved LagsSGD state does not match the parameters")
        pos = 0
        for o, d in zip(self.offsets, self.dims):
            buf[o:o + d].copy_(src[pos:pos + d])
            pos += d

    def remove_hooks(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []
