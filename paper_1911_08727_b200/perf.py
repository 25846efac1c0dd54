"""Communication cost model and adaptive per-layer ratio selector (R: perf.py), fed by device timings.

The reference prices messages with an alpha-beta model and chooses, per layer, the smallest
compression ratio whose exchange hides behind the next layer's backprop (R: perf.py:231-260).
It only ever sees scenario-file numbers.  Here the same selector is fed with measured costs:
per-layer backward times (CUDA events recorded in the gradient hooks), per-layer compress
times (bucket events), and a network model fitted to timed NCCL all-gathers.  On the device a
sparse entry is int32 index + fp32 value = 8 bytes (the reference prices u32 + f64 = 12).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .sparsify import CompressionPolicy

DEVICE_ENTRY_BYTES = 8      # int32 index + fp32 value (the device message)
REFERENCE_ENTRY_BYTES = 12  # u32 index + f64 value (R: perf.py:22)
DEFAULT_RATIO_GRID = (1, 2, 5, 10, 25, 50, 100, 250, 500, 1000)  # R: perf.py:25


def ring_multiplier(workers: int) -> float:
    return float(workers - 1)  # R: perf.py:28-29


@dataclass(frozen=True)
class NetworkModel:
    """Seconds per message (latency) and per byte (inverse bandwidth) -- R: perf.py:39-56."""

    latency: float
    inv_bandwidth: float
    multiplier: Callable[[int], float] | None = None

    def __post_init__(self):
        if self.latency < 0 or self.inv_bandwidth < 0:
            raise ValueError("latency and inv_bandwidth must be non-negative")

    def factor(self, workers: int) -> float:
        return (ring_multiplier if self.multiplier is None else self.multiplier)(workers)

    def message_time(self, nbytes: float, workers: int) -> float:
        return self.factor(workers) * (self.latency + self.inv_bandwidth * nbytes)


def comm_time(dim: int, ratio: float, network: NetworkModel, workers: int,
              entry_bytes: int = DEVICE_ENTRY_BYTES) -> float:
    """Exchange time of one layer's sparse message at a ratio -- R: perf.py:59-70."""
    if dim < 1:
        raise ValueError("dim must be >= 1")
    if ratio < 1:
        raise ValueError(f"ratio must be >= 1, got {ratio}")
    return network.message_time(max(1, int(dim // ratio)) * entry_bytes, workers)


def select_ratios(dims: Sequence[int], backward_times: Sequence[float], spar_times: Sequence[float],
                  network: NetworkModel, workers: int, ratio_cap: float,
                  ratio_grid: Sequence[float] = DEFAULT_RATIO_GRID,
                  entry_bytes: int = DEVICE_ENTRY_BYTES) -> CompressionPolicy:
    """Smallest grid ratio per layer whose message + sparsification hides behind compute.

    Same rule as R: perf.py:231-260: layer l >= 2 budgets against the backward time of layer
    l - 1 (the layer computed next in backprop), layer 1 against its own; a layer no grid
    ratio satisfies gets the cap; every ratio is clamped to the cap.
    """
    if ratio_cap < 1:
        raise ValueError("ratio_cap must be >= 1")
    grid = sorted(float(c) for c in ratio_grid)
    if not grid:
        raise ValueError("ratio grid must be non-empty")
    if grid[0] < 1:
        raise ValueError("ratios must be >= 1")
    if not (len(dims) == len(backward_times) == len(spar_times)):
        raise ValueError("dims, backward_times and spar_times must have equal length")
    ratios = {}
    for l in range(1, len(dims) + 1):
        budget = backward_times[l - 2] if l >= 2 else backward_times[0]
        chosen = None
        for c in grid:
            if comm_time(dims[l - 1], c, network, workers, entry_bytes) + spar_times[l - 1] <= budget:
                chosen = c
                break
        ratios[l] = min(chosen if chosen is not None else ratio_cap, ratio_cap)
    return CompressionPolicy(ratios, ratio_cap)


def pipelined_makespan(forward_time: float, backward_times: Sequence[float], spar_times: Sequence[float],
                       comm_times: Sequence[float]) -> float:
    """Compute resource L..1 (+ sparsify), one serial network channel in release order, next
    forward after the last arrival -- R: perf.py:173-195."""
    t = 0.0
    releases = []
    for l in range(len(backward_times), 0, -1):
        t += backward_times[l - 1]
        if spar_times[l - 1] > 0:
            t += spar_times[l - 1]
        releases.append((l, t))
    net = 0.0
    for l, rel in releases:
        net = max(net, rel) + comm_times[l - 1]
    return net + forward_time


def fit_network(message_bytes: Sequence[float], seconds: Sequence[float], workers: int) -> NetworkModel:
    """Least-squares alpha-beta fit of measured exchange times: t = m(P) * (a + b * bytes)."""
    x = np.asarray(message_bytes, dtype=np.float64)
    y = np.asarray(seconds, dtype=np.float64) / max(ring_multiplier(workers), 1.0)
    w = 1.0 / np.maximum(y, 1e-12)  # relative error: latency- and bandwidth-bound sizes count alike
    A = np.stack([np.ones_like(x), x], axis=1) * w[:, None]
    (a, b), *_ = np.linalg.lstsq(A, y * w, rcond=None)
    return NetworkModel(max(float(a), 0.0), max(float(b), 0.0))


def measure_allgather(group=None, device=None, sizes=(256, 4096, 65536, 1 << 20, 1 << 23, 1 << 26),
                      reps: int = 10):
    """Device-timed NCCL all-gather of uint8 messages (CUDA events, max over ranks).
    Returns (bytes per rank, seconds)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out_s = []
    for nb in sizes:
        src = torch.zeros(int(nb), dtype=torch.uint8, device=device)
        dst = torch.zeros(int(nb) * world, dtype=torch.uint8, device=device)
        for _ in range(3):
            dist.all_gather_into_tensor(dst, src, group=group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(device)
        e0.record()
        for _ in range(reps):
            dist.all_gather_into_tensor(dst, src, group=group)
        e1.record()
        torch.cuda.synchronize(device)
        t = torch.tensor([e0.elapsed_time(e1) / reps / 1e3], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        out_s.append(float(t))
    return list(sizes), out_s
