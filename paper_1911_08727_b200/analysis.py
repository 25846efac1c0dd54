"""Convergence diagnostics of the drop-in surface (R: analysis.py), computed on the B200.

``topk_aggregation_ratio`` is the reference's delta^(l): how much of the aggregate the summed
per-worker top-k picks miss, relative to the expectation of a uniformly random k-selection
(R: analysis.py:24-56).  The top-k selections and the fp64 sums (worker order, as the reference
adds them) run in liblagsb200.so; only the final dot products differ in summation order from
numpy's BLAS dot, so results agree to rounding (tests use rtol 1e-12).
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .engine import Bucket
from .errors import StructureError


def topk_aggregation_ratio(local_vectors: Sequence, k: int) -> float | None:
    """||sum_p x^p - sum_p decompress(top_k(x^p, k))||^2 / ((1 - k/d) ||sum_p x^p||^2), or None when
    the denominator vanishes (R: analysis.py:24-56).  Inputs are converted to float64 first, as
    the reference does."""
    if not local_vectors:
        raise StructureError("need at least one worker vector")
    arrays = [np.asarray(x, dtype=np.float64).reshape(-1) for x in local_vectors]
    d = arrays[0].size
    for x in arrays[1:]:
        if x.size != d:
            raise StructureError("worker vectors must share one dimension")
    if not 1 <= k <= d:
        raise ValueError(f"k={k} outside 1..{d}")
    P = len(arrays)
    stride = d + (d & 1)  # planes 16-byte aligned (the kernels' flat-buffer contract)
    b = Bucket([d], [k], N.F64, max_world=P)
    acc = torch.zeros(P * stride, dtype=torch.float64, device="cuda")
    for p, x in enumerate(arrays):
        acc[p * stride:p * stride + d].copy_(torch.from_numpy(x))
    r = acc.clone()
    g = torch.zeros(d, dtype=torch.float64, device="cuda")
    msg = b.new_messages(1)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for p in range(P):  # r_p = x^p with its top-k zeroed (alpha = 0: acc = x^p + 0 * 0)
        b.compress(g, r[p * stride:(p + 1) * stride], 0.0, msg, status, exact=True)
    # compress forms x + 0.0, which only turns -0.0 into +0.0: the sums below are unaffected
    out = b.delta(acc, r, P, plane_stride=stride)
    v = float(out.item())
    return None if math.isnan(v) else v
