"""Phase timeline of the pipelined drop-in lags_step (host marks, ms from the call's start).
Diagnostic only."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import training as T  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

dims = resnet50_dims()
ks = ks_for(dims)
n = sum(dims)
shape = [L.LayerShape(i + 1, d) for i, d in enumerate(dims)]
rng = np.random.default_rng(7)
v = L.LayeredVector(shape, rng.standard_normal(n).astype(np.float32))
gs = [L.LayeredVector(shape, rng.standard_normal(n).astype(np.float32)) for _ in range(2)]
res = [L.LayeredVector.zeros(shape, np.float32)]
counts = {i + 1: k for i, k in enumerate(ks)}
if len(sys.argv) > 1:
    T._COPY_THREADS = int(sys.argv[1])
for t in range(6):
    v = L.lags_step(v, [gs[t % 2]], 0.1, counts, res)
rows = []
for t in range(5):
    T.PIPELINE_TRACE = []
    v = L.lags_step(v, [gs[t % 2]], 0.1, counts, res)
    t0 = T.PIPELINE_TRACE[0][1]
    rows.append({k: round((x - t0) * 1e3, 3) for k, x in T.PIPELINE_TRACE})
T.PIPELINE_TRACE = None
torch.cuda.synchronize()
import time  # noqa: E402

t0 = time.perf_counter()
for t in range(10):
    v = L.lags_step(v, [gs[t % 2]], 0.1, counts, res)
ms = (time.perf_counter() - t0) / 10 * 1e3
print(json.dumps({"copy_threads": T._COPY_THREADS, "ms_per_step": round(ms, 3), "last": rows[-1]}))
