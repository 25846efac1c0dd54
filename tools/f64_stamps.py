"""Per-layer phase cycles of select64_kernel (fp64 / mixed fast path) from a -DLAGS_DBG_STAMPS build
(LAGS_B200_LIB=variants/libstamps.so): ResNet-50 shapes at rho = 0.001, graph-replayed P = 1
steps.  Prints the slowest layers' phases (counts, gather, radix select, compaction, state) and
their start / end in ns after the first layer's start.  Diagnostic only.  argv: f64 | acc64."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from paper_1911_08727_b200.workloads import resnet50  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "f64"
dims = [p.numel() for p in resnet50().parameters()]
ks = [min(d, max(1, d // 1000)) for d in dims]
n = sum(dims)
b = L.Bucket(dims, ks, N.F64 if mode == "f64" else N.F32_ACC64)
dt = torch.float64 if mode == "f64" else torch.float32
gen = torch.Generator(device="cuda").manual_seed(5)
gs = [torch.randn(n, device="cuda", generator=gen, dtype=dt) for _ in range(3)]
r = torch.zeros(n, device="cuda", dtype=dt)
v = torch.randn(n, device="cuda", generator=gen, dtype=dt)
msg = b.new_messages(1)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for t in range(40):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
torch.cuda.synchronize()
acc = []
for t in range(20):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (1024 * 8))()
    assert N.lib.lags_dbg_s64_read(buf) == 0
    acc.append(np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8)[:len(dims)].astype(np.int64))
a = np.stack(acc)
cyc = np.median(np.diff(a[:, :, :6], axis=2), axis=0)  # layers x 5 phases
t0 = a[:, :, 6].min(axis=1, keepdims=True)
start = np.median((a[:, :, 6] - t0) & 0xffffffff, axis=0)
end = np.median((a[:, :, 7] - t0) & 0xffffffff, axis=0)
print(f"{mode}: median over 20 steps; phases in cycles, times in ns after the first layer's start")
print(f"{'layer':>5} {'d':>8} {'k':>5} {'counts':>7} {'gather':>7} {'radix':>7} {'compact':>8} {'state':>6} "
      f"{'start':>7} {'end':>7}")
for j in np.argsort(-end)[:16]:
    c = cyc[j]
    print(f"{j:5d} {dims[j]:8d} {ks[j]:5d} {c[0]:7.0f} {c[1]:7.0f} {c[2]:7.0f} {c[3]:8.0f} {c[4]:6.0f} "
          f"{start[j]:7.0f} {end[j]:7.0f}")
