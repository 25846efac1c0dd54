"""Which layers of an fp64 / mixed bucket take the dense fallback in steady state (diagnostic):
ResNet-50 shapes at rho = 0.001, P = 1 steps; prints per falling-back layer d, k, fallbacks over
the measured steps, the last candidate count and the threshold's high word."""
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
for t in range(60):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
s0 = b.stats().astype(np.int64)
for t in range(30):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
s1 = b.stats().astype(np.int64)
fb = s1[:, 1] - s0[:, 1]
print(f"{mode}: {int(fb.sum())} fallbacks in 30 steps over {int((fb > 0).sum())} layers")
for j in np.nonzero(fb)[0]:
    print(f"  layer {j}: d={dims[j]} k={ks[j]} fallbacks={int(fb[j])} last_cands={int(s1[j, 2])} "
          f"thr_hi=0x{int(s1[j, 0]):08x} path={int(s1[j, 5])}")
