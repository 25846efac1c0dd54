"""K1 alone in steady state (diagnostic): the bench workload's compress with CUDA events around
each K1 launch (the bucket's probe events), median over 100 eager steps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

dims = resnet50_dims()
ks = ks_for(dims, 0.001)
n = sum(dims)
b = L.Bucket(dims, ks, N.F32)
gen = torch.Generator(device="cuda").manual_seed(1234)
gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
r = torch.zeros(n, device="cuda")
v = torch.randn(n, device="cuda", generator=gen)
msg = b.new_messages(1)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for t in range(60):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
ts = []
for t in range(100):
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    a1.record()  # torch creates the CUDA events lazily at the first record
    b.set_probe_events(a0, a1)
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
    torch.cuda.synchronize()
    ts.append(a0.elapsed_time(a1) * 1e3)
ts.sort()
print(f"K1 (probe events, eager): median {ts[50]:.1f} us, p10 {ts[10]:.1f}, p90 {ts[90]:.1f}")
