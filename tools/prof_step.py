"""A short eager run of the bench step (ResNet-50 layer shapes, P = 1 fused update) for ncu
captures: `--steps` steps after `--warmup` steps.  Diagnostic only (no timing printed)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--rho", type=float, default=0.001)
args = ap.parse_args()
dims = resnet50_dims()
ks = ks_for(dims, args.rho)
n = sum(dims)
b = L.Bucket(dims, ks, N.F32)
gen = torch.Generator(device="cuda").manual_seed(1234)
gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
r = torch.zeros(n, device="cuda")
v = torch.randn(n, device="cuda", generator=gen)
msg = b.new_messages(1)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for t in range(args.steps):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
torch.cuda.synchronize()
assert int(st.item()) == 0
print("ok", int(b.stats()[:, 1].sum()), "fallbacks")
