"""Single-GPU decode workload for ncu: P simulated ranks' messages (ResNet-50 shapes, rho = 0.001)
decoded in rank order (decode_scatter + decode_update) repeatedly; prints the event-timed
decode latency and its algorithmic bytes (8 B per received pair + 8 B per touched weight).
Usage: python tools/decode_run.py [P]   (ncu: -k regex:decode)"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dims = resnet50_dims()
ks = ks_for(dims)
n = sum(dims)
b = L.Bucket(dims, ks, N.F32, max_world=P)
gen = torch.Generator(device="cuda").manual_seed(3)
msgs = b.new_messages(P)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for p in range(P):
    r = torch.zeros(n, device="cuda")
    for _ in range(3):
        b.compress(torch.randn(n, device="cuda", generator=gen), r, 0.1, msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes], st)
v = torch.randn(n, device="cuda", generator=gen)
for _ in range(20):
    b.decode(msgs, P, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    b.decode(msgs, P, v)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 100 * 1e3
pairs = sum(int(b.counts_view(msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes]).sum()) for p in range(P))
union = len(np.unique(np.concatenate([ii + int(b.offsets[j]) for p in range(P)
                                      for j, (ii, _) in enumerate(b.unpack(msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes]))])))
byt = 8 * pairs + 8 * union
print(f"P={P} decode {us:.1f} us  pairs {pairs} union {union}  algorithmic {byt / 1e6:.2f} MB -> {byt / (us * 1e-6) / 1e9:.1f} GB/s")
