"""CUPTI kernel durations (torch.profiler) of the P-rank decode alone, eager back-to-back launches:
separates the kernel's own duration from the launch gaps.  Usage: decode_timeline.py [P]."""
import json
import os
import sys
import tempfile

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
r = torch.zeros(n, device="cuda")
for p in range(P):
    r.zero_()
    for _ in range(3):
        b.compress(torch.randn(n, device="cuda", generator=gen), r, 0.1, msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes], st)
v = torch.randn(n, device="cuda", generator=gen)
for _ in range(20):
    b.decode(msgs, P, v)
torch.cuda.synchronize()
tmp = tempfile.mkdtemp()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        b.decode(msgs, P, v)
    torch.cuda.synchronize()
prof.export_chrome_trace(os.path.join(tmp, "t.json"))
ev = [e for e in json.load(open(os.path.join(tmp, "t.json")))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
prev = None
for e in ev:
    gap = 0.0 if prev is None else e["ts"] - prev
    print(f"dur {e['dur']:7.2f} us  gap {gap:6.2f}  {e['name'][:70]}")
    prev = e["ts"] + e["dur"]
