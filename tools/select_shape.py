"""Shape of the candidate / cluster radix selects (needs a -DLAGS_DBG_SELECT build via
LAGS_B200_LIB): per layer, the threshold bin's size after the first pass, the highest differing
key bit, the passes run and whether the bin-list finish ran.  Diagnostic only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

dims = resnet50_dims()
ks = ks_for(dims)
n = sum(dims)
b = L.Bucket(dims, ks, N.F32)
gen = torch.Generator(device="cuda").manual_seed(1)
gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
r = torch.zeros(n, device="cuda")
v = torch.randn(n, device="cuda", generator=gen)
msg = b.new_messages(1)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for t in range(300):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
torch.cuda.synchronize()
s = b.stats().astype(np.int64)
rows = []
for j in range(len(dims)):
    if s[j, 5] not in (1, 3):
        continue
    w = int(s[j, 7])
    rows.append((dims[j], ks[j], int(s[j, 2]), int(s[j, 5]), w & 4095, (w >> 12) & 63, (w >> 18) & 15, (w >> 22) & 1))
rows.sort(key=lambda x: -x[0])
print("dim k m path in_bin1 hibit passes list")
for x in rows[:20]:
    print(*x)
print("list finish used:", sum(x[7] for x in rows), "of", len(rows), "; passes histogram:",
      np.bincount([x[6] for x in rows]).tolist())
