"""Per-phase cycles of the CTA small-dense path on buckets of identical tiny layers (diagnostic):
load, threshold (rounds of a block max for k <= 16, else radix), compaction."""
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1911_08727_b200 as L
from paper_1911_08727_b200 import _native as N
for d, k in [(4096, 4), (4096, 16), (2304, 2), (3000, 3)]:
    dims = [d] * 40
    ks = [k] * 40
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(1)
    gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
    r = torch.zeros(n, device="cuda"); v = torch.randn(n, device="cuda", generator=gen)
    msg = b.new_messages(1); st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for t in range(30):
        b.step_local(gs[t % 3], r, 0.1, v, msg, st)
    torch.cuda.synchronize()
    s = b.stats().astype(np.int64)
    ph = np.array([((int(w) & 2047) * 64, ((int(w) >> 11) & 2047) * 64, ((int(w) >> 22) & 2047) * 64) for w in s[:, 7]])
    print(d, k, "path", set(s[:, 5].tolist()), "cycles median", np.median(s[:, 4]), "phases median", np.median(ph, axis=0))
