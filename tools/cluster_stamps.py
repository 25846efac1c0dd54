"""Phase timing of one cluster-selected layer (the first cluster), per rank, from a
-DLAGS_DBG_STAMPS build (LAGS_B200_LIB=variants/libstamps.so).  Graph-replayed steps as in the
bench; prints per-phase cycles of each rank and the globaltimer offsets.  Diagnostic only."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402

NAMES = ["entry", "counts loaded", "block sums", "cluster wait", "histogram cut", "gather", "push",
         "cluster.sync", "resolve", "lower-rank counts", "-", "ordered compact", "zero histogram", "end"]

dims = resnet50_dims()
ks = ks_for(dims, float(sys.argv[1]) if len(sys.argv) > 1 else 0.001)
n = sum(dims)
b = L.Bucket(dims, ks, N.F32)
gen = torch.Generator(device="cuda").manual_seed(1)
gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
r = torch.zeros(n, device="cuda")
v = torch.randn(n, device="cuda", generator=gen)
msg = b.new_messages(1)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for t in range(200):
    b.step_local(gs[t % 3], r, 0.1, v, msg, st)
cap = torch.cuda.Stream()
graphs = []
for i in range(3):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        b.step_local(gs[i], r, 0.1, v, msg, st, stream=cap)
    graphs.append(g)
acc = []
for t in range(60):
    graphs[t % 3].replay()
    torch.cuda.synchronize()
    if t >= 20:
        buf = (C.c_ulonglong * (4 * 2 * 24))()
        assert N.lib.lags_dbg_stamps_read(buf) == 0
        acc.append(np.frombuffer(buf, dtype=np.uint64).reshape(4, 2, 24).astype(np.int64))
a = np.stack(acc)  # steps, rank, kind, stamp
cyc = a[:, :, 0, :]
gt = a[:, :, 1, :]
if True:
    sp = []
    for t in range(20):
        graphs[t % 3].replay()
        torch.cuda.synchronize()
        b5 = (C.c_ulonglong * 8)()
        N.lib.lags_dbg_sp_read(b5)
        sp.append(np.frombuffer(b5, dtype=np.uint64).astype(np.int64))
    sp = np.median(np.diff(np.stack(sp)[:, :5], axis=1), axis=0)
    print("spec_place of rank 0 (cycles): scan", sp[0], "takes", sp[1], "extras", sp[2], "leftovers", sp[3])
print("median cycles per phase (ranks 0..3):")
for i in range(1, 14):
    d = np.median(cyc[:, :, i] - cyc[:, :, i - 1], axis=0)
    print(f"  {NAMES[i]:18s}", " ".join(f"{x:7.0f}" for x in d))
tot = np.median(cyc[:, :, 13] - cyc[:, :, 0], axis=0)
print(f"  {'total':18s}", " ".join(f"{x:7.0f}" for x in tot))
w = np.median(cyc[:, :, 15] - cyc[:, :, 14], axis=0)
print(f"  {'griddep wait':18s}", " ".join(f"{x:7.0f}" for x in w))
g0 = gt[:, :, 15].min(axis=1, keepdims=True)
print("globaltimer ns after the first rank's wait: entry / end per rank (median):")
print("  entry", np.median(gt[:, :, 0] - g0, axis=0), " end", np.median(gt[:, :, 13] - g0, axis=0))
if np.any(cyc[:, 0, 16]):
    print("LAGS_DBG_TWICE: cycles of the first (dry) run per rank:", np.median(cyc[:, :, 16], axis=0))
# the candidate-path layer LAGS_DBG_J (one CTA)
cs_ = []
for t in range(30):
    graphs[t % 3].replay()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)()
    assert N.lib.lags_dbg_cstamps_read(buf) == 0
    cs_.append(np.frombuffer(buf, dtype=np.uint64).astype(np.int64))
c = np.stack(cs_)
CN = ["layer entry->counts start", "counts loaded", "block sums", "gather", "select", "ordered compact", "P=1 update",
      "state write"]
order = [8, 0, 1, 2, 3, 4, 5, 6, 7]
print("candidate-path layer: median cycles per phase")
for a_, b_, nm in zip(order[:-1], order[1:], CN):
    print(f"  {nm:26s} {np.median(c[:, b_] - c[:, a_]):7.0f}")
print(f"  {'total':26s} {np.median(c[:, 7] - c[:, 8]):7.0f}")
