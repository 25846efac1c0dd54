"""Which layers take the dense fallback in the bench's steady state, and what a fallback step costs.

ResNet-50 shapes, rho = 0.001, the bench's P = 1 step (compress + fused update) replayed from
CUDA graphs over 3 rotating gradient buffers.  Each step is timed alone (events around one
replay, synchronised), then the per-layer stats are read.  Prints one JSON line.  Diagnostic only."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from paper_1911_08727_b200.workloads import resnet50  # noqa: E402


def main(steps=int(os.environ.get("STEPS", "600")), warm=int(os.environ.get("WARM", "200"))):
    dims = [p.numel() for p in resnet50().parameters()]
    ks = [min(d, max(1, int(d // 1000.0))) for d in dims]
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
    r = torch.zeros(n, device="cuda")
    v = torch.randn(n, device="cuda", generator=gen)
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    for t in range(6):
        b.step_local(gs[t % 3], r, 0.1, v, msg, st, stream=cap)
    torch.cuda.synchronize()
    graphs = []
    for i in range(3):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            b.step_local(gs[i], r, 0.1, v, msg, st, stream=cap)
        graphs.append(g)
    for t in range(warm):
        graphs[t % 3].replay()
    torch.cuda.synchronize()
    prev = b.stats().astype(np.int64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, fb_steps, events = [], [], []
    for t in range(steps):
        e0.record()
        graphs[t % 3].replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
        cur = b.stats().astype(np.int64)
        d = cur[:, 1] - prev[:, 1]
        if d.any():
            fb_steps.append(t)
            for j in np.nonzero(d)[0]:
                events.append({"step": t, "layer": int(j), "dim": dims[j], "k": ks[j], "path": int(cur[j, 5]),
                               "cands_prev": int(prev[j, 2]), "cands": int(cur[j, 2]), "pf256": int(cur[j, 6]),
                               "cycles": int(cur[j, 4]), "us": round(times[-1], 1)})
        prev = cur
    times = np.array(times)
    mask = np.zeros(steps, bool)
    mask[fb_steps] = True
    out = {"steps": steps, "warm": warm, "fallback_steps": int(mask.sum()),
           "median_us_clean": round(float(np.median(times[~mask])), 2),
           "median_us_fallback": round(float(np.median(times[mask])), 2) if mask.any() else None,
           "mean_us_all": round(float(times.mean()), 2),
           "mean_us_clean": round(float(times[~mask].mean()), 2),
           "events": events[:40]}
    assert int(st.item()) == 0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
