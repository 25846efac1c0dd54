"""Kernel timeline of the bench step (CUPTI activity records via torch.profiler; no nsys here).

Prints, for the last steps, each kernel's start offset, duration and the idle gap before it, for
eager launches and for CUDA-graph replay.  Diagnostic only.
"""

import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402


def kernels_from_trace(path):
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    return [(e["ts"], e["dur"], e["name"]) for e in ks]


def show(title, ks, last=12):
    print(f"--- {title}")
    ks = ks[-last:]
    t0 = ks[0][0]
    prev_end = None
    for ts, dur, name in ks:
        gap = 0.0 if prev_end is None else ts - prev_end
        print(f"  +{ts - t0:9.1f} us  dur {dur:7.1f}  gap {gap:6.1f}  {name[:60]}")
        prev_end = ts + dur


def main():
    # optional workload: resnet50 (default) | resnet50:RHO | lstm | vgg16 | resnet20
    arg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    name, _, rho = arg.partition(":")
    rho = float(rho) if rho else 0.001
    if name == "lstm":
        from paper_1911_08727_b200.workloads import LSTMPTB
        dims = [p.numel() for p in LSTMPTB().parameters()]
    elif name == "vgg16":
        from paper_1911_08727_b200.workloads import vgg16_cifar
        dims = [p.numel() for p in vgg16_cifar().parameters()]
    elif name == "resnet20":
        from paper_1911_08727_b200.workloads import resnet20
        dims = [p.numel() for p in resnet20().parameters()]
    else:
        dims = resnet50_dims()
    ks = ks_for(dims, rho)
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(1)
    gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
    r = torch.zeros(n, device="cuda")
    v = torch.randn(n, device="cuda", generator=gen)
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for t in range(400):
        b.step_local(gs[t % 3], r, 0.1, v, msg, st)
    torch.cuda.synchronize()
    tmp = tempfile.mkdtemp()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for t in range(12):
            b.step_local(gs[t % 3], r, 0.1, v, msg, st)
        torch.cuda.synchronize()
    prof.export_chrome_trace(os.path.join(tmp, "eager.json"))
    show("eager", kernels_from_trace(os.path.join(tmp, "eager.json")))
    cap = torch.cuda.Stream()
    graphs = []
    for i in range(3):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cap):
            b.step_local(gs[i], r, 0.1, v, msg, st, stream=cap)
        graphs.append(gr)
    for t in range(30):
        graphs[t % 3].replay()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for t in range(12):
            graphs[t % 3].replay()
        torch.cuda.synchronize()
    prof.export_chrome_trace(os.path.join(tmp, "graph.json"))
    show("graph replay", kernels_from_trace(os.path.join(tmp, "graph.json")))
    # per-layer CTA spans inside the last selection kernel (globaltimer, ns)
    s = b.stats().astype(np.int64)
    ref = int(s[0, 10])
    rel = lambda x: ((int(x) - ref + 2**31) % 2**32 - 2**31) / 1e3  # noqa: E731  (us, wrap-safe)
    launch = [rel(s[j, 10]) for j in range(len(dims))]
    base = min(launch)
    start = [rel(s[j, 8]) - base for j in range(len(dims))]
    end = [rel(s[j, 9]) - base for j in range(len(dims))]
    launch = [x - base for x in launch]
    rows = sorted(range(len(dims)), key=lambda j: -(end[j] - start[j]))
    print("--- selection CTAs (us from the first CTA launch): launch, start, end, kcycles, path, dim, k, m, "
          "cut bin count")
    for j in rows[:8]:
        print(f"  {launch[j]:7.2f} {start[j]:7.2f} {end[j]:7.2f} {s[j, 4] // 1000:4d} {s[j, 5]} {dims[j]:8d}"
              f" {ks[j]:5d} {s[j, 2]:6d} {int(s[j, 11]) >> 8:5d}")
    print("  latest-ending:", [(dims[j], round(end[j], 2)) for j in sorted(range(len(dims)), key=lambda j: -end[j])[:6]])
    print("  latest-launched:", [(dims[j], round(launch[j], 2))
                                 for j in sorted(range(len(dims)), key=lambda j: -launch[j])[:6]])
    print("  start after griddep wait: min %.2f max %.2f" % (min(start), max(start)))
    ph = lambda w: (int(w) & 2047, (int(w) >> 11) & 2047, (int(w) >> 22) & 2047)  # noqa: E731
    print("  phases x64 cycles (gather, select, compact) of the slowest:", [ph(s[j, 7]) for j in rows[:6]])
    fb = [(dims[j], ks[j], int(s[j, 1]), int(s[j, 3])) for j in range(len(dims)) if s[j, 1]]
    print("  layers with dense fallbacks (dim, k, fallbacks, calls):", fb[:12])
    names = {0: "small-dense", 1: "candidate", 2: "dense-fallback", 3: "cluster"}
    for p in sorted(set(int(x) for x in s[:, 5])):
        js = [j for j in range(len(dims)) if s[j, 5] == p]
        du = np.array([end[j] - start[j] for j in js])
        big = max(js, key=lambda j: dims[j])
        print(f"  path {names.get(p, p)}: {len(js)} layers, us per layer median {np.median(du):.2f} max {du.max():.2f}"
              f" sum {du.sum():.1f}; largest dim {dims[big]} took {end[big] - start[big]:.2f}")
        if p in (0, 1, 3):
            print("    phases of the 4 largest:",
                  [(dims[j], ph(s[j, 7])) for j in sorted(js, key=lambda j: -dims[j])[:4]])


if __name__ == "__main__":
    main()
