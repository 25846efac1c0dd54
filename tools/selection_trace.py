"""Trace the predicted-threshold machinery on the bench workload (ResNet-50 layer shapes).

Prints, every `--every` steps: compress time (CUDA events), total candidates, dense fallbacks
so far, and the worst layers by candidates/k.  Diagnostic only (not part of the product).
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--every", type=int, default=25)
    ap.add_argument("--buffers", type=int, default=3)
    ap.add_argument("--rho", type=float, default=0.001)
    args = ap.parse_args()
    dims = resnet50_dims()
    ks = ks_for(dims, args.rho)
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(args.buffers)]
    r = torch.zeros(n, device="cuda")
    v = torch.randn(n, device="cuda", generator=gen)
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for t in range(args.steps):
        ev0.record()
        b.compress(gs[t % len(gs)], r, 0.1, msg, st)
        ev1.record()
        b.decode(msg, 1, v)
        torch.cuda.synchronize()
        times.append(ev0.elapsed_time(ev1))
        if (t + 1) % args.every == 0:
            s = b.stats()
            big = [j for j, d in enumerate(dims) if d > 16384]
            ratio = [(s[j, 2] / ks[j], j) for j in big]
            ratio.sort(reverse=True)
            print(f"step {t + 1:4d}  compress {np.median(times[-args.every:]) * 1e3:8.1f} us (median)  "
                  f"cands {int(s[:, 2].sum()):7d} (2k={2 * sum(ks[j] for j in big)})  fallbacks {int(s[:, 1].sum()):5d}  "
                  f"worst m/k {[(round(float(x), 1), dims[j]) for x, j in ratio[:4]]}", flush=True)
            slow = np.argsort(-s[:, 4].astype(np.int64))[:6]
            print("   slowest layers (kcycles, path, dim, k, m):",
                  [(int(s[j, 4]) // 1000, int(s[j, 5]), dims[j], ks[j], int(s[j, 2])) for j in slow], flush=True)
            ph = lambda w: (int(w) & 2047, (int(w) >> 11) & 2047, (int(w) >> 22) & 2047)  # noqa: E731
            print("   candidate-path phases x64 cycles (gather, select, compact):",
                  [ph(s[j, 7]) for j in slow], flush=True)
            print("   histogram cut (code 0 = resolved, cut bin's count):",
                  [(int(s[j, 11]) & 0xff, int(s[j, 11]) >> 8) for j in slow], flush=True)


if __name__ == "__main__":
    main()
