"""Host<->device copy bandwidth on this box (pinned memory): H2D, D2H, and both at once on two
streams; plus the phase timing of one pipelined drop-in lags_step.  Diagnostic only."""

import json
import time

import numpy as np
import torch


def bw(n_bytes=102 << 20, reps=5):
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in [
        ("h2d", lambda: d.copy_(h, non_blocking=True)),
        ("d2h", lambda: h.copy_(d, non_blocking=True)),
    ]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[name + "_GBs"] = round(reps * n_bytes / (time.perf_counter() - t0) / 1e9, 2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    out["bidir_each_GBs"] = round(reps * n_bytes / (time.perf_counter() - t0) / 1e9, 2)
    # 3 x H2D back to back (the step's 306 MB up) with 2 x D2H (204 MB down) concurrently
    hs = [torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(5)]
    ds = [torch.empty(n_bytes, dtype=torch.uint8, device="cuda") for _ in range(5)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        for i in range(3):
            ds[i].copy_(hs[i], non_blocking=True)
    with torch.cuda.stream(s2):
        for i in range(3, 5):
            hs[i].copy_(ds[i], non_blocking=True)
    torch.cuda.synchronize()
    out["step_like_306up_204down_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    return out


if __name__ == "__main__":
    print(json.dumps(bw()))
