"""The hot-path step (P = 1: compress with the fused update, CUDA-graph replay) over the layer
shapes of every SURVEY config: ResNet-20, VGG-16-CIFAR, ResNet-50, LSTM-PTB at rho = 0.001 (plus
ResNet-50 at rho = 0.01), and the fp64 / mixed-precision modes.  Reports us/step, algorithmic GB/s, the fraction of the measured HBM
copy peak, dense fallbacks, and which selection paths the layers took.  Diagnostic only."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from paper_1911_08727_b200.workloads import LSTMPTB, resnet20, resnet50, vgg16_cifar  # noqa: E402


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return None


def run(name, dims, rho, steps=100, f64=False, acc64=False):
    """f64: LAGS_F64 buckets; acc64: LAGS_F32_ACC64 (fp32 storage, fp64 acc and values)."""
    ks = [min(d, max(1, int(d // (1.0 / rho)))) for d in dims]
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F64 if f64 else (N.F32_ACC64 if acc64 else N.F32))
    dt = torch.float64 if f64 else torch.float32
    gen = torch.Generator(device="cuda").manual_seed(5)
    gs = [torch.randn(n, device="cuda", generator=gen, dtype=dt) for _ in range(3)]
    r = torch.zeros(n, device="cuda", dtype=dt)
    v = torch.randn(n, device="cuda", generator=gen, dtype=dt)
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for t in range(60):
        b.step_local(gs[t % 3], r, 0.1, v, msg, st)
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    graphs = []
    for i in range(3):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            b.step_local(gs[i], r, 0.1, v, msg, st, stream=cap)
        graphs.append(g)
    for t in range(6):
        graphs[t % 3].replay()
    torch.cuda.synchronize()
    s0 = b.stats().astype(np.int64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(steps):
        graphs[t % 3].replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    s1 = b.stats().astype(np.int64)
    paths = {}
    for p in s1[:, 5]:
        paths[int(p)] = paths.get(int(p), 0) + 1
    # algorithmic bytes: compress 12 d + 8 n_sel (fp32) / 24 d + 12 n_sel (fp64, and 12 d + 12 n_sel
    # for fp32 storage with fp64 values); the fp64 / mixed steps also run the P = 1 decode (weight
    # read + write per touched entry + the 12 B pair)
    k = sum(ks)
    byts = (24 * n + 12 * k + 28 * k) if f64 else ((12 * n + 12 * k + 20 * k) if acc64 else (12 * n + 8 * k))
    gbs = byts / (ms * 1e-3) / 1e9
    pk = peak_gbs()
    assert int(st.item()) == 0
    return {"config": name, "dtype": "f64" if f64 else ("f32/acc64" if acc64 else "f32"), "rho": rho, "layers": len(dims), "elements": n,
            "max_layer": max(dims),
            "sum_k": sum(ks), "us_per_step": round(ms * 1e3, 1), "GBs": round(gbs, 1),
            "frac_of_copy_peak": round(gbs / pk, 3) if pk else None,
            "dense_fallbacks_in_timed_steps": int((s1[:, 1] - s0[:, 1]).sum()),
            "paths": ({{0: "small/tiny", 1: "candidate", 2: "dense", 3: "cluster", 4: "cluster (radix)"}[k]: v
                       for k, v in sorted(paths.items())} if not (f64 or acc64) else
                      {{0: "small", 1: "candidate", 2: "dense"}[k]: v for k, v in sorted(paths.items())})}


def main():
    configs = [
        ("resnet20 (config 2)", [p.numel() for p in resnet20().parameters()], 0.001),
        ("vgg16-cifar (config 3)", [p.numel() for p in vgg16_cifar().parameters()], 0.001),
        ("resnet50 (config 4)", [p.numel() for p in resnet50().parameters()], 0.001),
        ("resnet50 (config 4)", [p.numel() for p in resnet50().parameters()], 0.01),
        ("lstm-ptb (config 5)", [p.numel() for p in LSTMPTB().parameters()], 0.001),
    ]
    only = sys.argv[1:]
    for name, dims, rho in configs:
        if not only or "f32" in only:
            print(json.dumps(run(name, dims, rho)), flush=True)
    if not only or "f64" in only:  # the reference's default dtype (R: layered.py:88-90)
        print(json.dumps(run("mlp 64-16-4 (config 1)", [1040, 68], 0.01, f64=True)), flush=True)
        print(json.dumps(run("resnet50 (config 4)", [p.numel() for p in resnet50().parameters()], 0.001, f64=True)),
              flush=True)
    if not only or "acc64" in only:  # fp32 storage with a numpy-float64 alpha (R: training.py:250, NEP 50)
        print(json.dumps(run("resnet50 (config 4)", [p.numel() for p in resnet50().parameters()], 0.001, acc64=True)),
              flush=True)


if __name__ == "__main__":
    main()
