"""Where does a ResNet-50 training iteration spend GPU time: LagsSGD vs plain SGD (N = 1).

CUPTI kernel records via torch.profiler; per iteration: kernels grouped by family, busy time of
the device (union of kernel intervals) and the span.  Diagnostic only.
"""

import collections
import json
import os
import sys
import tempfile

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_08727_b200.optim import LagsSGD  # noqa: E402
from paper_1911_08727_b200.workloads import resnet50, synthetic_images  # noqa: E402


def family(name: str) -> str:
    n = name.lower()
    if "lags::" in n or "accum_emit" in n or "select_" in n:
        return "lags"
    if "multi_tensor" in n or "foreach" in n:
        return "optimizer(foreach)"
    if "elementwise" in n or "vectorized" in n:
        return "elementwise"
    if "gemm" in n or "cutlass" in n or "sm90" in n or "sm100" in n or "xmma" in n or "conv" in n or "cudnn" in n:
        return "conv/gemm"
    if "batch_norm" in n or "bn_" in n:
        return "batchnorm"
    if "reduce" in n:
        return "reduce"
    return "other"


def profile(kind, iters=5):
    dev = torch.device("cuda")
    torch.backends.cudnn.benchmark = True
    x, y = synthetic_images(64, 224, 1000, dev, seed=0)
    torch.manual_seed(0)
    model = resnet50().to(dev)
    if kind == "sgd":
        opt = torch.optim.SGD(model.parameters(), lr=0.1)
    else:
        opt = LagsSGD(model.parameters(), lr=0.1, rho=0.001, bucket_cap_bytes=65536)

    def it():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = F.cross_entropy(model(x), y)
        loss.backward()
        opt.step()
        if kind == "sgd":
            opt.zero_grad(set_to_none=True)

    for _ in range(10):
        it()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        it()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    tmp = tempfile.mkdtemp()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(iters):
            it()
        torch.cuda.synchronize()
    path = os.path.join(tmp, f"{kind}.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    fam = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        f = family(e["name"])
        fam[f][0] += 1
        fam[f][1] += e["dur"]
    # busy = union of kernel intervals
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:
        s, t = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, t
        else:
            cur_e = max(cur_e, t)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
    out = {"kind": kind, "ms_per_iter_events": round(ms, 3), "kernels_per_iter": round(len(ev) / iters, 1),
           "busy_us_per_iter": round(busy / iters, 1), "span_us_per_iter": round(span / iters, 1),
           "families_us_per_iter": {k: (round(v[0] / iters, 1), round(v[1] / iters, 1)) for k, v in
                                    sorted(fam.items(), key=lambda kv: -kv[1][1])}}
    top = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        top[e["name"][:90]][0] += 1
        top[e["name"][:90]][1] += e["dur"]
    out["top_kernels"] = [(k, round(v[0] / iters, 1), round(v[1] / iters, 1))
                          for k, v in sorted(top.items(), key=lambda kv: -kv[1][1])[:12]]
    if kind == "lags":
        opt.remove_hooks()
    return out


if __name__ == "__main__":
    for kind in sys.argv[1:] or ["sgd", "lags"]:
        print(json.dumps(profile(kind), indent=1))
