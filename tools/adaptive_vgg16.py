"""Config 3: VGG-16 (CIFAR shapes, batch 32/GPU) with adaptive rho_l from measured costs.

Run under torchrun (NCCL).  Steps: train a few iterations at rho = 0.001 with per-layer hook
events and per-bucket compress events enabled; fit an alpha-beta network model to timed NCCL
all-gathers; choose per-layer ratios with the reference's rule (perf.select_ratios); continue
training with the adapted policy and report iteration times before/after.  JSON on rank 0.
"""

import json
import os
import sys

import torch
import torch.distributed as dist
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_08727_b200 import perf  # noqa: E402
from paper_1911_08727_b200.optim import LagsSGD  # noqa: E402
from paper_1911_08727_b200.workloads import synthetic_images, vgg16_cifar  # noqa: E402


def timed(it, n, dev):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(n):
        it()
    e1.record()
    torch.cuda.synchronize(dev)
    t = torch.tensor([e0.elapsed_time(e1) / n], device=dev)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.backends.cudnn.benchmark = True
    torch.manual_seed(0)
    model = vgg16_cifar().to(dev)
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.001, bucket_cap_bytes=1 << 14,
                  exchange=os.environ.get("LAGS_EXCHANGE", "p2p"))
    x, y = synthetic_images(32, 32, 10, dev, seed=rank)

    def it():
        F.cross_entropy(model(x), y).backward()
        opt.step()

    for _ in range(10):
        it()
    before = timed(it, 30, dev)
    opt.enable_layer_timing(True)
    opt.enable_timing(True)
    it()
    bt, st = opt.layer_backward_times(), opt.layer_spar_times()
    sizes, secs = perf.measure_allgather(device=dev)
    net = perf.fit_network(sizes, secs, world)
    pol = opt.adapt(net, ratio_cap=1000.0)
    opt.enable_layer_timing(False)
    opt.enable_timing(False)
    for _ in range(10):
        it()
    after = timed(it, 30, dev)
    if rank == 0:
        ratios = [pol.ratio_for(i + 1) for i in range(len(opt.dims))]
        print(json.dumps({"config": "vgg16-cifar adaptive rho_l", "world": world, "ms_per_iter_rho0.001": before,
                          "ms_per_iter_adaptive": after, "network_fit": {"latency_s": net.latency,
                                                                          "inv_bandwidth_s_per_B": net.inv_bandwidth},
                          "ratios": ratios, "k_total": sum(opt.ks), "dims_total": sum(opt.dims),
                          "buckets": len(opt.buckets), "exchange": opt.exchange_mode,
                          "measured_backward_ms": [round(x * 1e3, 4) for x in bt],
                          "measured_compress_ms": [round(x * 1e3, 4) for x in st]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
