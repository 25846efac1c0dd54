"""Multi-GPU parity check (run under torchrun, one process per GPU, NCCL).

Every rank trains the same MLP on its own data with LagsSGD (hook-driven compress on the side
stream -> exchange on the communication stream: the NCCL all-gather, or with `p2p` as the first
argument the peer-memory push -> rank-ordered decode).  Rank 0 gathers every rank's consumed gradients each step and
replays the oracle's lags_step with P = world simulated workers; parameters must match bitwise
on every rank.  Exit code 0 = parity.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lagsgd_oracle as orc  # noqa: E402
from paper_1911_08727_b200.optim import LagsSGD  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    torch.manual_seed(123 + rank)
    model = torch.nn.Sequential(torch.nn.Linear(256, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 1024),
                                torch.nn.ReLU(), torch.nn.Linear(1024, 10)).cuda()
    captured = {}
    for p in model.parameters():
        p.register_post_accumulate_grad_hook(lambda p: captured.__setitem__(id(p), p.grad.detach().clone()))
    mode = sys.argv[1] if len(sys.argv) > 1 else "nccl"
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.01, bucket_cap_bytes=8192, exchange=mode,
                  momentum=float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
    v = opt.params_vector().cpu().numpy().copy()
    res = [np.zeros_like(v) for _ in range(world)]
    ok = True
    for t in range(10):
        x = torch.randn(64, 256, device="cuda")
        y = torch.randint(0, 10, (64,), device="cuda")
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params])
        allg = [torch.zeros_like(g) for _ in range(world)]
        dist.all_gather(allg, g)
        v = orc.lags_step(v, [a.cpu().numpy() for a in allg], 0.05, opt.dims, opt.ks, res)
        if opt.mu == 0.0 and opt.params_vector().cpu().numpy().tobytes() != v.tobytes():
            print(f"rank {rank}: step {t} parameters differ from the oracle", flush=True)
            ok = False
            break
    digest = torch.tensor([float(opt.params_vector().double().sum())], device="cuda")
    all_d = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(all_d, digest)
    same = all(float(d) == float(all_d[0]) for d in all_d)
    flag = torch.tensor([1 if (ok and same) else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"multi-gpu parity world={world} exchange={mode} momentum={opt.mu} buckets={len(opt.buckets)}: "
              f"{'OK' if int(flag) else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) else 1)


if __name__ == "__main__":
    main()
