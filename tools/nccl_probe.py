"""All-gather latency of the bench's sparse message (~205 KB per rank) under the current NCCL
environment; run under torchrun with different NCCL_ALGO / NCCL_PROTO.  Diagnostic only."""

import os

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
for nbytes in (205 << 10, 64 << 10, 1 << 20):
    src = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(world * nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(50):
        dist.all_gather_into_tensor(dst, src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        dist.all_gather_into_tensor(dst, src)
    e1.record()
    torch.cuda.synchronize()
    if rank == 0:
        print(f"ALGO={os.environ.get('NCCL_ALGO', '-')} PROTO={os.environ.get('NCCL_PROTO', '-')} "
              f"world={world} {nbytes >> 10} KB/rank: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us")
dist.destroy_process_group()
