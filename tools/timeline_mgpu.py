"""Kernel timeline of the N > 1 bench step on rank 0 (CUPTI via torch.profiler): compress, the
exchange (NCCL all-gather, or `p2p` as argument: the peer-memory push + wait), decode, and the
gaps between them.  Run under torchrun.  Diagnostic only."""

import json
import os
import sys
import tempfile

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402
from bench import ks_for, resnet50_dims  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = resnet50_dims()
    ks = ks_for(dims)
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32, max_world=world)
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(3)]
    r = torch.zeros(n, device="cuda")
    v = torch.randn(n, device="cuda", generator=gen)
    msg = b.new_messages(1)
    msgs = b.new_messages(world)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")

    peer = None
    if len(sys.argv) > 1 and sys.argv[1] == "p2p":
        from paper_1911_08727_b200.p2p import PeerExchange

        peer = PeerExchange(b.msg_bytes)

    def step(t):
        b.compress(gs[t % 3], r, 0.1, msg, st)
        if peer is not None:
            b.decode(peer.exchange(msg), world, v)
        else:
            dist.all_gather_into_tensor(msgs, msg)
            b.decode(msgs, world, v)

    for t in range(300):
        step(t)
    torch.cuda.synchronize()
    dist.barrier()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for t in range(8):
            step(t)
        torch.cuda.synchronize()
    if rank == 0:
        path = os.path.join(tempfile.mkdtemp(), "t.json")
        prof.export_chrome_trace(path)
        ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
        ev.sort(key=lambda e: e["ts"])
        ev = ev[-15:]
        t0 = ev[0]["ts"]
        prev = None
        for e in ev:
            gap = 0.0 if prev is None else e["ts"] - prev
            print(f"  +{e['ts'] - t0:8.1f} us  dur {e['dur']:6.1f}  gap {gap:5.1f}  {e['name'][:70]}")
            prev = e["ts"] + e["dur"]
    dist.barrier()
    if peer is not None:
        peer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
