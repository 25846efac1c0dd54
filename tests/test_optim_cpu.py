"""LagsSGD host logic on CPU: fusion buckets (reference rule), hook-driven release-order launches,
world_size-2 gloo exchange, and equivalence with the oracle's lags_step over the same gradients.
The device engine is replaced by tests/stub_engine.py (oracle-backed, test-only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_json
from oracle import lagsgd_oracle as orc
from paper_1911_08727_b200.optim import LagsSGD, plan_buckets, selection_counts
from stub_engine import stub_factory


def test_plan_buckets_follows_reference_fusion_rule():
    # the reference's fusion decisions (tests/golden/wire_cases.json, from R: sparsify.py:209-238)
    for c in load_json("wire_cases.json")["flush"]:
        counts, cap = c["counts"], c["cap"]
        if not counts or c["error"]:
            continue
        # feed the chunks one by one as layers L..1 would arrive; flush decision at the last one
        dims = [64] * len(counts)
        ks = list(reversed([max(x, 1) for x in counts]))
        sizes = [8 + k * 12 for k in ks]
        if max(sizes) >= cap:
            continue
        plan = plan_buckets(dims, ks, cap, value_width=8)
        # rebuild the reference decision for the same stream of chunks
        want, pend, tot = [], [], 0
        for l in range(len(ks) - 1, -1, -1):
            pend.append(l)
            tot += sizes[l]
            if orc.fusion_should_flush([ks[x] for x in pend], cap, l == 0):
                want.append((min(pend), max(pend)))
                pend, tot = [], 0
        assert plan == want
    # every layer lands in exactly one bucket, buckets are contiguous and in release order
    dims = [100, 3, 5000, 7, 64, 20000]
    ks = selection_counts(dims, [10.0] * 6)
    plan = plan_buckets(dims, ks, 200)
    covered = sorted(l for lo, hi in plan for l in range(lo, hi + 1))
    assert covered == list(range(6))
    assert [hi for _, hi in plan] == sorted([hi for _, hi in plan], reverse=True)


class Tiny(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(12, 16)
        self.b = torch.nn.Linear(16, 8)
        self.c = torch.nn.Linear(8, 3)

    def forward(self, x):
        return self.c(torch.tanh(self.b(torch.tanh(self.a(x)))))


def consumed_grad(opt):
    """Flat gradient as the optimizer's compress calls saw it (before the fused zero_grad)."""
    g = np.zeros(sum(opt.dims), dtype=np.float32)
    ref = opt.ref_offsets
    for b in opt.buckets:
        g[ref[b.lo]:ref[b.lo] + b.numel] = b.engine.last_g
    return g


def _run_single(steps, rho, cap, mu=0.0):
    torch.manual_seed(0)
    model = Tiny()
    opt = LagsSGD(model.parameters(), lr=0.1, rho=rho, momentum=mu, bucket_cap_bytes=cap,
                  engine_factory=stub_factory)
    v = opt.params_vector().detach().numpy().copy()
    dims = opt.dims
    ks = opt.ks
    res = [np.zeros_like(v)]
    for t in range(steps):
        x = torch.randn(5, 12, generator=torch.Generator().manual_seed(100 + t))
        y = torch.randint(0, 3, (5,), generator=torch.Generator().manual_seed(200 + t))
        loss = torch.nn.functional.cross_entropy(model(x), y)
        loss.backward()
        opt.step()
        g = consumed_grad(opt)
        if mu == 0.0:
            v = orc.lags_step(v, [g], 0.1, dims, ks, res)
            assert opt.params_vector().numpy().tobytes() == v.tobytes(), t
        assert not np.any(opt.flat_grad.numpy()), "compress must clear the gradients"
    return opt


def test_single_rank_matches_oracle_and_hooks_launch_in_order():
    opt = _run_single(6, rho=0.25, cap=64)
    assert len(opt.buckets) > 1
    assert all(b.engine.calls == 6 for b in opt.buckets)
    # param views stay attached to the flat buffers
    for p, off, d in zip(opt.params, opt.offsets, opt.dims):
        assert p.data.data_ptr() == opt.flat_param[off:off + d].data_ptr()


def test_momentum_runs_and_state_dict_resumes():
    opt = _run_single(3, rho=0.5, cap=1 << 20, mu=0.9)
    sd = opt.state_dict()
    assert sd["lags"]["residual"].numel() == sum(opt.dims)  # the reference's layout, no padding
    r0 = opt.residual.clone()
    opt.residual.zero_()
    opt.load_state_dict(sd)
    assert torch.equal(opt.residual, r0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(1 + rank)  # different init per rank: LagsSGD must broadcast rank 0's
        model = Tiny()
        opt = LagsSGD(model.parameters(), lr=0.05, rho=0.2, bucket_cap_bytes=96, engine_factory=stub_factory,
                      delta_every=2)
        v = opt.params_vector().detach().numpy().copy()
        res = [np.zeros_like(v) for _ in range(world)]
        for t in range(steps):
            x = torch.randn(4, 12, generator=torch.Generator().manual_seed(10 * t + rank))
            y = torch.randint(0, 3, (4,), generator=torch.Generator().manual_seed(10 * t + rank + 5))
            torch.nn.functional.cross_entropy(model(x), y).backward()
            opt.step()
            g = torch.from_numpy(consumed_grad(opt))
            gathered = [torch.zeros_like(g) for _ in range(world)]
            dist.all_gather(gathered, g)
            accs = [res[p] + 0.05 * gathered[p].numpy() for p in range(world)]  # before lags_step mutates res
            v = orc.lags_step(v, [x.numpy() for x in gathered], 0.05, opt.dims, opt.ks, res)
            if opt.params_vector().numpy().tobytes() != v.tobytes():
                out.put((rank, f"step {t}: params differ from the oracle"))
                return
            if (t + 1) % 2 == 0:  # delta^(l) logged on this step (R: training.py:320-337)
                step, got = opt.last_delta()
                want = [orc.topk_aggregation_ratio([a[o:o + d] for a in accs], k)
                        for o, d, k in zip(opt.ref_offsets, opt.dims, opt.ks)]
                if step != t + 1 or got != want:
                    out.put((rank, f"step {t}: delta {got} != {want}"))
                    return
        out.put((rank, opt.params_vector().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_oracle_lags_step():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in results.items():
        assert isinstance(v, bytes), v
    assert results[0] == results[1], "ranks must hold bit-identical parameters"
