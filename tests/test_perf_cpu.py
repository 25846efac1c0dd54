"""Adaptive ratio selector (product perf.py) against the reference's own outputs (golden), the
network-model fit, and LagsSGD re-planning under a new policy (CPU, stub engine)."""

import numpy as np
import pytest
import torch

from conftest import load_json
from paper_1911_08727_b200 import CompressionPolicy
from paper_1911_08727_b200 import perf


def test_select_ratios_matches_reference_golden():
    cases = load_json("perf_cases.json")
    assert len(cases["select"]) >= 50
    for c in cases["select"]:
        net = perf.NetworkModel(c["lat"], c["inv_bw"])
        pol = perf.select_ratios(c["dims"], c["bwd"], c["spar"], net, c["P"], c["cap"],
                                 entry_bytes=perf.REFERENCE_ENTRY_BYTES)
        assert [pol.ratio_for(i + 1) for i in range(len(c["dims"]))] == c["ratios"]
    for c in cases["pipelined"]:
        net = perf.NetworkModel(c["lat"], c["inv_bw"])
        comm = [perf.comm_time(d, r, net, c["P"], perf.REFERENCE_ENTRY_BYTES) for d, r in zip(c["dims"], c["ratios"])]
        assert comm == c["comm"]
        assert perf.pipelined_makespan(1e-3, c["bwd"], c["spar"], comm) == c["makespan"]
    for c in cases["comm"]:
        net = perf.NetworkModel(c["lat"], c["inv_bw"])
        assert perf.comm_time(c["dim"], c["ratio"], net, c["P"], perf.REFERENCE_ENTRY_BYTES) == c["t"]


def test_select_ratios_reference_spot_cases():
    # R: tests/test_perf.py:241-291
    free = perf.select_ratios([100, 100, 100], [1.0] * 3, [0.0] * 3, perf.NetworkModel(1e-6, 1e-9), 4, 1000,
                              ratio_grid=(1, 10, 100, 1000))
    assert all(c == 1.0 for c in free.per_layer_ratio.values())
    net = perf.NetworkModel(0.0, 1.2 / (12000 * 12.0), multiplier=lambda p: 1.0)
    pol = perf.select_ratios([12000, 12000], [0.010, 0.010], [0.001, 0.001], net, 2, 1000,
                             ratio_grid=(1, 10, 100, 1000), entry_bytes=12)
    assert pol.ratio_for(2) == 1000.0
    cap = perf.select_ratios([1000, 1000], [0.001, 0.001], [0.01, 0.01], perf.NetworkModel(1e-5, 1e-9), 2, 500,
                             ratio_grid=(1, 10, 100, 500))
    assert all(c == 500.0 for c in cap.per_layer_ratio.values())
    with pytest.raises(ValueError):
        perf.select_ratios([10], [1.0], [0.0], perf.NetworkModel(0, 0), 2, 10, ratio_grid=())


def test_fit_network_recovers_alpha_beta():
    sizes = [256, 4096, 65536, 1 << 20]
    true = perf.NetworkModel(8e-6, 1.0 / 300e9)
    times = [true.message_time(s, 8) for s in sizes]
    fit = perf.fit_network(sizes, times, 8)
    assert abs(fit.latency - true.latency) / true.latency < 1e-6
    assert abs(fit.inv_bandwidth - true.inv_bandwidth) / true.inv_bandwidth < 1e-6


def test_lagssgd_set_policy_replans_buckets():
    from paper_1911_08727_b200.optim import LagsSGD
    from stub_engine import stub_factory

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(32, 64), torch.nn.Tanh(), torch.nn.Linear(64, 4))
    opt = LagsSGD(model.parameters(), lr=0.1, rho=0.5, bucket_cap_bytes=128, engine_factory=stub_factory)
    before = list(opt.ks)
    r0 = opt.residual_vector()
    L = len(opt.dims)
    opt.set_policy(CompressionPolicy({i + 1: 10.0 for i in range(L)}, 10.0))
    assert opt.ks == [min(d, max(1, d // 10)) for d in opt.dims] and opt.ks != before
    assert torch.equal(opt.residual_vector(), r0)  # carried over through the re-layout
    covered = sorted(l for b in opt.buckets for l in range(b.lo, b.hi + 1))
    assert covered == list(range(L))
    x = torch.randn(3, 32)
    model(x).sum().backward()
    opt.step()
    assert all(b.engine.calls == 1 for b in opt.buckets)
    assert np.all(np.isfinite(opt.flat_param.numpy()))
