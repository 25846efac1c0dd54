"""Device delta^(l) diagnostic (lags_bucket_reconstruct / lags_bucket_delta) against the reference's
analysis.topk_aggregation_ratio outputs (tests/golden/delta_cases.npz) and the oracle.  The fp64
sums follow the reference's order; only the final dot products' summation order differs from
numpy's BLAS dot, hence rtol 1e-12."""

import math

import numpy as np
import pytest
import torch

from conftest import load_npz
from oracle import lagsgd_oracle as orc

pytestmark = pytest.mark.gpu

import paper_1911_08727_b200 as L  # noqa: E402
from paper_1911_08727_b200 import _native as N  # noqa: E402

RTOL = 1e-12


def close(got, want):
    if want is None or (isinstance(want, float) and math.isnan(want)):
        return got is None
    return got is not None and abs(got - want) <= RTOL * max(1e-300, abs(want))


def test_topk_aggregation_ratio_golden():
    z = load_npz("delta_cases.npz")
    for i in range(int(z["n"])):
        P, d, k = (int(v) for v in z[f"meta{i}"])
        want = float(z[f"delta{i}"])
        got = L.topk_aggregation_ratio(list(z[f"x{i}"]), k)
        assert close(got, None if math.isnan(want) else want), (i, got, want)


def test_topk_aggregation_ratio_errors():
    with pytest.raises(L.StructureError):
        L.topk_aggregation_ratio([], 1)
    with pytest.raises(L.StructureError):
        L.topk_aggregation_ratio([np.ones(3), np.ones(4)], 1)
    with pytest.raises(ValueError):
        L.topk_aggregation_ratio([np.ones(3)], 4)


@pytest.mark.parametrize("P", [1, 3])
def test_bucket_delta_matches_oracle(P):
    dims = [4097, 36864, 64, 16385, 1000]
    ks = [max(1, d // 100) for d in dims]
    n = sum(dims)
    S = (n + 3) // 4 * 4  # plane stride: every plane 16-byte aligned
    b = L.Bucket(dims, ks, N.F32, max_world=P)
    gen = torch.Generator(device="cuda").manual_seed(11)
    r = torch.zeros(P * S, device="cuda")
    msgs = b.new_messages(P)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    accs = None
    for step in range(3):
        gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(P)]
        accs = [(r[p * S:p * S + n].cpu().numpy() + np.float32(0.1) * gs[p].cpu().numpy()) for p in range(P)]
        for p in range(P):
            b.compress(gs[p], r[p * S:p * S + n], 0.1, msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes], st)
    acc = torch.empty_like(r)
    b.reconstruct(msgs, P, r, acc, plane_stride=S)
    planes = acc.cpu().numpy().reshape(P, S)[:, :n]
    assert np.array_equal(planes, np.stack(accs)), "acc_p = r_p + sent_p must be exact"
    got = b.delta(acc, r, P, plane_stride=S).cpu().numpy()
    off = np.concatenate([[0], np.cumsum(dims)[:-1]])
    for j, (o, d, k) in enumerate(zip(off, dims, ks)):
        want = orc.topk_aggregation_ratio([a[o:o + d] for a in accs], k)
        assert close(None if math.isnan(got[j]) else float(got[j]), want), (j, got[j], want)


def test_optimizer_logs_delta_single_rank():
    from paper_1911_08727_b200.optim import LagsSGD

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.Tanh(), torch.nn.Linear(128, 10)).cuda()
    captured = {}

    def grab(p):
        captured[id(p)] = p.grad.detach().clone()

    for p in model.parameters():  # registered before the optimizer's hooks -> runs first
        p.register_post_accumulate_grad_hook(grab)
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.05, delta_every=2)
    res = np.zeros(sum(opt.dims), dtype=np.float32)
    for t in range(4):
        x = torch.randn(32, 64, device="cuda")
        y = torch.randint(0, 10, (32,), device="cuda")
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params]).cpu().numpy()
        acc = res + np.float32(0.05) * g
        res = opt.residual_vector().cpu().numpy().copy()
        if (t + 1) % 2 == 0:
            step, got = opt.last_delta()
            assert step == t + 1
            for o, d, k, dv in zip(opt.ref_offsets, opt.dims, opt.ks, got):
                assert close(dv, orc.topk_aggregation_ratio([acc[o:o + d]], k))
