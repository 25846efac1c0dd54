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


def close(got, want, rel=None, abs_=0.0):
    if want is None or (isinstance(want, float) and math.isnan(want)):
        return got is None
    return got is not None and abs(got - want) <= max((RTOL if rel is None else rel) * max(1e-300, abs(want)), abs_)


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


def test_lagssgd_residual_identity_monitor():
    """The residual-identity monitor (R: training.py:356-369): a dense fp64 shadow sequence x
    advanced with every step's gradient (R: training.py:197-200) and, on logged steps, ||v - x||,
    max |(v - x) - mean residual| and the per-layer mean-residual norms -- against the same
    quantities computed in numpy from the oracle's parameter and residual trajectory (the
    optimizer's own trajectory is bit-exact to it, test_gpu_optim.py).  Eq. 10 holds: the deviation
    is rounding-sized next to the residual."""
    from paper_1911_08727_b200.optim import LagsSGD

    torch.manual_seed(7)
    model = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.Tanh(), torch.nn.Linear(128, 10)).cuda()
    captured = {}
    for p in model.parameters():
        p.register_post_accumulate_grad_hook(lambda p: captured.__setitem__(id(p), p.grad.detach().clone()))
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.05, monitor_every=2, bucket_cap_bytes=512)
    assert len(opt.buckets) > 1
    v = opt.params_vector().cpu().numpy().copy()
    x = v.astype(np.float64)
    res = [np.zeros_like(v)]
    off = np.concatenate([[0], np.cumsum(opt.dims)])
    for t in range(6):
        xin = torch.randn(32, 64, device="cuda")
        y = torch.randint(0, 10, (32,), device="cuda")
        torch.nn.functional.cross_entropy(model(xin), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params]).cpu().numpy()
        v = orc.lags_step(v, [g], 0.05, opt.dims, opt.ks, res)
        x = x - (0.05 * g.astype(np.float64)) / 1.0
        if (t + 1) % 2 == 0:
            step, got = opt.last_identity()
            assert step == t + 1
            gap = v.astype(np.float64) - x
            mres = res[0].astype(np.float64)
            assert close(got["v_x_gap"], float(np.sqrt(gap @ gap)), rel=1e-9)
            assert close(got["resid_dev"], float(np.max(np.abs(gap - mres))), rel=1e-6, abs_=1e-12)
            want = [float(np.sqrt(mres[a:b] @ mres[a:b])) for a, b in zip(off[:-1], off[1:])]
            assert all(close(a, b, rel=1e-9) for a, b in zip(got["residual_norms"], want))
            assert got["resid_dev"] < 1e-5 * max(got["residual_norms"])  # Eq. 10 up to fp32 rounding of v
