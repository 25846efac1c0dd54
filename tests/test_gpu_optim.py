"""LagsSGD on the B200 (real CUDA buckets, hook-driven side-stream launches) against the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lagsgd_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1911_08727_b200 as lib

    return lib


class MLP(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.l1 = torch.nn.Linear(256, 512)
        self.l2 = torch.nn.Linear(512, 512)
        self.l3 = torch.nn.Linear(512, 10)

    def forward(self, x):
        return self.l3(torch.relu(self.l2(torch.relu(self.l1(x)))))


def test_lagssgd_matches_oracle(L):
    from paper_1911_08727_b200.optim import LagsSGD

    torch.manual_seed(0)
    model = MLP().cuda()
    captured = {}

    def grab(p):
        captured[id(p)] = p.grad.detach().clone()

    for p in model.parameters():  # registered before the optimizer's hooks -> runs first
        p.register_post_accumulate_grad_hook(grab)
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.01, bucket_cap_bytes=4096)
    assert len(opt.buckets) > 1
    v = opt.params_vector().cpu().numpy().copy()
    res = [np.zeros_like(v)]
    for t in range(8):
        x = torch.randn(32, 256, device="cuda")
        y = torch.randint(0, 10, (32,), device="cuda")
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params]).cpu().numpy()
        v = orc.lags_step(v, [g], 0.05, opt.dims, opt.ks, res)
        assert opt.params_vector().cpu().numpy().tobytes() == v.tobytes(), t
        assert opt.residual_vector().cpu().numpy().tobytes() == res[0].tobytes(), t
        if opt.flat_grad is not None:
            assert not torch.any(opt.flat_grad), "compress clears the gradients"
        else:
            assert all(p.grad is None for p in opt.params), "gradient tensors are released to autograd"
    # the model's parameters are views of the updated flat buffer
    w = model.l1.weight.detach().reshape(-1).cpu().numpy()
    assert w.tobytes() == v[:w.size].tobytes()


def test_lagssgd_divergence(L):
    from paper_1911_08727_b200.optim import LagsSGD

    model = MLP().cuda()
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.01)
    out = model(torch.randn(4, 256, device="cuda")).sum() * float("nan")
    out.backward()
    opt.step()  # the flag is read back asynchronously ...
    with pytest.raises(L.DivergenceError):
        opt.check_divergence()  # ... or synchronously on demand
    torch.cuda.synchronize()
    with pytest.raises(L.DivergenceError):
        for _ in range(3):  # ... and surfaces at a later step() once the copy has landed
            model(torch.randn(4, 256, device="cuda")).sum().backward()
            opt.step()
            torch.cuda.synchronize()


class Odd(torch.nn.Module):
    """Odd parameter sizes: layer offsets that are not multiples of 4 elements (the per-layer
    gradient tensors are then aligned differently from the flat residual -> scalar K1 tasks)."""

    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(37, 301)
        self.b = torch.nn.Linear(301, 7)
        self.c = torch.nn.Linear(7, 3)

    def forward(self, x):
        return self.c(torch.tanh(self.b(torch.tanh(self.a(x)))))


@pytest.mark.parametrize("model_cls", [MLP, Odd])
def test_grad_modes_bit_identical(L, model_cls):
    """grads="tensors" (autograd tensors through the device pointer table) == grads="flat"."""
    from paper_1911_08727_b200.optim import LagsSGD

    outs = {}
    for mode in ("flat", "tensors"):
        torch.manual_seed(3)
        model = model_cls().cuda()
        opt = LagsSGD(model.parameters(), lr=0.05, rho=0.02, bucket_cap_bytes=2048, grads=mode)
        assert opt.grads_mode == mode
        gen = torch.Generator(device="cuda").manual_seed(9)
        nin = model.l1.in_features if hasattr(model, "l1") else model.a.in_features
        for t in range(6):
            x = torch.randn(16, nin, device="cuda", generator=gen)
            y = torch.randint(0, 3, (16,), device="cuda", generator=gen)
            torch.nn.functional.cross_entropy(model(x), y).backward()
            opt.step()
        torch.cuda.synchronize()
        outs[mode] = (opt.params_vector().cpu().numpy().tobytes(), opt.residual_vector().cpu().numpy().tobytes())
        opt.remove_hooks()
    assert outs["flat"] == outs["tensors"]


def _train_vs_oracle(opt, model, steps, gen, nin, ncls, captured, v, res):
    """Run steps of LagsSGD and the oracle's lags_step side by side; bit-exact every step."""
    for t in range(steps):
        x = torch.randn(16, nin, device="cuda", generator=gen)
        y = torch.randint(0, ncls, (16,), device="cuda", generator=gen)
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params]).cpu().numpy()
        lr = opt.param_groups[0]["lr"]
        v = orc.lags_step(v, [g], lr, opt.dims, opt.ks, res)
        assert opt.params_vector().cpu().numpy().tobytes() == v.tobytes(), t
        assert opt.residual_vector().cpu().numpy().tobytes() == res[0].tobytes(), t
    return v


def _capture(model):
    captured = {}

    def grab(p):
        captured[id(p)] = p.grad.detach().clone()

    for p in model.parameters():  # registered before the optimizer's hooks -> runs first
        p.register_post_accumulate_grad_hook(grab)
    return captured


def test_adapt_from_device_timings_matches_oracle_rule(L):
    """Config 3's mechanism on one GPU: LagsSGD.adapt feeds the reference's selector (R: perf.py:231-260)
    with the hook-event backward times and the bucket compress times of the last step; the chosen
    ratios must be the oracle's select_ratios on exactly those inputs, and training continues
    bit-exact against the oracle's lags_step with the new per-layer k_l."""
    from paper_1911_08727_b200 import perf
    from paper_1911_08727_b200.optim import LagsSGD

    torch.manual_seed(1)
    model = MLP().cuda()
    captured = _capture(model)
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.001, bucket_cap_bytes=4096)
    gen = torch.Generator(device="cuda").manual_seed(5)
    v = opt.params_vector().cpu().numpy().copy()
    res = [np.zeros_like(v)]
    v = _train_vs_oracle(opt, model, 3, gen, 256, 10, captured, v, res)
    opt.enable_layer_timing(True)
    opt.enable_timing(True)
    v = _train_vs_oracle(opt, model, 1, gen, 256, 10, captured, v, res)
    bt, st = opt.layer_backward_times(), opt.layer_spar_times()
    assert all(x > 0 for x in bt) and all(x >= 0 for x in st)
    # a slow network priced for 8 workers, so the choice depends on the measured times
    net = perf.NetworkModel(latency=2e-6, inv_bandwidth=1.0 / 5e9)
    pol = opt.adapt(net, ratio_cap=1000.0, workers=8)
    want = orc.select_ratios(opt.dims, bt, st, net.latency, net.inv_bandwidth, 8, 1000.0,
                             ratio_grid=LagsSGD.ADAPT_GRID, entry_bytes=perf.DEVICE_ENTRY_BYTES)
    got = {i + 1: pol.ratio_for(i + 1) for i in range(len(opt.dims))}
    assert got == {int(k): float(c) for k, c in want.items()}, (got, want)
    assert opt.ks == [orc.selection_count(d, got[i + 1]) for i, d in enumerate(opt.dims)]
    opt.enable_layer_timing(False)
    opt.enable_timing(False)
    _train_vs_oracle(opt, model, 4, gen, 256, 10, captured, v, res)


def test_odd_model_small_buckets_unaligned_offsets(L):
    """Buckets whose first element is not 16-byte aligned in the reference layout: with the Odd
    model's sizes and a 1 KiB fusion capacity the buckets start at element offsets like 11137.
    The padded flat layout keeps every bucket aligned; results stay bit-exact vs the oracle."""
    from paper_1911_08727_b200.optim import LagsSGD

    torch.manual_seed(2)
    model = Odd().cuda()
    captured = _capture(model)
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.02, bucket_cap_bytes=1024)
    assert len(opt.buckets) > 1
    ref = opt.ref_offsets
    assert any(ref[b.lo] % 4 for b in opt.buckets), "the test needs an unaligned bucket start"
    assert all(b.offset % 4 == 0 for b in opt.buckets)
    v = opt.params_vector().cpu().numpy().copy()
    res = [np.zeros_like(v)]
    _train_vs_oracle(opt, model, 6, torch.Generator(device="cuda").manual_seed(3), 37, 3, captured, v, res)


def test_compress_accepts_unaligned_buffers(L):
    """The C ABI takes element-aligned (not 16-byte aligned) g / r / v: results equal the aligned run."""
    from paper_1911_08727_b200 import _native as N

    dims = [70_001, 3, 40_000]
    ks = [70, 1, 40]
    n = sum(dims)
    outs = []
    for shift in (0, 1, 3):
        b = L.Bucket(dims, ks, N.F32)
        gen = torch.Generator(device="cuda").manual_seed(8)
        gbuf = torch.zeros(n + 4, device="cuda")
        rbuf = torch.zeros(n + 4, device="cuda")
        vbuf = torch.zeros(n + 4, device="cuda")
        v = vbuf[shift:shift + n]
        v.copy_(torch.randn(n, device="cuda", generator=gen))
        msg = b.new_messages(1)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        for t in range(4):
            g = gbuf[(shift + t) % 4:(shift + t) % 4 + n]
            g.copy_(torch.randn(n, device="cuda", generator=gen))
            b.step_local(g, rbuf[shift:shift + n], 0.1, v, msg, st)
        torch.cuda.synchronize()
        outs.append((v.cpu().numpy().tobytes(), rbuf[shift:shift + n].cpu().numpy().tobytes(), msg.cpu().numpy().tobytes()))
    assert outs[0] == outs[1] == outs[2]


def test_second_backward_before_step_raises(L):
    """Gradients are consumed during backward: a second backward() before step() would be lost, so
    the hook refuses it."""
    from paper_1911_08727_b200.optim import LagsSGD

    model = MLP().cuda()
    opt = LagsSGD(model.parameters(), lr=0.05, rho=0.01)
    x = torch.randn(4, 256, device="cuda")
    model(x).sum().backward()
    with pytest.raises(RuntimeError, match="step"):
        model(x).sum().backward()


def test_state_dict_resume_bit_exact(L):
    """True resume: params + optimizer state (residual, momentum, ratios) saved after 3 steps and
    loaded into a fresh model/optimizer reproduce the uninterrupted run bit for bit."""
    from paper_1911_08727_b200.optim import LagsSGD

    def batches():
        gen = torch.Generator(device="cuda").manual_seed(21)
        return [(torch.randn(16, 256, device="cuda", generator=gen), torch.randint(0, 10, (16,), device="cuda",
                                                                                  generator=gen)) for _ in range(7)]

    data = batches()

    def run(model, opt, rng):
        for x, y in (data[i] for i in rng):
            torch.nn.functional.cross_entropy(model(x), y).backward()
            opt.step()

    torch.manual_seed(4)
    m1 = MLP().cuda()
    o1 = LagsSGD(m1.parameters(), lr=0.05, rho=0.01, momentum=0.9, bucket_cap_bytes=4096)
    run(m1, o1, range(3))
    sd_model = {k: t.clone() for k, t in m1.state_dict().items()}
    sd_opt = o1.state_dict()
    run(m1, o1, range(3, 7))
    torch.manual_seed(99)  # different init: everything must come from the checkpoint
    m2 = MLP().cuda()
    o2 = LagsSGD(m2.parameters(), lr=0.05, rho=0.01, momentum=0.9, bucket_cap_bytes=4096)
    m2.load_state_dict(sd_model)
    o2.load_state_dict(sd_opt)
    run(m2, o2, range(3, 7))
    torch.cuda.synchronize()
    assert o1.params_vector().cpu().numpy().tobytes() == o2.params_vector().cpu().numpy().tobytes()
    assert o1.residual_vector().cpu().numpy().tobytes() == o2.residual_vector().cpu().numpy().tobytes()
