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
