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
    v = opt.flat_param.cpu().numpy().copy()
    res = [np.zeros_like(v)]
    for t in range(8):
        x = torch.randn(32, 256, device="cuda")
        y = torch.randint(0, 10, (32,), device="cuda")
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        g = torch.cat([captured[id(p)].reshape(-1) for p in opt.params]).cpu().numpy()
        v = orc.lags_step(v, [g], 0.05, opt.dims, opt.ks, res)
        assert opt.flat_param.cpu().numpy().tobytes() == v.tobytes(), t
        assert opt.residual.cpu().numpy().tobytes() == res[0].tobytes(), t
        assert not torch.any(opt.flat_grad), "compress clears the gradients"
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
