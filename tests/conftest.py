import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")
    config.addinivalue_line("markers", "gpu2: needs two B200s (gpurun --gpus 2; selected only by -m gpu2)")


def pytest_collection_modifyitems(config, items):
    """Two-GPU tests run only when asked for (-m gpu2): on one GPU they could only skip."""
    if "gpu2" in (config.getoption("markexpr") or ""):
        return
    keep = [it for it in items if it.get_closest_marker("gpu2") is None]
    dropped = [it for it in items if it.get_closest_marker("gpu2") is not None]
    if dropped:
        config.hook.pytest_deselected(items=dropped)
        items[:] = keep


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def topk_cases():
    z = load_npz("topk_cases.npz")
    return [(z[f"x{i}"], int(z[f"k{i}"]), z[f"idx{i}"], z[f"val{i}"]) for i in range(int(z["n"]))]


@pytest.fixture(scope="session")
def step_cases():
    z = load_npz("lags_step_cases.npz")
    out = []
    for i in range(int(z["n"])):
        alpha = float(z[f"alpha{i}"])
        if bool(z[f"alpha_np64_{i}"]):
            alpha = np.float64(alpha)
        out.append(dict(dims=[int(d) for d in z[f"dims{i}"]], counts=[int(c) for c in z[f"counts{i}"]],
                        alpha=alpha, v=z[f"v{i}"], g=z[f"g{i}"], r_in=z[f"r_in{i}"],
                        r_out=z[f"r_out{i}"], v_out=z[f"v_out{i}"]))
    return out


@pytest.fixture(scope="session")
def config1():
    return load_npz("config1_trajectory.npz")


def same_bits_nan(a, b) -> bool:
    """Bit equality except that any NaN matches any NaN at the same position (the NaN payload of
    inf - inf is platform-defined: x86 numpy yields 0xffc00000, the GPU 0x7fffffff)."""
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    if a.dtype != b.dtype or a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb)) and a[~na].tobytes() == b[~nb].tobytes()


@pytest.fixture(scope="session")
def nonfinite_cases():
    """top_k and lags_step with NaN / +-inf inside the accumulated vector, made by the reference."""
    z = load_npz("nonfinite_cases.npz")
    topk = [(z[f"tx{i}"], int(z[f"tk{i}"]), z[f"tidx{i}"], z[f"tval{i}"]) for i in range(int(z["n_topk"]))]
    steps = [dict(dims=[int(d) for d in z[f"dims{i}"]], counts=[int(c) for c in z[f"counts{i}"]],
                  alpha=float(z[f"alpha{i}"]), v=z[f"v{i}"], g=z[f"g{i}"], r_in=z[f"r_in{i}"],
                  r_out=z[f"r_out{i}"], v_out=z[f"v_out{i}"]) for i in range(int(z["n_step"]))]
    return topk, steps
