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
