"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  If the oracle disagrees with them anywhere it
is not trusted as the GPU parity checker.
"""

import hashlib
import itertools

import numpy as np
import pytest

from conftest import load_json, same_bits_nan
from oracle import lagsgd_oracle as orc


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("ranking", orc.RANKINGS)
def test_topk_golden(topk_cases, ranking):
    assert len(topk_cases) > 100
    for x, k, idx, val in topk_cases:
        got_i, got_v = orc.top_k(x, k, ranking)
        assert got_i.dtype == np.int64
        np.testing.assert_array_equal(got_i, idx)
        assert got_v.dtype == val.dtype
        assert _bits(got_v).tobytes() == _bits(val).tobytes()


def test_topk_known_answers():
    # R: tests/test_sparsify.py:36-72
    i, v = orc.top_k(np.array([3.0, -5.0, 1.0, 0.5]), 2)
    assert i.tolist() == [0, 1] and v.tolist() == [3.0, -5.0]
    i, v = orc.top_k(np.array([2.0, -2.0, 1.0]), 1)
    assert i.tolist() == [0]
    i, v = orc.top_k(np.zeros(3), 2)
    assert len(i) == 0
    with pytest.raises(ValueError):
        orc.top_k(np.array([1.0, 2.0]), 0)
    with pytest.raises(ValueError):
        orc.top_k(np.array([1.0, 2.0]), 3)
    with pytest.raises(ValueError):
        orc.top_k(np.zeros((2, 2)), 1)


def test_topk_brute_force():
    # R: tests/test_acceptance.py:75-97 (criterion 03), smaller sample
    rng = np.random.default_rng(46)
    for _ in range(200):
        d = int(rng.integers(2, 11))
        k = int(rng.integers(1, min(d, 5) + 1))
        x = rng.standard_normal(d)
        sq = x * x
        i, _ = orc.top_k(x, k)
        mask = np.ones(d, bool)
        mask[i] = False
        ours = float(np.sum(sq[mask]))
        best = min(float(np.sum(np.delete(sq, list(s)))) for s in itertools.combinations(range(d), k))
        assert ours == best


@pytest.mark.parametrize("ranking", orc.RANKINGS)
def test_lags_step_golden(step_cases, ranking):
    for c in step_cases:
        res = [r.copy() for r in c["r_in"]]
        out = orc.lags_step(c["v"], list(c["g"]), c["alpha"], c["dims"], c["counts"], res, ranking=ranking)
        assert out.dtype == c["v_out"].dtype
        assert _bits(out).tobytes() == _bits(c["v_out"]).tobytes()
        for a, b in zip(res, c["r_out"]):
            assert _bits(a).tobytes() == _bits(b).tobytes()


def test_lags_step_threads_identical(step_cases):
    c = step_cases[4]
    r1 = [r.copy() for r in c["r_in"]]
    r2 = [r.copy() for r in c["r_in"]]
    a = orc.lags_step(c["v"], list(c["g"]), c["alpha"], c["dims"], c["counts"], r1, threads=1)
    b = orc.lags_step(c["v"], list(c["g"]), c["alpha"], c["dims"], c["counts"], r2, threads=4)
    assert a.tobytes() == b.tobytes()
    assert all(x.tobytes() == y.tobytes() for x, y in zip(r1, r2))


def test_config1_trajectory(config1):
    dims = [int(d) for d in config1["dims"]]
    counts = [int(c) for c in config1["counts"]]
    v = config1["v0"].copy()
    res = [np.zeros_like(v) for _ in range(config1["grads"].shape[1])]
    for t in range(len(config1["alpha"])):
        alpha = np.float64(config1["alpha"][t])
        v = orc.lags_step(v, list(config1["grads"][t]), alpha, dims, counts, res, t=t + 1)
        h = hashlib.sha256()
        for a in (v, *res):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(config1["digest"][t]), f"diverged at step {t + 1}"
    assert v.tobytes() == config1["final_v"].tobytes()


def test_divergence_and_structure_errors():
    v = np.zeros(4)
    with pytest.raises(orc.DivergenceError) as ei:
        orc.lags_step(v, [np.array([0, np.nan, 0, 0.0])], 0.1, [4], [1], [np.zeros(4)], t=7)
    assert ei.value.iteration == 7
    with pytest.raises(orc.StructureError):
        orc.lags_step(v, [np.zeros(3)], 0.1, [4], [1], [np.zeros(4)])


def test_selection_counts():
    # R: tests/test_sparsify.py:218-225
    assert [orc.selection_count(d, 10.0) for d in (100, 15, 3)] == [10, 1, 1]
    assert orc.selection_count(68, 1 / 0.01) == 1
    assert orc.selection_count(2359296, 1 / 0.001) == 2359


def test_perf_golden():
    cases = load_json("perf_cases.json")
    for c in cases["select"]:
        got = orc.select_ratios(c["dims"], c["bwd"], c["spar"], c["lat"], c["inv_bw"], c["P"], c["cap"])
        assert [got[i + 1] for i in range(len(c["dims"]))] == c["ratios"]
    for c in cases["pipelined"]:
        comm = [orc.comm_time(d, r, c["lat"], c["inv_bw"], c["P"]) for d, r in zip(c["dims"], c["ratios"])]
        assert comm == c["comm"]
        assert orc.pipelined_makespan(1e-3, c["bwd"], c["spar"], comm) == c["makespan"]
    for c in cases["comm"]:
        assert orc.comm_time(c["dim"], c["ratio"], c["lat"], c["inv_bw"], c["P"]) == c["t"]


def test_wire_golden():
    cases = load_json("wire_cases.json")
    for c in cases["chunks"]:
        raw = orc.encode_chunk(c["layer_id"], c["dim"], c["idx"], c["vals"])
        assert raw.hex() == c["hex"]
        lid, dim, idx, vals, off = orc.decode_chunk(raw)
        assert (lid, dim, off) == (c["layer_id"], c["dim"], len(raw))
        assert idx.tolist() == c["idx"] and vals.tolist() == c["vals"]
    for c in cases["flush"]:
        try:
            got = orc.fusion_should_flush(c["counts"], c["cap"], c["first"])
        except ValueError as exc:
            assert c["error"] == type(exc).__name__
            continue
        assert c["error"] is None
        assert bool(got) == (c["result"] is not None)


def test_slgs_golden():
    from conftest import load_npz

    z = load_npz("slgs_cases.npz")
    for i in range(int(z["n"])):
        res = [r.copy() for r in z[f"r_in{i}"]]
        out = orc.slgs_step(z[f"v{i}"], list(z[f"g{i}"]), float(z[f"alpha{i}"]), int(z[f"k{i}"]), res)
        assert _bits(out).tobytes() == _bits(z[f"v_out{i}"]).tobytes()
        for a, b in zip(res, z[f"r_out{i}"]):
            assert _bits(a).tobytes() == _bits(b).tobytes()


def test_delta_golden():
    """Oracle delta^(l) against the reference's analysis.topk_aggregation_ratio outputs (numpy dot
    products on both sides: same BLAS, exact agreement expected up to summation order)."""
    from conftest import load_npz

    z = load_npz("delta_cases.npz")
    for i in range(int(z["n"])):
        P, d, k = (int(v) for v in z[f"meta{i}"])
        xs = list(z[f"x{i}"])
        want = float(z[f"delta{i}"])
        got = orc.topk_aggregation_ratio(xs, k)
        if np.isnan(want):
            assert got is None
        else:
            assert got is not None and abs(got - want) <= 1e-12 * max(1.0, abs(want)), (i, got, want)


def test_nonfinite_golden(nonfinite_cases):
    """NaN never selected (ranked after every number, then dropped by `mag > 0`), +-inf first; an
    overflowed acc leaves inf - inf = NaN in the residual (R: sparsify.py:84-90, training.py:252)."""
    topk, steps = nonfinite_cases
    for x, k, idx, val in topk:
        got_i, got_v = orc.top_k(x, k)
        np.testing.assert_array_equal(got_i, idx)
        assert same_bits_nan(got_v, val)
    for c in steps:
        res = [r.copy() for r in c["r_in"]]
        with np.errstate(all="ignore"):
            v = orc.lags_step(c["v"], list(c["g"]), c["alpha"], c["dims"], c["counts"], res)
        assert same_bits_nan(v, c["v_out"])
        for a, b in zip(res, c["r_out"]):
            assert same_bits_nan(a, b)
