"""Generate golden fixtures for the hot path by running the REFERENCE package itself.

Run in the authoring container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``lagsgd`` from /root/reference/pkg/src (read-only, never copied)
and writes small ``.npz`` / ``.json`` fixtures next to this file.  The GPU box
has no /root/reference, so tests there read only these fixtures.

Fixtures:
  topk_cases.npz         top_k(x, k) -> (indices, values)          R: sparsify.py:71-90
  lags_step_cases.npz    lags_step(v, grads, alpha, counts, res)   R: training.py:227-255
  config1_trajectory.npz train() config 1 with lags_step recorded  R: training.py:261-384
  slgs_cases.npz         slgs_step(v, grads, alpha, global_k, res) R: training.py:203-224
  perf_cases.json        select_ratios / comm_time / schedules     R: perf.py:59-260
  wire_cases.json        encode_chunk / fusion_flush               R: sparsify.py:209-310
  delta_cases.npz        topk_aggregation_ratio (delta^(l))        R: analysis.py:24-56
  nonfinite_cases.npz    top_k / lags_step with NaN and +-inf      R: sparsify.py:84-90, training.py:250-254
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import lagsgd  # noqa: E402
from lagsgd import training as ref_training  # noqa: E402
from lagsgd.layered import LayeredVector, LayerShape, concat  # noqa: E402
from lagsgd.models import DatasetSpec, MlpModel, SyntheticDataset  # noqa: E402
from lagsgd.perf import NetworkModel, PipelineScenario, comm_time, schedule, select_ratios  # noqa: E402
from lagsgd.sparsify import (  # noqa: E402
    CompressionPolicy,
    SparseChunk,
    encode_chunk,
    encode_message,
    fusion_flush,
    top_k,
)


def _dist(rng, kind, d, dtype):
    if kind == "normal":
        x = rng.standard_normal(d)
    elif kind == "heavy":
        x = rng.standard_normal(d) * np.exp(2.0 * rng.standard_normal(d))
    elif kind == "ties":
        x = rng.integers(-3, 4, size=d).astype(np.float64)
    elif kind == "zeros50":
        x = rng.standard_normal(d) * (rng.random(d) < 0.5)
    elif kind == "allequal":
        x = np.full(d, -1.25)
    elif kind == "denormal":
        tiny = np.finfo(dtype).smallest_subnormal
        x = rng.integers(-40, 41, size=d) * float(tiny)
    elif kind == "signedzero":
        x = np.where(rng.random(d) < 0.5, -0.0, 0.0)
        hit = rng.random(d) < 0.1
        x[hit] = rng.standard_normal(int(hit.sum()))
    elif kind == "scales":
        x = rng.standard_normal(d) * 10.0 ** rng.integers(-30, 30, size=d)
    else:
        raise ValueError(kind)
    return x.astype(dtype)


KINDS = ("normal", "heavy", "ties", "zeros50", "allequal", "denormal", "signedzero", "scales")


def make_topk():
    rng = np.random.default_rng(20261018)
    cases = []
    # known-answer vectors of the reference's own tests (R: tests/test_sparsify.py:36-64)
    cases.append((np.array([3.0, -5.0, 1.0, 0.5]), 2))
    cases.append((np.array([2.0, -2.0, 1.0]), 1))
    cases.append((np.zeros(3), 2))
    cases.append((np.random.default_rng(4).standard_normal(17), 17))
    cases.append((np.array([0.0, -0.0, 0.0]), 3))
    cases.append((np.array([7.0]), 1))
    for dtype in (np.float64, np.float32):
        for kind in KINDS:
            for _ in range(6):
                d = int(rng.integers(1, 5000))
                k = int(rng.integers(1, d + 1)) if rng.random() < 0.5 else max(1, d // 100)
                cases.append((_dist(rng, kind, d, dtype), k))
        for d, k in ((40_000, 40), (65_536, 65), (9_000, 9_000), (32_768, 1)):
            cases.append((_dist(rng, "normal", d, dtype), k))
        cases.append((_dist(rng, "ties", 50_000, dtype), 1000))
    out = {"n": np.array(len(cases))}
    for i, (x, k) in enumerate(cases):
        ch = top_k(x, k)
        out[f"x{i}"] = x
        out[f"k{i}"] = np.array(k)
        out[f"idx{i}"] = ch.indices
        out[f"val{i}"] = ch.values
    np.savez_compressed(os.path.join(HERE, "topk_cases.npz"), **out)
    return len(cases)


def make_lags_step():
    rng = np.random.default_rng(7)
    cases = []
    # the reference's hand trace (R: tests/test_training.py:161-172)
    cases.append(dict(dims=[2, 2], P=2, dtype=np.float64, alpha=1.0, counts=[1, 1],
                      v=np.zeros(4), g=[np.array([1.0, 2.0, 3.0, 1.0]), np.array([2.0, -1.0, 0.0, 1.0])],
                      r=[np.zeros(4), np.zeros(4)]))
    specs = [
        ([5000, 37, 1, 2048], 3, np.float32, 0.1, "py"),
        ([5000, 37, 1, 2048], 3, np.float32, 0.1, "np64"),   # NEP 50: fp64 acc, fp32 store
        ([1040, 68], 2, np.float64, 1.0 / np.sqrt(500), "np64"),
        ([9408, 64, 64, 6912, 256, 1000], 3, np.float64, 0.05, "py"),
        ([2304, 64, 64, 4608, 256, 1000], 8, np.float32, 0.05, "py"),
        ([20_000, 3, 6_553], 2, np.float32, 0.3, "py"),
        ([4, 6], 2, np.float64, 0.15, "py"),
    ]
    for dims, P, dtype, alpha, atype in specs:
        n = sum(dims)
        ratio = float(rng.choice([1.0, 10.0, 100.0, 1000.0]))
        counts = [min(d, max(1, int(d // ratio))) for d in dims]
        g = [_dist(rng, "heavy", n, dtype) for _ in range(P)]
        for gg in g:  # inject ties and zeros
            gg[rng.integers(0, n, size=max(1, n // 50))] = 0
            gg[rng.integers(0, n, size=max(1, n // 50))] = dtype(0.5)
        r = [(0.01 * _dist(rng, "normal", n, dtype)).astype(dtype) for _ in range(P)]
        a = np.float64(alpha) if atype == "np64" else float(alpha)
        cases.append(dict(dims=dims, P=P, dtype=dtype, alpha=a, counts=counts,
                          v=_dist(rng, "normal", n, dtype), g=g, r=r))
    out = {"n": np.array(len(cases))}
    for i, c in enumerate(cases):
        shape = [LayerShape(j + 1, d) for j, d in enumerate(c["dims"])]
        v = LayeredVector(shape, np.array(c["v"], dtype=c["dtype"]))
        grads = [LayeredVector(shape, np.array(x, dtype=c["dtype"])) for x in c["g"]]
        res = [LayeredVector(shape, np.array(x, dtype=c["dtype"]).copy()) for x in c["r"]]
        counts = {j + 1: k for j, k in enumerate(c["counts"])}
        new_v = ref_training.lags_step(v, grads, c["alpha"], counts, res)
        out[f"dims{i}"] = np.array(c["dims"], dtype=np.int64)
        out[f"counts{i}"] = np.array(c["counts"], dtype=np.int64)
        out[f"alpha{i}"] = np.array(float(c["alpha"]))
        out[f"alpha_np64_{i}"] = np.array(isinstance(c["alpha"], np.float64))
        out[f"v{i}"] = v.data
        out[f"g{i}"] = np.stack([x.data for x in grads])
        out[f"r_in{i}"] = np.stack([np.array(x, dtype=c["dtype"]) for x in c["r"]])
        out[f"r_out{i}"] = np.stack([x.data for x in res])
        out[f"v_out{i}"] = new_v.data
    np.savez_compressed(os.path.join(HERE, "lags_step_cases.npz"), **out)
    return len(cases)


def make_slgs():
    """slgs_step(v, grads, alpha, global_k, residuals) cases -- R: training.py:203-224."""
    rng = np.random.default_rng(9)
    out = {}
    specs = [([300, 17, 2048], 2, np.float64, 0.2, 40), ([5000, 3], 3, np.float32, 0.05, 50),
             ([64, 64], 1, np.float64, 1.0, 128)]
    for i, (dims, P, dtype, alpha, gk) in enumerate(specs):
        shape = [LayerShape(j + 1, d) for j, d in enumerate(dims)]
        n = sum(dims)
        v = LayeredVector(shape, _dist(rng, "normal", n, dtype))
        grads = [LayeredVector(shape, _dist(rng, "heavy", n, dtype)) for _ in range(P)]
        r_in = [(0.01 * _dist(rng, "normal", n, dtype)).astype(dtype) for _ in range(P)]
        res = [LayeredVector(shape, r.copy()) for r in r_in]
        new_v = ref_training.slgs_step(v, grads, alpha, gk, res)
        out.update({f"dims{i}": np.array(dims), f"k{i}": np.array(gk), f"alpha{i}": np.array(alpha),
                    f"v{i}": v.data, f"g{i}": np.stack([g.data for g in grads]), f"r_in{i}": np.stack(r_in),
                    f"r_out{i}": np.stack([r.data for r in res]), f"v_out{i}": new_v.data})
    out["n"] = np.array(len(specs))
    np.savez_compressed(os.path.join(HERE, "slgs_cases.npz"), **out)
    return len(specs)


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def make_config1(iterations=100):
    """Config 1 (BASELINE.json configs[0]): MLP 64-16-4, P = 2, rho = 0.01 -> c = 100.

    Dataset/seed follow R: tests/test_acceptance.py:38-51 and pkg/README.md:57-71.
    Every lags_step call is recorded (inputs: alpha, gradients; outputs: digests).
    """
    dataset = SyntheticDataset(DatasetSpec("synthetic-gaussian-classification", 4096, 64, 4, seed=123))
    model = MlpModel((64, 16, 4))
    cfg = lagsgd.TrainerConfig("lags", 2, CompressionPolicy.uniform(100.0, model.shape),
                               lagsgd.StepSizeSchedule("inv-sqrt-T", 1.0), iterations, seed=42,
                               batch_size=32, loss_log_every=1)
    rec = {"alpha": [], "grads": [], "digest": []}
    real = ref_training.lags_step

    def recording(v, grads, alpha, counts, residuals, t=None):
        if not rec["alpha"]:
            rec["v0"] = v.data.copy()
        rec["alpha"].append(float(alpha))
        rec["grads"].append(np.stack([g.data.copy() for g in grads]))
        out = real(v, grads, alpha, counts, residuals, t)
        rec["digest"].append(_digest(out.data, *[r.data for r in residuals]))
        return out

    ref_training.lags_step = recording
    try:
        run = lagsgd.train(cfg, model, dataset)
    finally:
        ref_training.lags_step = real
    counts = cfg.policy.selection_counts(model.shape)
    np.savez_compressed(
        os.path.join(HERE, "config1_trajectory.npz"),
        dims=np.array([ls.dim for ls in model.shape], dtype=np.int64),
        counts=np.array([counts[ls.layer_id] for ls in model.shape], dtype=np.int64),
        v0=rec["v0"], alpha=np.array(rec["alpha"]), grads=np.stack(rec["grads"]),
        digest=np.array(rec["digest"]), final_v=run.final_params.data,
        final_r=np.stack([r.data for r in run.final_residuals]),
        losses=run.losses(), alpha_is_np64=np.array(True),
    )
    return iterations


def make_perf():
    out = {"select": [], "comm": [], "pipelined": []}
    rng = np.random.default_rng(11)
    ring = None
    for _ in range(60):
        L = int(rng.integers(1, 12))
        dims = [int(x) for x in rng.integers(1, 3_000_000, size=L)]
        bwd = [float(x) for x in rng.uniform(1e-5, 5e-3, size=L)]
        spar = [float(x) for x in rng.uniform(0, 5e-4, size=L)]
        lat = float(rng.uniform(0, 5e-5))
        inv_bw = float(10.0 ** rng.uniform(-11, -8))
        P = int(rng.integers(2, 9))
        cap = float(rng.choice([100, 500, 1000]))
        net = NetworkModel(lat, inv_bw, ring)
        sc = PipelineScenario(tuple(dims), tuple(bwd), 1e-3, tuple(spar), net,
                              CompressionPolicy({i + 1: 1.0 for i in range(L)}, cap), P)
        pol = select_ratios(sc, ratio_cap=cap)
        out["select"].append(dict(dims=dims, bwd=bwd, spar=spar, lat=lat, inv_bw=inv_bw, P=P, cap=cap,
                                  ratios=[pol.ratio_for(i + 1) for i in range(L)]))
        sc2 = PipelineScenario(tuple(dims), tuple(bwd), 1e-3, tuple(spar), net, pol, P)
        out["pipelined"].append(dict(dims=dims, bwd=bwd, spar=spar, lat=lat, inv_bw=inv_bw, P=P,
                                     ratios=[pol.ratio_for(i + 1) for i in range(L)],
                                     comm=list(sc2.comm_times()),
                                     makespan=schedule(sc2, "pipelined").makespan))
    for dim, ratio, P in ((12000, 1, 2), (12000, 1000, 2), (1, 1000, 8), (2359296, 1000, 8)):
        net = NetworkModel(1e-5, 1e-9)
        out["comm"].append(dict(dim=dim, ratio=ratio, P=P, lat=1e-5, inv_bw=1e-9,
                                t=comm_time(dim, ratio, net, P)))
    with open(os.path.join(HERE, "perf_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0)


def make_wire():
    rng = np.random.default_rng(10)
    out = {"chunks": [], "flush": []}
    for _ in range(12):
        x = rng.standard_normal(50)
        ch = top_k(x, int(rng.integers(1, 20)), layer_id=int(rng.integers(0, 9)))
        out["chunks"].append(dict(layer_id=ch.layer_id, dim=ch.dim, idx=ch.indices.tolist(),
                                  vals=[float(v) for v in ch.values], hex=encode_chunk(ch).hex()))
    for _ in range(40):
        n = int(rng.integers(0, 5))
        counts = [int(c) for c in rng.integers(0, 20, size=n)]
        cap = int(rng.integers(50, 600))
        first = bool(rng.random() < 0.3)
        chunks = [SparseChunk(i + 1, 64, np.arange(c), np.arange(1.0, c + 1.0), k_target=max(c, 1))
                  for i, c in enumerate(counts)]
        try:
            msg = fusion_flush(chunks, cap, first)
            res = None if msg is None else [c.layer_id for c in msg.chunks]
            hexmsg = None if msg is None else encode_message(msg).hex()
            err = None
        except ValueError as exc:
            res, hexmsg, err = None, None, type(exc).__name__
        out["flush"].append(dict(counts=counts, cap=cap, first=first, result=res, hex=hexmsg, error=err))
    with open(os.path.join(HERE, "wire_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0)


def make_delta():
    from lagsgd.analysis import topk_aggregation_ratio

    rng = np.random.default_rng(24)
    out = {}
    n = 0
    specs = [(1, 50, 5, "normal"), (2, 50, 5, "normal"), (3, 200, 7, "heavy"), (4, 64, 64, "normal"),
             (2, 64, 3, "ties"), (3, 100, 10, "zeros50"), (2, 30, 4, "allequal"), (4, 1000, 1, "normal"),
             (2, 1, 1, "normal"), (5, 333, 20, "heavy"), (2, 40, 5, "zerosall")]
    for P, d, k, kind in specs:
        for dt in (np.float64, np.float32):
            if kind == "zerosall":
                xs = [np.zeros(d, dtype=dt) for _ in range(P)]
            else:
                xs = [_dist(rng, kind, d, dt).astype(dt) for _ in range(P)]
            got = topk_aggregation_ratio(xs, k)
            out[f"x{n}"] = np.stack(xs)
            out[f"meta{n}"] = np.array([P, d, k], dtype=np.int64)
            out[f"delta{n}"] = np.array(np.nan if got is None else got, dtype=np.float64)
            n += 1
    out["n"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "delta_cases.npz"), **out)
    return n


def make_nonfinite():
    """NaN / +-inf inside the accumulated vector (gradients stay finite, R: training.py:174).

    top_k ranks NaN after every number (stable argsort of -|x|) and then drops it with `mag > 0`;
    +-inf is the largest magnitude.  In lags_step a NaN reaches acc through the residual, and an
    overflowing r + alpha * g makes acc = +-inf, whose residual becomes inf - inf = NaN
    (R: sparsify.py:84-90, training.py:250-254)."""
    rng = np.random.default_rng(11)
    out = {}
    topk = [
        (np.array([np.nan, 1.0, 2.0, -3.0]), 2),
        (np.array([np.nan, np.nan, 1.0]), 3),
        (np.array([np.inf, -np.inf, 1.0, np.nan]), 2),
        (np.array([np.inf, -np.inf, 1.0, np.nan]), 4),
        (np.array([np.nan, 0.0, -0.0, np.nan]), 2),
        (np.array([np.nan, np.nan, np.nan]), 1),
    ]
    for dtype in (np.float64, np.float32):
        for d, k in ((3000, 30), (12_000, 120), (20_000, 20)):
            x = _dist(rng, "heavy", d, dtype)
            x[rng.integers(0, d, size=d // 100)] = np.nan
            x[rng.integers(0, d, size=3)] = np.inf
            x[rng.integers(0, d, size=3)] = -np.inf
            topk.append((x, k))
    out["n_topk"] = np.array(len(topk))
    for i, (x, k) in enumerate(topk):
        ch = top_k(x, k)
        out[f"tx{i}"] = x
        out[f"tk{i}"] = np.array(k)
        out[f"tidx{i}"] = ch.indices
        out[f"tval{i}"] = ch.values
    steps = []
    for dtype, big in ((np.float32, np.float32(3.0e38)), (np.float64, np.float64(1.5e308))):
        for P in (1, 3):
            dims = [3000, 40, 1500]
            n = sum(dims)
            counts = [30, 4, 150]
            g = [_dist(rng, "normal", n, dtype) for _ in range(P)]
            r = [(0.01 * _dist(rng, "normal", n, dtype)).astype(dtype) for _ in range(P)]
            for p in range(P):
                r[p][rng.integers(0, n, size=40)] = np.nan      # NaN residual entries
                hit = rng.integers(0, n, size=6)
                r[p][hit] = big                                   # r + alpha * g overflows to +inf
                g[p][hit] = np.abs(g[p][hit]) + dtype(1.0)
                neg = rng.integers(0, n, size=6)
                r[p][neg] = -big
                g[p][neg] = -(np.abs(g[p][neg]) + dtype(1.0))
            steps.append(dict(dims=dims, P=P, dtype=dtype, alpha=float(big) / 2 if dtype == np.float32 else 1e308,
                              counts=counts, v=_dist(rng, "normal", n, dtype), g=g, r=r))
    out["n_step"] = np.array(len(steps))
    with np.errstate(all="ignore"):
        for i, c in enumerate(steps):
            shape = [LayerShape(j + 1, d) for j, d in enumerate(c["dims"])]
            v = LayeredVector(shape, np.array(c["v"], dtype=c["dtype"]))
            grads = [LayeredVector(shape, np.array(x, dtype=c["dtype"])) for x in c["g"]]
            res = [LayeredVector(shape, np.array(x, dtype=c["dtype"]).copy()) for x in c["r"]]
            counts = {j + 1: k for j, k in enumerate(c["counts"])}
            new_v = ref_training.lags_step(v, grads, c["alpha"], counts, res)
            out[f"dims{i}"] = np.array(c["dims"], dtype=np.int64)
            out[f"counts{i}"] = np.array(c["counts"], dtype=np.int64)
            out[f"alpha{i}"] = np.array(float(c["alpha"]))
            out[f"v{i}"] = v.data
            out[f"g{i}"] = np.stack([x.data for x in grads])
            out[f"r_in{i}"] = np.stack([np.array(x, dtype=c["dtype"]) for x in c["r"]])
            out[f"r_out{i}"] = np.stack([x.data for x in res])
            out[f"v_out{i}"] = new_v.data
    np.savez_compressed(os.path.join(HERE, "nonfinite_cases.npz"), **out)
    return len(topk), len(steps)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named fixtures, e.g. `make_golden.py delta`
        for name in sys.argv[1:]:
            print(name, globals()["make_" + name]())
        sys.exit(0)
    print("topk cases", make_topk())
    print("lags_step cases", make_lags_step())
    print("config1 iterations", make_config1())
    print("slgs cases", make_slgs())
    make_perf()
    make_wire()
    print("reference version", lagsgd.__version__)
