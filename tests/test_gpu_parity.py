"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and the
pinned CPU oracle.  Integer/index results and all values must be bit-exact."""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import same_bits_nan  # noqa: E402
from oracle import lagsgd_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1911_08727_b200 as lib

    return lib


def _same_bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def test_topk_golden(L, topk_cases):
    for x, k, idx, val in topk_cases:
        ch = L.top_k(x, k)
        np.testing.assert_array_equal(ch.indices, idx)
        assert _same_bits(ch.values, val), (x.dtype, x.size, k)
        assert ch.k_target == k and ch.dim == x.size


def test_topk_errors(L):
    with pytest.raises(ValueError):
        L.top_k(np.array([1.0, 2.0]), 0)
    with pytest.raises(ValueError):
        L.top_k(np.array([1.0, 2.0]), 3)
    with pytest.raises(ValueError):
        L.top_k(np.zeros(0), 1)


def test_topk_adversarial_fuzz(L):
    rng = np.random.default_rng(123)
    kinds = ["normal", "ties", "zeros", "denormal", "signedzero", "huge", "const"]
    for it in range(120):
        kind = kinds[it % len(kinds)]
        dtype = np.float32 if it % 2 else np.float64
        d = int(rng.integers(1, 300_000)) if it % 10 == 0 else int(rng.integers(1, 20_000))
        if kind == "normal":
            x = rng.standard_normal(d)
        elif kind == "ties":
            x = rng.integers(-2, 3, size=d).astype(np.float64)
        elif kind == "zeros":
            x = rng.standard_normal(d) * (rng.random(d) < 0.02)
        elif kind == "denormal":
            x = rng.integers(-5, 6, size=d) * float(np.finfo(dtype).smallest_subnormal)
        elif kind == "signedzero":
            x = np.where(rng.random(d) < 0.5, -0.0, 0.0)
        elif kind == "huge":
            x = rng.standard_normal(d) * 10.0 ** rng.integers(-35, 35, size=d)
        else:
            x = np.full(d, 3.0)
        x = x.astype(dtype)
        k = int(rng.integers(1, d + 1)) if rng.random() < 0.3 else max(1, d // 1000)
        ch = L.top_k(x, k)
        wi, wv = orc.top_k(x, k)
        np.testing.assert_array_equal(ch.indices, wi, err_msg=f"{kind} d={d} k={k}")
        assert _same_bits(ch.values, wv)


def test_decompress_matches(L):
    rng = np.random.default_rng(9)
    x = rng.standard_normal(25)
    ch = L.top_k(x, 6)
    dense = L.decompress(ch)
    np.testing.assert_array_equal(dense[ch.indices], ch.values)
    assert _same_bits(dense, orc.decompress(ch.indices, ch.values, 25))
    empty = L.SparseChunk(0, 3, np.array([], dtype=np.int64), np.array([]), k_target=2)
    assert _same_bits(L.decompress(empty), np.zeros(3))


def _lv(L, dims, data):
    return L.LayeredVector([L.LayerShape(i + 1, d) for i, d in enumerate(dims)], data)


def test_lags_step_golden(L, step_cases):
    for c in step_cases:
        dims = c["dims"]
        res = [_lv(L, dims, r.copy()) for r in c["r_in"]]
        out = L.lags_step(_lv(L, dims, c["v"]), [_lv(L, dims, g) for g in c["g"]], c["alpha"],
                          {i + 1: k for i, k in enumerate(c["counts"])}, res)
        assert _same_bits(out.data, c["v_out"]), dims
        for a, b in zip(res, c["r_out"]):
            assert _same_bits(a.data, b)


def test_nonfinite_golden(L, nonfinite_cases):
    """NaN / +-inf in the accumulated vector, against the reference's own outputs: NaN is never
    selected, +-inf is the largest magnitude, and a selected +-inf leaves inf - inf = NaN in the
    residual (R: sparsify.py:84-90, training.py:252).  Every call runs twice so the second takes
    the predicted-threshold candidate path."""
    topk, steps = nonfinite_cases
    for x, k, idx, val in topk:
        ch = L.top_k(x, k)
        np.testing.assert_array_equal(ch.indices, idx)
        assert same_bits_nan(ch.values, val)
    for c in steps:
        dims = c["dims"]
        counts = {i + 1: k for i, k in enumerate(c["counts"])}
        for _ in range(2):
            res = [_lv(L, dims, r.copy()) for r in c["r_in"]]
            out = L.lags_step(_lv(L, dims, c["v"]), [_lv(L, dims, g) for g in c["g"]], c["alpha"], counts, res)
            assert same_bits_nan(out.data, c["v_out"]), dims
            for a, b in zip(res, c["r_out"]):
                assert same_bits_nan(a.data, b)


def test_config1_trajectory_bitexact(L, config1):
    """Config 1 (MLP 64-16-4, P=2, rho=0.01): replay the reference train()'s recorded gradients;
    params and residuals must match the reference's digest at every one of 100 steps."""
    dims = [int(d) for d in config1["dims"]]
    counts = {i + 1: int(c) for i, c in enumerate(config1["counts"])}
    v = _lv(L, dims, config1["v0"].copy())
    P = config1["grads"].shape[1]
    res = [_lv(L, dims, np.zeros_like(config1["v0"])) for _ in range(P)]
    for t in range(len(config1["alpha"])):
        grads = [_lv(L, dims, g) for g in config1["grads"][t]]
        v = L.lags_step(v, grads, np.float64(config1["alpha"][t]), counts, res, t=t + 1)
        h = hashlib.sha256()
        for a in (v.data, *[r.data for r in res]):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(config1["digest"][t]), f"step {t + 1}"
    assert _same_bits(v.data, config1["final_v"])


def test_lags_step_fuzz_vs_oracle(L):
    rng = np.random.default_rng(77)
    for it in range(12):
        dtype = [np.float32, np.float64][it % 2]
        P = int(rng.integers(1, 6))
        dims = [int(x) for x in rng.integers(1, 50_000, size=int(rng.integers(1, 7)))]
        n = sum(dims)
        counts = [max(1, d // int(rng.choice([1, 10, 100, 1000]))) for d in dims]
        v = rng.standard_normal(n).astype(dtype)
        grads = [(rng.standard_normal(n) * np.exp(rng.standard_normal(n))).astype(dtype) for _ in range(P)]
        for g in grads:
            g[rng.integers(0, n, size=n // 20 + 1)] = 0.0
        res0 = [(0.01 * rng.standard_normal(n)).astype(dtype) for _ in range(P)]
        alpha = float(rng.uniform(0.01, 1.0))
        if it % 4 == 3:
            alpha = np.float64(alpha)
        rr = [r.copy() for r in res0]
        want = orc.lags_step(v, grads, alpha, dims, counts, rr)
        rg = [_lv(L, dims, r.copy()) for r in res0]
        got = L.lags_step(_lv(L, dims, v), [_lv(L, dims, g) for g in grads], alpha,
                          {i + 1: k for i, k in enumerate(counts)}, rg)
        assert _same_bits(got.data, want), (it, dtype, dims)
        for a, b in zip(rg, rr):
            assert _same_bits(a.data, b)


def test_lags_step_errors(L):
    dims = [4]
    v = _lv(L, dims, np.zeros(4))
    bad = _lv(L, dims, np.array([0.0, np.inf, 0.0, 0.0]))
    ok = _lv(L, dims, np.ones(4))
    res = [_lv(L, dims, np.full(4, 0.5)), _lv(L, dims, np.full(4, 0.5))]
    with pytest.raises(L.DivergenceError) as ei:
        L.lags_step(v, [ok, bad], 0.1, {1: 1}, res, t=5)
    assert ei.value.iteration == 5
    assert all(np.all(r.data == 0.5) for r in res), "residuals must be untouched on divergence"
    other = _lv(L, [2, 2], np.zeros(4))
    with pytest.raises(L.StructureError):
        L.lags_step(v, [ok, other], 0.1, {1: 1}, res)
    # reference order: worker 1 non-finite is reported before worker 2's layout error
    with pytest.raises(L.DivergenceError):
        L.lags_step(v, [bad, other], 0.1, {1: 1}, res)
    with pytest.raises(ValueError):
        L.lags_step(v, [ok], 0.1, {1: 5}, res[:1])


def test_bucket_device_api_and_momentum(L):
    from paper_1911_08727_b200 import _native as N

    dims, ks = [5000, 1, 123457, 64], [5, 1, 123, 64]
    b = L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(5)
    g = torch.randn(n, device="cuda", generator=gen)
    r = torch.randn(n, device="cuda", generator=gen) * 0.01
    r0 = r.clone()
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    b.compress(g, r, 0.1, msg, st)
    got = b.unpack(msg)
    acc = (r0.cpu().numpy() + np.float32(0.1) * g.cpu().numpy()).astype(np.float32)
    off = 0
    for j, (d, k) in enumerate(zip(dims, ks)):
        wi, wv = orc.top_k(acc[off:off + d], k)
        np.testing.assert_array_equal(got[j][0], wi)
        assert _same_bits(got[j][1], wv)
        off += d
    # momentum (parity unpinned): m = mu*m + total/P ; v -= m, checked against float64 math
    v = torch.zeros(n, device="cuda")
    m = torch.ones(n, device="cuda")
    b.decode(msg, 1, v, momentum=m, mu=0.9)
    dense = np.zeros(n)
    off = 0
    for j, d in enumerate(dims):
        dense[off + got[j][0]] = got[j][1]
        off += d
    want_m = (0.9 * np.ones(n) + dense).astype(np.float32)
    np.testing.assert_allclose(m.cpu().numpy(), want_m, rtol=1e-6)
    np.testing.assert_allclose(v.cpu().numpy(), -want_m, rtol=1e-6)
    assert int(st.item()) == 0


def test_fast_path_equals_exact_path(L):
    """The predicted-threshold fast path (K1 candidate emission + K2 candidate select) must be
    bit-identical to the dense exact path on every call: steady state, mispredictions (scale
    drops), task-list overflow (concentrated gradients) and all-zero layers."""
    from paper_1911_08727_b200 import _native as N

    dims = [20000, 64, 300000, 5000, 2359296 // 4, 70001, 1000]
    ks = [max(1, d // 1000) for d in dims]
    ks[1] = 64
    fast = L.Bucket(dims, ks, N.F32)
    exact = L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(3)
    r_f = torch.zeros(n, device="cuda")
    r_e = torch.zeros(n, device="cuda")
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    off = np.concatenate([[0], np.cumsum(dims)])
    for it in range(24):
        g = torch.randn(n, device="cuda", generator=gen)
        if it in (9, 10):
            g *= 1e-3  # threshold collapses -> too few candidates -> dense fallback
        if it == 14:  # one layer's mass concentrated in one task -> candidate list overflow
            g[off[2]:off[2] + 8192] *= 1e4
        if it == 17:
            g[off[4]:off[5]] = 0.0
            r_f[off[4]:off[5]] = 0.0
            r_e[off[4]:off[5]] = 0.0
        fast.compress(g, r_f, 0.05, m_f, st)
        exact.compress(g, r_e, 0.05, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"messages differ at iteration {it}"
        assert torch.equal(r_f.view(torch.int32), r_e.view(torch.int32)), f"residuals differ at {it}"
    s = fast.stats()
    big = [j for j, d in enumerate(dims) if d > 16384]
    assert all(s[j, 3] == 24 for j in range(len(dims)))  # calls
    on_candidates = sum(1 for j in big if s[j, 2] > 0)
    assert on_candidates >= len(big) - 2, s  # candidate path active on (almost) all big layers
    assert int(s[big, 1].sum()) < 8 * len(big), s  # dense fallbacks are the exception
    assert int(st.item()) == 0


def test_fast_path_ties_equal_exact_path(L):
    """Tie-heavy data through the fast paths (cluster layers, candidate layers, small fallbacks):
    integer gradients with alpha = 1 keep every accumulated value an integer, so the threshold's
    radix bin (and the bin-list finish) holds many equal keys, and zeros are frequent.  The
    selection must still take the lower indices first among equal keys, exactly as the dense path."""
    from paper_1911_08727_b200 import _native as N

    dims = [600_000, 300_000, 9_000, 2_100_000, 40_000, 1_000]
    ks = [max(1, d // 1000) for d in dims]
    fast = L.Bucket(dims, ks, N.F32)
    exact = L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(11)
    r_f = torch.zeros(n, device="cuda")
    r_e = torch.zeros(n, device="cuda")
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for it in range(20):
        g = torch.randint(-6, 7, (n,), device="cuda", generator=gen).float()
        if it % 5 == 4:
            g[::3] = 0.0
        fast.compress(g, r_f, 1.0, m_f, st)
        exact.compress(g, r_e, 1.0, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"messages differ at iteration {it}"
        assert torch.equal(r_f.view(torch.int32), r_e.view(torch.int32)), f"residuals differ at {it}"
    s = fast.stats()
    assert int(((s[:, 5] == 3) | (s[:, 5] == 4)).sum()) >= 1, s  # a cluster layer took the cluster path
    assert int(st.item()) == 0


def test_fast_path_decode_multi_rank_equals_oracle(L):
    """P simulated ranks through one bucket: fast compress per rank, rank-ordered decode."""
    from paper_1911_08727_b200 import _native as N

    dims = [40000, 17, 123457]
    ks = [40, 1, 123]
    P = 5
    b = L.Bucket(dims, ks, N.F32, max_world=P)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(8)
    rs = [torch.zeros(n, device="cuda") for _ in range(P)]
    v = torch.randn(n, device="cuda", generator=gen)
    msgs = b.new_messages(P)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    v_h = v.cpu().numpy().copy()
    r_h = [np.zeros(n, np.float32) for _ in range(P)]
    for it in range(6):
        gs = [torch.randn(n, device="cuda", generator=gen) for _ in range(P)]
        for p in range(P):
            b.compress(gs[p], rs[p], 0.1, msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes], st)
        b.decode(msgs, P, v)
        v_h = orc.lags_step(v_h, [g.cpu().numpy() for g in gs], 0.1, dims, ks, r_h)
        assert _same_bits(v.cpu().numpy(), v_h), it
        for p in range(P):
            assert _same_bits(rs[p].cpu().numpy(), r_h[p])


@pytest.mark.parametrize("dims,ks", [
    ([300000, 64, 1000003, 16000, 70001, 9], [300, 64, 1000, 16, 70, 1]),  # fused update; 1000003 -> cluster
    ([2000000, 300000, 5000], [40000, 12000, 50]),  # > 49152 selected: step_local runs the separate decode
])
def test_step_local_equals_compress_plus_decode(L, dims, ks):
    """P = 1 step (lags_bucket_step_local) == compress + decode, over the dense first call, the
    candidate path and a forced misprediction."""
    from paper_1911_08727_b200 import _native as N

    a, b = L.Bucket(dims, ks, N.F32), L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(21)
    ra, rb = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    va = torch.randn(n, device="cuda", generator=gen)
    vb = va.clone()
    ma, mb = a.new_messages(1), b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for it in range(8):
        g = torch.randn(n, device="cuda", generator=gen) * (1e-3 if it == 5 else 1.0)
        a.step_local(g, ra, 0.1, va, ma, st)
        b.compress(g, rb, 0.1, mb, st)
        b.decode(mb, 1, vb)
        assert torch.equal(ma, mb), it
        assert torch.equal(ra.view(torch.int32), rb.view(torch.int32)), it
        assert torch.equal(va.view(torch.int32), vb.view(torch.int32)), it


def test_large_layer_properties(L):
    """Full-size layer (LSTM embedding, 15M) through the bucket API: size-independent checks
    (count == k, ascending, residual + sent == acc bitwise, selected keys dominate)."""
    from paper_1911_08727_b200 import _native as N

    d, k = 15_000_000, 15_000
    b = L.Bucket([d], [k], N.F32)
    gen = torch.Generator(device="cuda").manual_seed(11)
    g = torch.randn(d, device="cuda", generator=gen)
    r = torch.randn(d, device="cuda", generator=gen) * 0.05
    acc = r + torch.tensor(0.1, dtype=torch.float32, device="cuda") * g  # two roundings in fp32
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    b.compress(g, r, 0.1, msg, st)
    idx, val = b.unpack(msg)[0]
    assert idx.size == k
    assert np.all(np.diff(idx) > 0)
    acc_h = acc.cpu().numpy()
    assert _same_bits(val, acc_h[idx])
    r_h = r.cpu().numpy()
    assert np.all(r_h[idx] == 0) and not np.any(np.signbit(r_h[idx]))
    mask = np.ones(d, bool)
    mask[idx] = False
    assert _same_bits(r_h[mask], acc_h[mask])
    assert np.abs(val).min() >= np.abs(acc_h[mask]).max()


def test_slgs_step_golden(L):
    """SLGS arm (R: training.py:203-224): whole-vector selection with the same kernels."""
    from conftest import load_npz

    z = load_npz("slgs_cases.npz")
    for i in range(int(z["n"])):
        dims = [int(d) for d in z[f"dims{i}"]]
        res = [_lv(L, dims, r.copy()) for r in z[f"r_in{i}"]]
        out = L.slgs_step(_lv(L, dims, z[f"v{i}"]), [_lv(L, dims, g) for g in z[f"g{i}"]], float(z[f"alpha{i}"]),
                          int(z[f"k{i}"]), res)
        assert _same_bits(out.data, z[f"v_out{i}"])
        for a, b in zip(res, z[f"r_out{i}"]):
            assert _same_bits(a.data, b)


def test_tiny_layer_warp_path_vs_oracle(L):
    """Tiny layers (d <= 2048, k <= 8) take one warp each (register top-k), larger tiny ones a CTA
    (rounds of a block max for k <= 16, else radix) -- checked against the
    oracle's top_k on every call: odd sizes (unaligned layer offsets), k from 1 to 8, ties across
    lanes, all-equal layers, zeros, signed zeros, subnormals, a layer with fewer nonzeros than k."""
    from paper_1911_08727_b200 import _native as N

    rng = np.random.default_rng(17)
    # the last four: 2048 < d <= 4096 take a whole CTA (k <= 16: rounds of a block max, else radix)
    dims = [1, 3, 7, 64, 65, 127, 256, 511, 1000, 1023, 2048, 4095, 4096, 33, 97, 600, 3000, 2500, 4096, 3333]
    ks = [1, 1, 3, 8, 5, 2, 4, 8, 1, 7, 2, 8, 4, 8, 6, 3, 16, 12, 17, 1]
    b = L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    off = np.concatenate([[0], np.cumsum(dims)]).astype(np.int64)
    r = np.zeros(n, dtype=np.float32)
    r_d = torch.zeros(n, device="cuda")
    msg = b.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    alpha = 0.25
    for it in range(12):
        g = rng.standard_normal(n).astype(np.float32)
        if it % 4 == 1:  # heavy ties: few distinct magnitudes across lanes
            g = rng.integers(-3, 4, size=n).astype(np.float32)
        if it % 4 == 2:
            g[off[5]:off[6]] = -1.5  # all-equal layer (plus whatever residual it carries)
            g[off[7]:off[8]] = 0.0
            g[off[12]:off[13]] = np.where(rng.random(dims[12]) < 0.5, -0.0, 0.0)
            g[off[12] + 5] = 2.0  # fewer nonzeros than k there
            g[off[16]:off[17]] = 0.75  # all-equal again, k = 16 (one round takes every tie)
            g[off[17]:off[18]] = 0.0
            g[off[17] + 7] = np.nan if it == 2 else np.inf  # non-finite entries
        if it % 4 == 3:
            g[off[10]:off[11]] = (rng.integers(-40, 41, size=dims[10]) * np.finfo(np.float32).smallest_subnormal)
        acc = (r + np.float32(alpha) * g).astype(np.float32)
        b.compress(torch.from_numpy(g).cuda(), r_d, alpha, msg, st)
        got = b.unpack(msg)
        for j, (d, k) in enumerate(zip(dims, ks)):
            idx, val = orc.top_k(acc[off[j]:off[j + 1]], k)
            np.testing.assert_array_equal(got[j][0], idx, err_msg=f"iteration {it} layer {j}")
            assert _same_bits(got[j][1], val), (it, j)
        r = acc.copy()
        with np.errstate(invalid="ignore"):
            for j in range(len(dims)):
                sel = off[j] + got[j][0]
                r[sel] = acc[sel] - acc[sel]  # +0.0, NaN for a selected inf (R: training.py:252)
        assert same_bits_nan(r_d.cpu().numpy(), r), it  # NaN payloads are platform-defined
    s = b.stats()
    assert all(int(s[j, 5]) == 0 for j in range(len(dims)))  # every layer on the warp / dense-small path


def test_large_k_cluster_modes_equal_exact_path(L):
    """Large k (rho = 0.01 on multi-million-element layers): the cluster selection's candidate
    sets exceed one CTA's shared memory, so the CTAs keep their own keys and run the distributed
    radix select -- bit-identical to the dense exact path on every call, incl. mispredictions."""
    from paper_1911_08727_b200 import _native as N

    dims = [2359296, 1048576, 3000001, 70000]
    ks = [d // 100 for d in dims]
    fast = L.Bucket(dims, ks, N.F32)
    exact = L.Bucket(dims, ks, N.F32)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(21)
    r_f = torch.zeros(n, device="cuda")
    r_e = torch.zeros(n, device="cuda")
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for it in range(10):
        g = torch.randn(n, device="cuda", generator=gen)
        if it == 6:
            g *= 1e-3  # scale drop -> too few candidates -> dense fallback, then recovery
        fast.compress(g, r_f, 0.05, m_f, st)
        exact.compress(g, r_e, 0.05, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"messages differ at iteration {it}"
        assert torch.equal(r_f.view(torch.int32), r_e.view(torch.int32)), f"residuals differ at {it}"
    s = fast.stats()
    assert sum(1 for j in range(3) if s[j, 5] == 3) >= 2, s  # the big layers ran on clusters
    assert int(st.item()) == 0


@pytest.mark.parametrize("config", ["resnet20", "vgg16", "resnet50", "resnet50-rho0.01", "lstm"])
def test_survey_config_full_size_vs_oracle(L, config):
    """Every SURVEY config's full layer shapes (BASELINE.json configs 2-5) through the bench's
    path (fast candidate / cluster / warp selection): 10 chained compress calls bit-identical to
    the dense exact path, and calls 0 and 9 checked per layer against the oracle's top_k
    (R: sparsify.py:71-90) and residual rule (R: training.py:250-252) on the same fp32 inputs."""
    from paper_1911_08727_b200 import _native as N
    from paper_1911_08727_b200.workloads import LSTMPTB, resnet20, resnet50, vgg16_cifar

    make = {"resnet20": resnet20, "vgg16": vgg16_cifar, "resnet50": resnet50,
            "resnet50-rho0.01": resnet50, "lstm": LSTMPTB}[config]
    rho = 0.01 if config.endswith("0.01") else 0.001
    dims = [p.numel() for p in make().parameters()]
    ks = [orc.selection_count(d, 1.0 / rho) for d in dims]
    n = sum(dims)
    off = np.concatenate([[0], np.cumsum(dims)])
    fast = L.Bucket(dims, ks, N.F32)
    exact = L.Bucket(dims, ks, N.F32)
    gen = torch.Generator(device="cuda").manual_seed(17)
    # per-layer gradient scales spread over 4 decades, like a real backward pass
    scale = torch.repeat_interleave(
        torch.logspace(-2, 2, len(dims), device="cuda")[torch.randperm(len(dims), device="cuda", generator=gen)],
        torch.tensor(dims, device="cuda"))
    r_f = torch.zeros(n, device="cuda")
    r_e = torch.zeros(n, device="cuda")
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    alpha = 0.1
    for it in range(10):
        g = torch.randn(n, device="cuda", generator=gen) * scale
        check = it in (0, 9)
        if check:
            g_h, r_h = g.cpu().numpy(), r_f.cpu().numpy()
            acc = r_h + np.float32(alpha) * g_h  # two fp32 roundings, as the kernel (-fmad=false)
        fast.compress(g, r_f, alpha, m_f, st)
        exact.compress(g, r_e, alpha, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"{config}: messages differ at call {it}"
        assert torch.equal(r_f.view(torch.int32), r_e.view(torch.int32)), f"{config}: residuals differ at {it}"
        if check:
            got = fast.unpack(m_f)
            r_new = r_f.cpu().numpy()
            want_r = acc.copy()
            for j, (idx, val) in enumerate(got):
                a = acc[off[j]:off[j + 1]]
                w_idx, w_val = orc.top_k(a, ks[j])
                assert np.array_equal(idx, w_idx), (config, it, j)
                assert _same_bits(val, w_val), (config, it, j)
                want_r[off[j] + w_idx] = 0.0
            assert _same_bits(r_new, want_r), (config, it)
    assert int(st.item()) == 0


@pytest.mark.parametrize("P", [1, 3, 8])
def test_multi_rank_momentum_decode_exact(L, P):
    """Decode of P > 1 messages with heavy-ball momentum (one cooperative launch: scatter, grid
    barrier, dense update).  The reference has no momentum (R: SPEC.md:366), so its definition is
    this library's: total = fp64 rank-ordered sum of the sent values (R: training.py:248,253),
    m = fl32(mu * m + total / P), v = fl32(v - m) with fp64 intermediates -- emulated exactly in
    numpy over 6 chained steps (bit equality, not a tolerance)."""
    from paper_1911_08727_b200 import _native as N

    dims = [300_000, 7, 5_000, 70_001]
    ks = [300, 1, 50, 70]
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32, max_world=P)
    gen = torch.Generator(device="cuda").manual_seed(17 + P)
    rs = [torch.zeros(n, device="cuda") for _ in range(P)]
    v = torch.randn(n, device="cuda", generator=gen)
    m = torch.zeros(n, device="cuda")
    v_h = v.cpu().numpy().copy()
    m_h = m.cpu().numpy().copy()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    off = np.concatenate([[0], np.cumsum(dims)])
    mu = 0.9
    for t in range(6):
        msgs = b.new_messages(P)
        for p in range(P):
            b.compress(torch.randn(n, device="cuda", generator=gen), rs[p],
                       0.1, msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes], st)
        b.decode(msgs, P, v, momentum=m, mu=mu)
        total = np.zeros(n)
        for p in range(P):  # rank order, fp64 adds (entries a rank did not send add nothing)
            sent = np.zeros(n)
            for j, (ii, vv) in enumerate(b.unpack(msgs[p * b.msg_bytes:(p + 1) * b.msg_bytes])):
                sent[off[j] + ii] = vv
            total = total + sent
        mnew = np.float64(mu) * m_h.astype(np.float64) + total / np.float64(P)
        m_h = mnew.astype(np.float32)
        v_h = (v_h.astype(np.float64) - mnew).astype(np.float32)
        torch.cuda.synchronize()
        assert m.cpu().numpy().tobytes() == m_h.tobytes(), t
        assert v.cpu().numpy().tobytes() == v_h.tobytes(), t
    assert int(st.item()) == 0


def test_mixed_fast_path_equals_exact_path_and_oracle(L):
    """LAGS_F32_ACC64 (fp32 storage, numpy-float64 alpha: acc and values fp64, residual fp32; R:
    training.py:250-252 under NEP 50) on the fp64 fast path against its dense exact path and the
    oracle, bit for bit, through steady state, a threshold collapse and tie-heavy data."""
    from paper_1911_08727_b200 import _native as N

    dims = [20000, 64, 300000, 5000, 589824, 1000]
    ks = [max(1, d // 1000) for d in dims]
    fast = L.Bucket(dims, ks, N.F32_ACC64)
    exact = L.Bucket(dims, ks, N.F32_ACC64)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(17)
    r_f = torch.zeros(n, device="cuda")
    r_e = torch.zeros(n, device="cuda")
    r_h = np.zeros(n, dtype=np.float32)
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    off = np.concatenate([[0], np.cumsum(dims)])
    paths = set()
    for it in range(14):
        if it >= 11:  # integer-valued: many ties
            g = torch.randint(-6, 7, (n,), device="cuda", generator=gen).float()
        else:
            g = torch.randn(n, device="cuda", generator=gen)
        if it in (6, 7):
            g *= 1e-3
        alpha = np.float64(1.0 if it >= 11 else 0.05)
        fast.compress(g, r_f, alpha, m_f, st)
        exact.compress(g, r_e, alpha, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"messages differ at iteration {it}"
        assert torch.equal(r_f.view(torch.int32), r_e.view(torch.int32)), f"residuals differ at {it}"
        gh = g.cpu().numpy()
        acc = r_h.astype(np.float64) + alpha * gh.astype(np.float64)
        acc_sent = acc.copy()
        for j, (ii, vv) in enumerate(fast.unpack(m_f)):
            wi, wv = orc.top_k(acc[off[j]:off[j + 1]], ks[j])
            np.testing.assert_array_equal(ii, wi)
            assert vv.dtype == np.float64 and _same_bits(vv, wv), (it, j)
            acc_sent[off[j] + ii] = acc[off[j] + ii] - vv
        r_h = acc_sent.astype(np.float32)
        assert r_f.cpu().numpy().tobytes() == r_h.tobytes(), it
        paths.update(int(x) for x in fast.stats()[:, 5])
    assert 1 in paths, "the candidate path never ran"
    assert int(st.item()) == 0


def test_f64_fast_path_equals_exact_path_and_oracle(L):
    """The fp64 fast path (K1 on 64-bit keys with candidate lists + one CTA per layer) against the
    dense exact path and the oracle, bit for bit: steady state, a threshold collapse (too few
    candidates), a task-list overflow, an all-zero layer, tie-heavy integer data."""
    from paper_1911_08727_b200 import _native as N

    dims = [20000, 64, 300000, 5000, 589824, 70001, 1000]
    ks = [max(1, d // 1000) for d in dims]
    fast = L.Bucket(dims, ks, N.F64)
    exact = L.Bucket(dims, ks, N.F64)
    n = sum(dims)
    gen = torch.Generator(device="cuda").manual_seed(13)
    r_f = torch.zeros(n, device="cuda", dtype=torch.float64)
    r_e = torch.zeros(n, device="cuda", dtype=torch.float64)
    r_h = np.zeros(n)
    m_f, m_e = fast.new_messages(1), exact.new_messages(1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    off = np.concatenate([[0], np.cumsum(dims)])
    for it in range(20):
        if it >= 16:  # integer-valued: many ties
            g = torch.randint(-6, 7, (n,), device="cuda", generator=gen).double()
        else:
            g = torch.randn(n, device="cuda", generator=gen, dtype=torch.float64)
        if it in (7, 8):
            g *= 1e-3
        if it == 11:
            g[off[2]:off[2] + 8192] *= 1e4
        if it == 13:
            g[off[4]:off[5]] = 0.0
            r_f[off[4]:off[5]] = 0.0
            r_e[off[4]:off[5]] = 0.0
            r_h[off[4]:off[5]] = 0.0
        alpha = 1.0 if it >= 16 else 0.05
        fast.compress(g, r_f, alpha, m_f, st)
        exact.compress(g, r_e, alpha, m_e, st, exact=True)
        assert torch.equal(m_f, m_e), f"messages differ at iteration {it}"
        assert torch.equal(r_f.view(torch.int64), r_e.view(torch.int64)), f"residuals differ at {it}"
        gh = g.cpu().numpy()
        acc = r_h + alpha * gh
        for j, (ii, vv) in enumerate(fast.unpack(m_f)):
            wi, wv = orc.top_k(acc[off[j]:off[j + 1]], ks[j])
            np.testing.assert_array_equal(ii, wi)
            assert _same_bits(vv, wv), (it, j)
        acc_sent = acc.copy()
        for j, (ii, vv) in enumerate(fast.unpack(m_f)):
            acc_sent[off[j] + ii] = acc[off[j] + ii] - vv
        r_h = acc_sent
        assert r_f.cpu().numpy().tobytes() == r_h.tobytes(), it
    assert int(st.item()) == 0
