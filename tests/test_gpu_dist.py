"""Multi-rank paths on the GPU.

* ``lags_step(..., group=...)`` with one worker per process must return, on every rank, the bits
  the single-process P-worker step returns (checked against the pinned oracle), update each rank's
  own residual exactly, and raise the same DivergenceError on every rank before any residual is
  written back: over NCCL with one GPU per rank (2 GPUs), and over gloo with both workers on one GPU.
* The peer-memory exchange: two ranks emulated in one process on one GPU (every push queued before
  every wait, so no kernel spins on a concurrently running one), and over CUDA IPC between two
  processes on two GPUs against the NCCL all-gather."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lagsgd_oracle as orc  # noqa: E402

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(it):
    rng = np.random.default_rng(500 + it)
    dtype = [np.float32, np.float64][it % 2]
    dims = [int(x) for x in rng.integers(1, 300_000, size=int(rng.integers(1, 9)))]
    if it == 2:
        dims = [5_000_000, 3, 70_000]  # spans several pipeline chunks
    n = sum(dims)
    counts = [max(1, d // int(rng.choice([1, 10, 100, 1000]))) for d in dims]
    v = rng.standard_normal(n).astype(dtype)
    grads = [(rng.standard_normal(n) * np.exp(rng.standard_normal(n))).astype(dtype) for _ in range(WORLD)]
    res = [(0.01 * rng.standard_normal(n)).astype(dtype) for _ in range(WORLD)]
    alpha = float(rng.uniform(0.01, 1.0))
    return dims, counts, v, grads, res, alpha


SLGS_K = 50


def _slgs_case():
    rng = np.random.default_rng(900)
    dims = [30_000, 5_000, 17]
    n = sum(dims)
    v = rng.standard_normal(n).astype(np.float32)
    grads = [rng.standard_normal(n).astype(np.float32) for _ in range(WORLD)]
    res = [(0.01 * rng.standard_normal(n)).astype(np.float32) for _ in range(WORLD)]
    return dims, v, grads, res, 0.3


def _worker(rank, port, out_dir):
    import torch.distributed as dist

    import paper_1911_08727_b200 as L

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    grp = dist.group.WORLD
    lv = lambda dims, a: L.LayeredVector([L.LayerShape(i + 1, d) for i, d in enumerate(dims)], a)  # noqa: E731
    save = {}
    for it in range(4):
        dims, counts, v, grads, res, alpha = _case(it)
        r = lv(dims, res[rank].copy())
        vv = lv(dims, v)
        for t in range(2):  # two chained steps (residuals carry over)
            vv = L.lags_step(vv, [lv(dims, grads[rank] * (t + 1))], alpha, {i + 1: k for i, k in enumerate(counts)},
                             [r], t=t, group=grp)
        save[f"v{it}"] = vv.data
        save[f"r{it}"] = r.data
    # SLGS arm in group mode (whole-vector selection, fp64 parameters out)
    dims, v, grads, res, alpha = _slgs_case()
    r = lv(dims, res[rank].copy())
    out = L.slgs_step(lv(dims, v), [lv(dims, grads[rank])], alpha, SLGS_K, [r], t=0, group=grp)
    save["slgs_v"] = out.data
    save["slgs_r"] = r.data
    # divergence: rank 1's gradient is non-finite -> both ranks raise naming worker 2, residuals untouched
    dims = [1000]
    g = np.ones(1000, np.float32)
    if rank == 1:
        g[7] = np.nan
    r = lv(dims, np.full(1000, 0.5, np.float32))
    try:
        L.lags_step(lv(dims, np.zeros(1000, np.float32)), [lv(dims, g)], 0.1, {1: 3}, [r], t=9, group=grp)
        save["div"] = np.array("no error")
    except L.DivergenceError as e:
        save["div"] = np.array(f"{e.iteration}:{e}")
    save["div_res_ok"] = np.array(bool(np.all(r.data == 0.5)))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **save)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu2
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < WORLD, reason="needs 2 GPUs")
def test_two_rank_nccl_lags_step_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    outs = [np.load(tmp_path / f"rank{p}.npz") for p in range(WORLD)]
    for it in range(4):
        dims, counts, v, grads, res, alpha = _case(it)
        for t in range(2):
            v = orc.lags_step(v, [g * (t + 1) for g in grads], alpha, dims, counts, res)
        for p in range(WORLD):
            assert outs[p][f"v{it}"].tobytes() == v.tobytes(), (it, p)
            assert outs[p][f"r{it}"].tobytes() == res[p].tobytes(), (it, p)
    dims, v, grads, res, alpha = _slgs_case()
    want = orc.slgs_step(v, grads, alpha, SLGS_K, res)
    for p in range(WORLD):
        assert outs[p]["slgs_v"].dtype == want.dtype and outs[p]["slgs_v"].tobytes() == want.tobytes(), p
        assert outs[p]["slgs_r"].tobytes() == res[p].tobytes(), p
    for p in range(WORLD):
        msg = str(outs[p]["div"])
        assert msg.startswith("9:") and "worker 2" in msg, msg
        assert bool(outs[p]["div_res_ok"])


def _p2p_worker(rank, port, out_dir):
    import torch.distributed as dist

    import paper_1911_08727_b200 as L
    from paper_1911_08727_b200 import _native as N
    from paper_1911_08727_b200.p2p import PeerExchange

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    dims = [600_000, 70_001, 4_096, 300_000, 1_000]
    ks = [max(1, d // 1000) for d in dims]
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32, max_world=WORLD)
    gen = torch.Generator(device="cuda").manual_seed(40 + rank)
    r = torch.zeros(n, device="cuda")
    v0 = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
    v_p2p, v_nccl = v0.clone(), v0.clone()
    msg = b.new_messages(1)
    msgs = b.new_messages(WORLD)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ex = PeerExchange(b.msg_bytes, ctas_per_peer=2, timeout_s=10.0)
    ok = True
    for t in range(40):
        g = torch.randn(n, device="cuda", generator=gen)
        b.compress(g, r, 0.1, msg, st)
        b.decode(ex.exchange(msg), WORLD, v_p2p)  # peer-memory exchange
        dist.all_gather_into_tensor(msgs, msg)     # reference: NCCL all-gather
        b.decode(msgs, WORLD, v_nccl)
        ok &= bool(torch.equal(v_p2p.view(torch.int32), v_nccl.view(torch.int32)))
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"p2p{rank}.npz"), ok=np.array(ok), status=np.array(int(ex.status.item())),
             st=np.array(int(st.item())), v=v_p2p.cpu().numpy())
    ex.close()
    dist.destroy_process_group()


@pytest.mark.gpu2
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < WORLD, reason="needs 2 GPUs")
def test_two_rank_peer_memory_exchange_equals_nccl(tmp_path):
    """The peer-memory exchange (CUDA IPC push + flag wait, double-buffered) delivers exactly the
    NCCL all-gather's messages: decoded weights bit-identical on every rank, 40 chained steps."""
    import torch.multiprocessing as mp

    mp.spawn(_p2p_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    outs = [np.load(tmp_path / f"p2p{p}.npz") for p in range(WORLD)]
    for o in outs:
        assert bool(o["ok"]) and int(o["status"]) == 0 and int(o["st"]) == 0
    assert outs[0]["v"].tobytes() == outs[1]["v"].tobytes()  # replicas agree


@pytest.mark.parametrize("fused", [False, True])
def test_peer_memory_protocol_two_ranks_one_process(fused):
    """The peer-memory exchange kernels (lags_p2p_push / lags_p2p_wait; fused: the selection pushes
    every finished layer itself, lags_bucket_compress_push) with two ranks emulated in
    ONE process on one GPU: both receive areas are plain device allocations, both pushes are queued
    before either wait on the same stream (no kernel ever spins on another running kernel), and the
    epochs / parities advance as in PeerExchange.  Each emulated rank decodes its own area; both
    must equal the decode of the directly concatenated messages, and the oracle's P = 2 step,
    bit for bit over 24 chained steps (both parities, the epoch wrap of the flags)."""
    import ctypes as C

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1911_08727_b200 as L
    from paper_1911_08727_b200 import _native as N
    from paper_1911_08727_b200.engine import stream_handle

    P, G = 2, 2
    dims = [300_000, 70_001, 4_096, 1_000]
    ks = [max(1, d // 1000) for d in dims]
    n = sum(dims)
    b = L.Bucket(dims, ks, N.F32, max_world=P)
    mb = b.msg_bytes
    flags_bytes = (P * G * 4 + 255) // 256 * 256
    area_bytes = flags_bytes + 2 * P * mb
    areas = []
    for _ in range(P):
        ptr, handle = C.c_void_p(), (C.c_char * 64)()
        N.check(N.lags_ipc_malloc(area_bytes, C.byref(ptr), handle), "lags_ipc_malloc")
        areas.append(int(ptr.value))
    bases = torch.tensor([a - (1 << 64) if a >= (1 << 63) else a for a in areas], dtype=torch.int64, device="cuda")
    epochs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(P)]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = stream_handle(torch.cuda.current_stream())
    rng = np.random.default_rng(31)
    v_host = rng.standard_normal(n).astype(np.float32)
    res_host = [np.zeros(n, np.float32) for _ in range(P)]
    r = [torch.zeros(n, device="cuda") for _ in range(P)]
    v_rank = [torch.from_numpy(v_host).cuda() for _ in range(P)]
    v_cat = torch.from_numpy(v_host).cuda()
    msgs = [b.new_messages(1) for _ in range(P)]
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    try:
        for t in range(24):
            grads = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
            for p in range(P):  # every push first ...
                if fused:
                    desc = N.PeerPushDesc(bases.data_ptr(), P, p, G, flags_bytes, epochs[p].data_ptr())
                    N.check(N.lags_bucket_compress_push(b._h, torch.from_numpy(grads[p]).cuda().data_ptr(),
                                                        r[p].data_ptr(), 0.1, msgs[p].data_ptr(), st.data_ptr(), 0,
                                                        C.byref(desc), s), "lags_bucket_compress_push")
                    torch.cuda.synchronize()  # the gradient tensor above is a temporary
                else:
                    b.compress(torch.from_numpy(grads[p]).cuda(), r[p], 0.1, msgs[p], st)
                    N.check(N.lags_p2p_push(msgs[p].data_ptr(), mb, bases.data_ptr(), P, p, G, flags_bytes,
                                            epochs[p].data_ptr(), s), "lags_p2p_push")
            for p in range(P):  # ... then every wait: the flags are already published
                N.check(N.lags_p2p_wait(areas[p], P * G, epochs[p].data_ptr(), status.data_ptr(), int(5e9), s),
                        "lags_p2p_wait")
            par = (t + 1) & 1  # the epoch of exchange t is t + 1
            for p in range(P):
                addr = areas[p] + flags_bytes + par * P * mb

                class _View:
                    def data_ptr(self, a=addr):
                        return a

                    def numel(self):
                        return P * mb

                b.decode(_View(), P, v_rank[p])
            b.decode(torch.cat(msgs), P, v_cat)
            v_host = orc.lags_step(v_host, grads, 0.1, dims, ks, res_host)
            torch.cuda.synchronize()
            assert int(status.item()) == 0 and int(st.item()) == 0
            for p in range(P):
                assert torch.equal(v_rank[p].view(torch.int32), v_cat.view(torch.int32)), (t, p)
                assert r[p].cpu().numpy().tobytes() == res_host[p].tobytes(), (t, p)
            assert v_cat.cpu().numpy().tobytes() == v_host.tobytes(), t
            assert [int(e.item()) for e in epochs] == [t + 1] * P
    finally:
        torch.cuda.synchronize()
        for a in areas:
            N.lags_ipc_free(a)


def _gloo_worker(rank, port, out_dir):
    import torch.distributed as dist

    import paper_1911_08727_b200 as L

    torch.cuda.set_device(0)  # both workers share the one GPU; gloo moves the messages via the host
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    grp = dist.group.WORLD
    lv = lambda dims, a: L.LayeredVector([L.LayerShape(i + 1, d) for i, d in enumerate(dims)], a)  # noqa: E731
    save = {}
    for it in range(4):
        dims, counts, v, grads, res, alpha = _case(it)
        r = lv(dims, res[rank].copy())
        vv = lv(dims, v)
        for t in range(2):
            vv = L.lags_step(vv, [lv(dims, grads[rank] * (t + 1))], alpha, {i + 1: k for i, k in enumerate(counts)},
                             [r], t=t, group=grp)
        save[f"v{it}"] = vv.data
        save[f"r{it}"] = r.data
    dims = [1000]
    g = np.ones(1000, np.float32)
    if rank == 1:
        g[7] = np.nan
    r = lv(dims, np.full(1000, 0.5, np.float32))
    try:
        L.lags_step(lv(dims, np.zeros(1000, np.float32)), [lv(dims, g)], 0.1, {1: 3}, [r], t=9, group=grp)
        save["div"] = np.array("no error")
    except L.DivergenceError as e:
        save["div"] = np.array(f"{e.iteration}:{e}")
    save["div_res_ok"] = np.array(bool(np.all(r.data == 0.5)))
    np.savez(os.path.join(out_dir, f"gloo{rank}.npz"), **save)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_group_dropin_one_gpu_gloo(tmp_path):
    """lags_step(..., group=) with two worker processes sharing one GPU over a gloo group (host-staged
    gathers, no kernel waits on another process's kernel): every rank returns the oracle's
    P-worker parameters and its own residual bit for bit, and both raise the same DivergenceError
    before any residual is written back."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp

    mp.spawn(_gloo_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    outs = [np.load(tmp_path / f"gloo{p}.npz") for p in range(WORLD)]
    for it in range(4):
        dims, counts, v, grads, res, alpha = _case(it)
        for t in range(2):
            v = orc.lags_step(v, [g * (t + 1) for g in grads], alpha, dims, counts, res)
        for p in range(WORLD):
            assert outs[p][f"v{it}"].tobytes() == v.tobytes(), (it, p)
            assert outs[p][f"r{it}"].tobytes() == res[p].tobytes(), (it, p)
    for p in range(WORLD):
        msg = str(outs[p]["div"])
        assert msg.startswith("9:") and "worker 2" in msg, msg
        assert bool(outs[p]["div_res_ok"])


@pytest.mark.gpu2
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < WORLD, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", ["p2p", "fused", "nccl"])
def test_two_rank_lagssgd_matches_oracle(mode):
    """LagsSGD on two ranks (compress on the side stream, exchange + decode on the communication
    stream; peer-memory push or NCCL all-gather): parameters bit-identical to the oracle's P = 2
    step on every rank, 10 steps (tools/multi_gpu_check.py under torchrun)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={WORLD}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tools", "multi_gpu_check.py"), mode]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "OK" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
