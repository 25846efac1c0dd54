"""C-ABI library checks that need no GPU: it loads, exports every declared symbol, and rejects bad
arguments with the reference's error classes before touching the device."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lags_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|size_t|const char\*|unsigned long long)\s+(lags_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("lags_bucket_compress", "lags_bucket_decode_update", "lags_bucket_create", "lags_top_k",
                 "lags_decompress", "lags_check_finite"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_1911_08727_b200._native as N

    lib = ctypes.CDLL(N.library_path())
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(N.EXPORTS) == set(declared_functions())
    assert N.lags_abi_version() == 3


def test_argument_errors_map_to_reference_exceptions():
    import paper_1911_08727_b200._native as N

    rc = N.lags_top_k(N.F32, None, 10, 3, None, None, None, None, 0, None)
    assert rc == N.ERR_INVALID_ARG
    with pytest.raises(ValueError):
        N.check(rc)
    # k outside 1..dim with non-null (never dereferenced) pointers
    fake = 16
    rc = N.lags_top_k(N.F32, fake, 10, 11, fake, fake, fake, fake, 1 << 20, None)
    assert rc == N.ERR_K_OUT_OF_RANGE
    with pytest.raises(ValueError, match="outside 1..10"):
        N.check(rc)
    assert N.lags_bucket_compress(None, None, None, 0.0, None, None, 0, None) == N.ERR_INVALID_ARG
    assert N.lags_bucket_decode_update(None, fake, 64, 1, fake, None, 0.0, 0, None) == N.ERR_INVALID_ARG
    # bucket creation validates k before touching the device (R: sparsify.py:82-83)
    dims = np.array([10, 5], dtype=np.int64)
    ks = np.array([3, 6], dtype=np.int32)
    assert N.lags_bucket_device_bytes(N.F32, dims.ctypes.data, ks.ctypes.data, 2, 1) == 0
    h = ctypes.c_void_p()
    rc = N.lags_bucket_create(N.F32, dims.ctypes.data, ks.ctypes.data, 2, 1, fake, 1 << 20, None, ctypes.byref(h))
    assert rc == N.ERR_K_OUT_OF_RANGE and b"outside 1..5" in N.lags_last_error()


def test_workspace_sizes():
    import paper_1911_08727_b200._native as N
    from bench import resnet50_dims, ks_for

    dims = resnet50_dims()
    d = np.asarray(dims, dtype=np.int64)
    k = np.asarray(ks_for(dims), dtype=np.int32)
    n = int(d.sum())
    b1 = N.lags_bucket_device_bytes(N.F32, d.ctypes.data, k.ctypes.data, len(dims), 1)
    b8 = N.lags_bucket_device_bytes(N.F32, d.ctypes.data, k.ctypes.data, len(dims), 8)
    assert b8 - b1 >= 7 * 4 * n - 4096  # one decode plane per extra rank
    assert b1 < 512 * 2**20
    assert N.lags_top_k_workspace_bytes(N.F64, 1000) >= 8000


def test_host_policy_and_chunk_invariants():
    from paper_1911_08727_b200 import CompressionPolicy, LayerShape, SparseChunk, StructureError
    from paper_1911_08727_b200.training import mode_for
    import paper_1911_08727_b200._native as N

    shape = (LayerShape(1, 100), LayerShape(2, 15), LayerShape(3, 3))
    pol = CompressionPolicy({1: 10.0, 2: 10.0, 3: 10.0}, ratio_cap=10.0)
    assert pol.selection_counts(shape) == {1: 10, 2: 1, 3: 1}
    assert pol.effective_max_ratio(shape) == 15.0
    assert CompressionPolicy.from_density(0.01, [LayerShape(1, 68)]).selection_counts([LayerShape(1, 68)]) == {1: 1}
    with pytest.raises(ValueError):
        CompressionPolicy({1: 0.5}, ratio_cap=10.0)
    with pytest.raises(ValueError):
        CompressionPolicy({1: 20.0}, ratio_cap=10.0)
    with pytest.raises(StructureError):
        SparseChunk(0, 4, np.array([2, 1]), np.array([1.0, 2.0]), k_target=2)
    with pytest.raises(StructureError):
        SparseChunk(0, 4, np.array([0, 5]), np.array([1.0, 2.0]), k_target=2)
    assert mode_for(np.float32, 0.1) == N.F32
    assert mode_for(np.float32, np.float64(0.1)) == N.F32_ACC64
    assert mode_for(np.float64, 0.1) == N.F64
