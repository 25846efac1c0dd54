"""ctypes binding of liblagsb200.so (include/lags_b200.h).

The library is the product: there is no CPU fallback.  Importing this module
fails loudly if the in-tree library has not been built.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import StructureError

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblagsb200.so")

F32, F64, F32_ACC64 = 0, 1, 2
STATUS_NONFINITE = 0x1
OK, ERR_INVALID_ARG, ERR_K_OUT_OF_RANGE, ERR_STRUCTURE, ERR_WORKSPACE, ERR_CUDA = 0, -1, -2, -3, -4, -5

# lags_layer_t: {int64 offset, int64 dim, int32 k, int32 slot} -- 24 bytes, no padding
LAYER_DTYPE = np.dtype([("offset", "<i8"), ("dim", "<i8"), ("k", "<i4"), ("slot", "<i4")])
# lags_layer_state_t: {uint64 pred_key, uint32 flags, uint32 last_cands} -- 16 bytes
STATE_BYTES = 16

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
    )

lib = C.CDLL(_LIB_PATH)

_vp, _i32, _i64, _u32p, _i32p, _sz, _dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t, C.c_double


def _fn(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


lags_abi_version = _fn("lags_abi_version", C.c_int)
lags_last_error = _fn("lags_last_error", C.c_char_p)
lags_kernel_launches = _fn("lags_kernel_launches", C.c_ulonglong)
lags_compress_workspace_bytes = _fn("lags_compress_workspace_bytes", _sz, _i32, _i32, _i64, _i64)
lags_compress = _fn("lags_compress", C.c_int, _i32, _vp, _i32, _i64, _i64, _vp, _vp, _dbl, _vp, _vp, _vp, _vp,
                    _vp, _vp, _sz, _vp)
lags_check_finite = _fn("lags_check_finite", C.c_int, _i32, _vp, _i64, _vp, _vp)
lags_top_k_workspace_bytes = _fn("lags_top_k_workspace_bytes", _sz, _i32, _i64)
lags_top_k = _fn("lags_top_k", C.c_int, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
lags_decompress = _fn("lags_decompress", C.c_int, _i32, _vp, _vp, _vp, _i64, _vp, _vp)
lags_decode_workspace_bytes = _fn("lags_decode_workspace_bytes", _sz, _i32, _i64, _i32)
lags_decode_update = _fn("lags_decode_update", C.c_int, _i32, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _i64, _i32,
                         _vp, _vp, _dbl, _vp, _sz, _vp)

EXPORTS = [
    "lags_abi_version", "lags_last_error", "lags_kernel_launches", "lags_compress_workspace_bytes", "lags_compress",
    "lags_check_finite", "lags_top_k_workspace_bytes", "lags_top_k", "lags_decompress",
    "lags_decode_workspace_bytes", "lags_decode_update",
]


def check(rc: int, what: str = "") -> None:
    """Map a lags_status_t to the reference's exception types (R: errors.py, sparsify.py:80-83)."""
    if rc == OK:
        return
    msg = (lags_last_error() or b"").decode(errors="replace") or what
    if rc in (ERR_INVALID_ARG, ERR_K_OUT_OF_RANGE):
        raise ValueError(msg)
    if rc == ERR_STRUCTURE:
        raise StructureError(msg)
    raise RuntimeError(f"liblagsb200 error {rc}: {msg}")


def library_path() -> str:
    return _LIB_PATH
