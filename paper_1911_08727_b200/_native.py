"""ctypes binding of liblagsb200.so (include/lags_b200.h).

The library is the product: there is no CPU fallback.  Importing this module
fails loudly if the in-tree library has not been built.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import StructureError

# LAGS_B200_LIB: an alternative build of the same library (kernel variants under study); the
# default is the in-tree build
_LIB_PATH = os.environ.get("LAGS_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "liblagsb200.so")

F32, F64, F32_ACC64 = 0, 1, 2
STATUS_NONFINITE = 0x1
COMPRESS_EXACT = 0x1
COMPRESS_ZERO_GRAD = 0x2
OK, ERR_INVALID_ARG, ERR_K_OUT_OF_RANGE, ERR_STRUCTURE, ERR_WORKSPACE, ERR_CUDA = 0, -1, -2, -3, -4, -5

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
    )

lib = C.CDLL(_LIB_PATH)

_vp, _i32, _u32, _i64, _sz, _dbl = C.c_void_p, C.c_int32, C.c_uint32, C.c_int64, C.c_size_t, C.c_double
_i64p = C.POINTER(C.c_int64)


def _fn(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


lags_abi_version = _fn("lags_abi_version", C.c_int)
lags_last_error = _fn("lags_last_error", C.c_char_p)
lags_kernel_launches = _fn("lags_kernel_launches", C.c_ulonglong)
lags_bucket_device_bytes = _fn("lags_bucket_device_bytes", _sz, _i32, _vp, _vp, _i32, _i32)
lags_bucket_create = _fn("lags_bucket_create", C.c_int, _i32, _vp, _vp, _i32, _i32, _vp, _sz, _vp,
                         C.POINTER(_vp))
lags_bucket_destroy = _fn("lags_bucket_destroy", None, _vp)
lags_bucket_message_layout = _fn("lags_bucket_message_layout", C.c_int, _vp, _i64p, _i64p, _i64p, _i64p)
lags_bucket_compress = _fn("lags_bucket_compress", C.c_int, _vp, _vp, _vp, _dbl, _vp, _vp, _u32, _vp)


class PeerPushDesc(C.Structure):
    """lags_peer_push_t (include/lags_b200.h)."""
    _fields_ = [("bases", C.c_void_p), ("P", C.c_int32), ("rank", C.c_int32), ("ctas_per_peer", C.c_int32),
                ("flags_bytes", C.c_uint64), ("epoch", C.c_void_p)]


lags_bucket_compress_push = _fn("lags_bucket_compress_push", C.c_int, _vp, _vp, _vp, _dbl, _vp, _vp, _u32,
                                C.POINTER(PeerPushDesc), _vp)
lags_bucket_decode_update = _fn("lags_bucket_decode_update", C.c_int, _vp, _vp, _i64, _i32, _vp, _vp, _dbl, _u32,
                                _vp)
DECODE_V64 = 0x1
lags_bucket_stats = _fn("lags_bucket_stats", C.c_int, _vp, _vp, _vp)
lags_bucket_step_local = _fn("lags_bucket_step_local", C.c_int, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _u32, _vp)
lags_bucket_set_probe_events = _fn("lags_bucket_set_probe_events", C.c_int, _vp, _vp, _vp)
lags_bucket_set_grad_table = _fn("lags_bucket_set_grad_table", C.c_int, _vp, _vp)
lags_bucket_reconstruct = _fn("lags_bucket_reconstruct", C.c_int, _vp, _vp, _i64, _i32, _vp, _vp, _i64, _vp)
lags_bucket_delta = _fn("lags_bucket_delta", C.c_int, _vp, _vp, _vp, _i64, _i32, _vp, _vp)
lags_bucket_shadow_step = _fn("lags_bucket_shadow_step", C.c_int, _vp, _vp, _vp, _dbl, _i32, _vp)
lags_bucket_identity = _fn("lags_bucket_identity", C.c_int, _vp, _vp, _vp, _vp, _i32, _vp, _vp)
lags_check_finite = _fn("lags_check_finite", C.c_int, _i32, _vp, _i64, _vp, _vp)
lags_top_k_workspace_bytes = _fn("lags_top_k_workspace_bytes", _sz, _i32, _i64)
lags_top_k = _fn("lags_top_k", C.c_int, _i32, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp)
lags_decompress = _fn("lags_decompress", C.c_int, _i32, _vp, _vp, _vp, _i64, _vp, _vp)
lags_wire_encode = _fn("lags_wire_encode", C.c_int, _u32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _i64, _vp,
                       _vp, _vp)
lags_wire_decode = _fn("lags_wire_decode", C.c_int, _u32, _vp, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                       _vp, _i32, _vp, _vp, _vp, _vp)
lags_ipc_malloc = _fn("lags_ipc_malloc", C.c_int, _sz, C.POINTER(_vp), _vp)
lags_ipc_open = _fn("lags_ipc_open", C.c_int, _vp, C.POINTER(_vp))
lags_ipc_close = _fn("lags_ipc_close", C.c_int, _vp)
lags_ipc_free = _fn("lags_ipc_free", C.c_int, _vp)
lags_p2p_push = _fn("lags_p2p_push", C.c_int, _vp, _i64, _vp, _i32, _i32, _i32, C.c_uint64, _vp, _vp)
lags_p2p_wait = _fn("lags_p2p_wait", C.c_int, _vp, _i32, _vp, _vp, C.c_uint64, _vp)
STATUS_P2P_TIMEOUT = 0x100
WIRE_MESSAGE, WIRE_CHUNK = 0, 1
WIRE_MAX_CHUNKS = 4096
(WIRE_ERR_TRUNCATED_MESSAGE, WIRE_ERR_TRUNCATED_HEADER, WIRE_ERR_TRUNCATED_PAYLOAD, WIRE_ERR_INDEX_RANGE,
 WIRE_ERR_INDEX_ORDER, WIRE_ERR_TRAILING, WIRE_ERR_CAPACITY) = range(1, 8)
WIRE_OK = (1 << 64) - 1

EXPORTS = [
    "lags_abi_version", "lags_last_error", "lags_kernel_launches", "lags_bucket_device_bytes",
    "lags_bucket_create", "lags_bucket_destroy", "lags_bucket_message_layout", "lags_bucket_compress",
    "lags_bucket_compress_push",
    "lags_bucket_decode_update", "lags_bucket_stats", "lags_bucket_step_local", "lags_bucket_set_probe_events", "lags_bucket_set_grad_table",
    "lags_check_finite", "lags_bucket_reconstruct", "lags_bucket_delta", "lags_bucket_shadow_step",
    "lags_bucket_identity",
    "lags_top_k_workspace_bytes",
    "lags_top_k", "lags_decompress", "lags_wire_encode", "lags_wire_decode",
    "lags_ipc_malloc", "lags_ipc_open", "lags_ipc_close", "lags_ipc_free", "lags_p2p_push", "lags_p2p_wait",
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
