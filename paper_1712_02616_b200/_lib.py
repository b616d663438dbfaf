"""ctypes binding of libiabn.so (include/iabn.h).  Argument marshalling only.

The shared library is loaded from this package directory (built in-tree by
``paper_1712_02616_b200/build.py``).  There is no fallback: if the library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libiabn.so")

# status codes (iabn_status)
OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_ALIAS, ERR_DEGENERATE, ERR_WORKSPACE, ERR_CUDA, \
    ERR_NCCL = range(8)
# dtype / layout
F32, BF16 = 0, 1
NCHW, NHWC = 0, 1
# flags
GAMMA_PLAIN = 1 << 0
GAMMA_FIXED_ONE = 1 << 1
RUNNING_VAR_BIASED = 1 << 2
SYNC_GLOBAL_PARAM_GRADS = 1 << 3
EVAL = 1 << 4
VARIANT_I = 1 << 5
FORCE_STREAMING = 1 << 8
FORCE_FUSED = 1 << 9
FORCE_RESIDENT = 1 << 11
SYNC_FUSED = 1 << 12
ACT_SIGMOID = 1 << 13
ACT_TANH = 1 << 14

EXPORTS = ["iabn_version", "iabn_status_string", "iabn_last_error", "iabn_launch_count",
           "iabn_workspace_bytes", "iabn_query_schedule", "iabn_forward", "iabn_backward",
           "iabn_comm_get_unique_id", "iabn_comm_init", "iabn_comm_destroy", "iabn_forward_sync",
           "iabn_backward_sync", "iabn_forward_reduce", "iabn_forward_apply",
           "iabn_backward_reduce", "iabn_backward_apply", "iabn_fold_conv",
           "iabn_forward_sync_emulated", "iabn_backward_sync_emulated", "iabn_comm_set_timing",
           "iabn_comm_phase_ms"]


class Desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("c", ctypes.c_int64), ("hw", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("layout", ctypes.c_int32)]


class IabnError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        super().__init__(f"{fn} -> {_status_name(status)}: {detail}")
        self.status = status


_P = ctypes.c_void_p
_F = ctypes.c_float
_U32 = ctypes.c_uint32
_SZ = ctypes.c_size_t
_DP = ctypes.POINTER(Desc)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1712_02616_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.iabn_version.restype = ctypes.c_int
    lib.iabn_status_string.restype = ctypes.c_char_p
    lib.iabn_status_string.argtypes = [ctypes.c_int]
    lib.iabn_last_error.restype = ctypes.c_char_p
    lib.iabn_launch_count.restype = ctypes.c_uint64
    lib.iabn_workspace_bytes.restype = _SZ
    lib.iabn_workspace_bytes.argtypes = [_DP]
    lib.iabn_query_schedule.argtypes = [_DP, ctypes.c_int, _U32, ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int)]
    lib.iabn_forward.argtypes = [_DP, _P, _P, _P, _P, _P, _P, _P, _P, _F, _F, _F, _U32, _P, _SZ, _P]
    lib.iabn_backward.argtypes = [_DP, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _F, _U32, _P, _SZ,
                                  _P]
    lib.iabn_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.iabn_comm_init.argtypes = [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
    lib.iabn_comm_destroy.argtypes = [_P]
    lib.iabn_comm_set_timing.argtypes = [_P, ctypes.c_int]
    lib.iabn_comm_phase_ms.argtypes = [_P, ctypes.POINTER(ctypes.c_float)]
    lib.iabn_forward_sync.argtypes = lib.iabn_forward.argtypes + [_P]
    lib.iabn_backward_sync.argtypes = lib.iabn_backward.argtypes + [_P]
    lib.iabn_forward_reduce.argtypes = [_DP, _P, _P, _P, _SZ, _P]
    lib.iabn_forward_apply.argtypes = [_DP, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _F, _F, _U32,
                                       _P, _SZ, _P]
    lib.iabn_backward_reduce.argtypes = [_DP, _P, _P, _P, _P, _P, _F, _F, _U32, _P, _SZ, _P]
    lib.iabn_backward_apply.argtypes = [_DP, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _F, _U32,
                                        _P, _SZ, _P]
    lib.iabn_fold_conv.argtypes = [ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _F,
                                   _U32, _P, _P, _P]
    lib.iabn_forward_sync_emulated.argtypes = [_DP, ctypes.c_int] + lib.iabn_forward.argtypes[1:]
    lib.iabn_backward_sync_emulated.argtypes = [_DP, ctypes.c_int] + lib.iabn_backward.argtypes[1:]
    for name in EXPORTS:
        if name not in ("iabn_version", "iabn_status_string", "iabn_last_error",
                        "iabn_launch_count", "iabn_workspace_bytes"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


def _status_name(s: int) -> str:
    return lib.iabn_status_string(s).decode()


def check(status: int, fn: str) -> None:
    if status != OK:
        raise IabnError(status, fn, lib.iabn_last_error().decode())


_FNS: dict = {}


def call(name: str, *args) -> None:
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib, name)
    st = fn(*args)
    if st != OK:
        check(st, name)


def launch_count() -> int:
    return int(lib.iabn_launch_count())


def desc(n: int, c: int, hw: int, dtype: int, layout: int) -> Desc:
    return Desc(n, c, hw, dtype, layout)


def workspace_bytes(d: Desc) -> int:
    return int(lib.iabn_workspace_bytes(ctypes.byref(d)))


def query_schedule(d: Desc, pass_: int, flags: int = 0) -> tuple[int, int]:
    s, k = ctypes.c_int(0), ctypes.c_int(0)
    call("iabn_query_schedule", ctypes.byref(d), pass_, flags, ctypes.byref(s), ctypes.byref(k))
    return s.value, k.value
