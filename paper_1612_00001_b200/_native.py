"""ctypes binding of libbri_b200.so (C ABI: include/bri_b200.h).

The product path has no CPU fallback: if the shared library or a CUDA device
is missing, every entry point raises DeviceError.  The library is built
in-tree (`make -C paper_1612_00001_b200/csrc` or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BRI_LIB") or os.path.join(_HERE, "libbri_b200.so")

# (name, restype, argtypes) — must match include/bri_b200.h
_c_int, _c_void_p, _c_double, _c_ll = ctypes.c_int, ctypes.c_void_p, ctypes.c_double, ctypes.c_longlong
_P_INT = ctypes.POINTER(ctypes.c_int)
SIGNATURES = [
    ("bri_version", _c_int, []),
    ("bri_launch_count", _c_ll, []),
    ("bri_flop_count", _c_ll, [_c_int]),
    ("bri_last_error", ctypes.c_char_p, []),
    ("bri_ctx_create", _c_int, [_c_int, ctypes.POINTER(_c_void_p)]),
    ("bri_ctx_destroy", None, [_c_void_p]),
    ("bri_arena_create", _c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, ctypes.POINTER(_c_void_p)]),
    ("bri_arena_destroy", None, [_c_void_p]),
    ("bri_schur_batch", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_void_p]),
    ("bri_invert_batch", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_void_p]),
    ("bri_getrf_batch", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_void_p, _c_void_p, _c_void_p]),
    ("bri_getrs_batch", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_void_p]),
    ("bri_gemm", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT] + [_c_int] * 9 + [_c_double, _c_double]),
    ("bri_axpby", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_double, _c_double]),
    ("bri_transpose", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT]),
    ("bri_gather_blocks", _c_int, [_c_void_p, _c_void_p, _c_void_p, _c_ll, _c_int, _P_INT]),
    ("bri_gather_elements", _c_int, [_c_void_p, _c_void_p, _c_void_p, _c_ll, _c_int, _c_void_p, _c_void_p,
                                     _c_int, _P_INT]),
    ("bri_rbf_blocks", _c_int, [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_double, _c_double,
                                _c_void_p, _c_void_p, _c_int, _P_INT]),
    ("bri_rbf_dense", _c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_double, _c_double, _c_void_p, _c_ll]),
    ("bri_randn_blocks", _c_int, [_c_void_p, _c_void_p, _c_ll, ctypes.c_ulonglong, _c_double, _c_void_p,
                                  _c_void_p, _c_int, _P_INT]),
    ("bri_randn_window", _c_int, [_c_void_p, _c_ll, ctypes.c_ulonglong, _c_double, _c_ll, _c_ll, _c_int, _c_int,
                                  _c_void_p, _c_ll]),
    ("bri_load_host_blocks", _c_int, [_c_void_p, _c_void_p, _c_void_p, _c_ll, _c_int, _P_INT]),
    ("bri_schur_batch_gated", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_void_p, _c_void_p, _c_void_p]),
    ("bri_fp64_peak", _c_int, [_c_void_p, _c_int, ctypes.POINTER(_c_double)]),
    ("bri_level_batch", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_int, _P_INT, _c_int, _P_INT, _c_void_p]),
    ("bri_store_host", _c_int, [_c_void_p, _c_void_p, ctypes.c_longlong, _c_void_p, ctypes.c_longlong, _c_int,
                                _c_int]),
    ("bri_dag_small", _c_int, [_c_void_p, _c_void_p, _c_void_p, _c_ll, _c_int, _P_INT, _c_int, _P_INT, _P_INT,
                               _c_void_p, _c_int, _P_INT, _c_void_p]),
    ("bri_level_batch_ex", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_int, _P_INT, _c_int, _P_INT, _c_int,
                                    _P_INT, _c_int, _P_INT, _c_void_p, _c_void_p, _c_void_p]),
    ("bri_level_batch_gated", _c_int, [_c_void_p, _c_void_p, _c_int, _P_INT, _c_int, _P_INT, _c_int, _P_INT,
                                       _c_void_p, _c_void_p, _c_void_p]),
]

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no CUDA call is made)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"{path} not built: run `make -C {os.path.join(_HERE, 'csrc')}` "
                    "(there is no CPU fallback for the BRI hot path)")
            lib = ctypes.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().bri_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed ({rc}): {msg}")


def int_array(values):
    arr = (ctypes.c_int * len(values))(*values)
    return arr


_ctx = {}


def context(device: int):
    """Process-wide bri_ctx for a device, driven from one stream per thread."""
    key = (device, threading.get_ident())
    ctx = _ctx.get(key)
    if ctx is None:
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("CUDA device required: the BRI hot path runs only on the GPU")
        lib = load_library()
        out = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(lib.bri_ctx_create(device, ctypes.byref(out)), "bri_ctx_create")
        ctx = out
        _ctx[key] = ctx
    return ctx
