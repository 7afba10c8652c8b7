"""ctypes binding of libnncp_b200.so (include/nncp_b200.h).

The product path has no CPU fallback: if the in-tree library is missing or no
CUDA device is present, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# NNCP_LIB_PATH: an instrumented build for the tools (tools/sliced_stats.py); never set by the product
LIB_PATH = os.environ.get("NNCP_LIB_PATH") or os.path.join(_HERE, "libnncp_b200.so")

NNCP_OK = 0
NNCP_ERR_VALUE = 1
NNCP_ERR_RUNTIME = 2
NNCP_ERR_CUDA = 3
NNCP_ERR_UNSUPPORTED = 4
SIDE_LEFT, SIDE_RIGHT = 0, 1
TTV_TRAILING, TTV_LEADING = 0, 1
ALGO_CODES = {"mu": 1, "hals": 2, "bpp": 3, "ucp": 4}
MAX_ORDER = 8
MAX_RANK = 64
STATUS_WORDS = 4
INT32_MAX = 2**31 - 1

c_i64p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p

# (name, restype, argtypes) for every symbol declared in include/nncp_b200.h
SIGNATURES = [
    ("nncp_abi_version", ctypes.c_int, []),
    ("nncp_last_error", ctypes.c_char_p, []),
    ("nncp_device_sms", ctypes.c_int, []),
    ("nncp_launch_count", ctypes.c_ulonglong, []),
    ("nncp_choose_split", ctypes.c_int, [ctypes.c_int, c_i64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("nncp_workspace_bytes", ctypes.c_size_t, [ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int]),
    ("nncp_norm_squared", ctypes.c_int, [vp, ctypes.c_int64, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_norm_squared_min", ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_partial_mttkrp", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int, vp, vp,
      ctypes.c_size_t, vp]),
    ("nncp_sliced_tensor_bytes", ctypes.c_int,
     [ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    ("nncp_norm_rowmax", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_slice_tensor_planes", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t, vp]),
    ("nncp_slice_tensor", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t, vp]),
    ("nncp_sliced_workspace_bytes", ctypes.c_size_t,
     [ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("nncp_partial_mttkrp_sliced", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, vp,
      vp, ctypes.c_size_t, vp]),
    ("nncp_partial_mttkrp_sliced_deferred", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, vp,
      vp, ctypes.c_size_t, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64), vp]),
    ("nncp_sliced_trailing_supported", ctypes.c_int,
     [ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("nncp_partial_mttkrp_sliced_trailing", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, vp, vp, vp,
      ctypes.c_size_t, vp]),
    ("nncp_multi_ttv", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), c_i64p, ctypes.c_int, vp, vp]),
    ("nncp_khatri_rao", ctypes.c_int, [vp, c_i64p, ctypes.c_int, ctypes.c_int, vp, vp]),
    ("nncp_temp_to_rows", ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int, vp, vp]),
    ("nncp_status_reset", ctypes.c_int, [vp, vp]),
    ("nncp_status_reset_n", ctypes.c_int, [vp, ctypes.c_int, vp]),
    ("nncp_update", ctypes.c_int,
     [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp, vp,
      ctypes.c_size_t, vp]),
    ("nncp_update_normalize", ctypes.c_int,
     [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp,
      ctypes.c_double, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp, vp,
      ctypes.c_size_t, vp]),
    ("nncp_bpp_sets_words", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int]),
    ("nncp_bpp_prepare", ctypes.c_int,
     [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, vp]),
    ("nncp_update_grouped", ctypes.c_int,
     [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
      vp, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_double, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_update_ex", ctypes.c_int,
     [ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp,
      ctypes.c_double, vp, ctypes.c_int64, vp, ctypes.c_size_t, vp]),
    ("nncp_normalize_gram", ctypes.c_int,
     [vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_gram", ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_gamma", ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]),
    ("nncp_normalize_from_gram", ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp]),
    ("nncp_normalize_gram_publish", ctypes.c_int,
     [vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp, vp, vp, ctypes.c_size_t, vp, ctypes.c_int, vp, vp, ctypes.c_int,
      vp, ctypes.c_int, ctypes.c_int, vp, vp]),
    ("nncp_gamma_publish", ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int,
                                          ctypes.c_int, vp, vp]),
    ("nncp_inner", ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_admm_step", ctypes.c_int,
     [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, vp, vp, vp, vp, ctypes.c_int64,
      vp, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_nes_hyper", ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, vp, vp]),
    ("nncp_nes_step", ctypes.c_int,
     [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int64, vp, vp,
      ctypes.c_size_t, vp]),
    ("nncp_scale_columns", ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp]),
    ("nncp_extrapolate", ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_double, vp, vp]),
    ("nncp_nes_lambda", ctypes.c_int, [vp, vp, ctypes.c_int, ctypes.c_int, vp, vp]),
    ("nncp_colsumsq", ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int, vp, vp, ctypes.c_size_t, vp]),
    ("nncp_synthetic", ctypes.c_int,
     [vp, ctypes.c_int, c_i64p, c_i64p, c_i64p, ctypes.POINTER(vp), ctypes.c_int, ctypes.c_double,
      ctypes.c_uint64, vp]),
]

_lib = None


def load(require_device: bool = True):
    """Load the in-tree library (raises loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1909_01149_b200.build_ext` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device and not torch.cuda.is_available():
        raise RuntimeError("paper_1909_01149_b200 needs a CUDA device (B200); no CPU fallback exists")
    return _lib


def check(rc: int):
    if rc == NNCP_OK:
        return
    msg = _lib.nncp_last_error().decode(errors="replace")
    if rc == NNCP_ERR_VALUE:
        raise ValueError(msg)
    if rc == NNCP_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def i64(values):
    values = [int(v) for v in values]
    return (ctypes.c_int64 * max(1, len(values)))(*values)


def ptrs(tensors):
    out = [t.data_ptr() if t is not None else None for t in tensors]
    return (vp * max(1, len(out)))(*out)


def ptr(t):
    return None if t is None else vp(t.data_ptr())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return vp(s.cuda_stream)
