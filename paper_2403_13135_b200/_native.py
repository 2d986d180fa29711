"""ctypes binding of the C ABI in include/icelabel_b200.h (libicelabel_b200.so).

There is no CPU fallback: if the library is missing or no CUDA device is present, every
product call raises.  `load()` only needs the file (symbol checks work without a GPU).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ICE_LIB_PATH") or os.path.join(_HERE, "_C", "libicelabel_b200.so")

ICE_OK, ICE_EINVAL, ICE_EWINDOW, ICE_ETOOBIG, ICE_ENODRIVER = 0, -1, -2, -3, -4
_ERRNAMES = {ICE_EINVAL: "ICE_EINVAL", ICE_EWINDOW: "ICE_EWINDOW", ICE_ETOOBIG: "ICE_ETOOBIG",
             ICE_ENODRIVER: "ICE_ENODRIVER"}


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int):
        self.code = code
        what = _ERRNAMES.get(code, f"CUDA error {code}")
        super().__init__(f"{fn} failed: {what}")


class IceFilterCfg(ctypes.Structure):
    _fields_ = [("bg_dilate_k", ctypes.c_int32), ("bg_median_k", ctypes.c_int32),
                ("noise_median_k", ctypes.c_int32), ("mask_mode_fixed", ctypes.c_int32),
                ("fixed_t", ctypes.c_int32), ("diff_truncate", ctypes.c_int32),
                ("truncate_t", ctypes.c_int32)]


class IceScheme(ctypes.Structure):
    _fields_ = [("lo", (ctypes.c_uint8 * 3) * 3), ("hi", (ctypes.c_uint8 * 3) * 3),
                ("cls", ctypes.c_uint8 * 3), ("pad", ctypes.c_uint8 * 5)]


_V = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F32 = ctypes.c_float

# name -> argtypes (restype is always int32).  Kept in sync with include/icelabel_b200.h;
# tests/test_native_abi.py checks both directions.
SIGNATURES = {
    "ice_autolabel": [_V, _I64, _I32, _I32, ctypes.POINTER(IceFilterCfg), ctypes.POINTER(IceScheme),
                      _V, _V, _V, _V, _V, _V, _V],
    "ice_autolabel_set_path": [_I32],
    "ice_cut_tiles": [_V, _I32, _I32, _I32, _I32, _V, _V],
    "ice_stitch_tiles": [_V, _I32, _I32, _I32, _I32, _I32, _V, _V],
    "ice_encode_labels": [_V, _I64, _V, _I32, _V, _V, _V],
    "ice_decode_labels": [_V, _I64, _V, _I32, _V, _V, _V],
    "ice_head_argmax": [_V, _I64, _V, _V, _V, _V],
    "ice_confusion": [_V, _V, _I64, _I32, _V, _V, _V],
    "ice_segment": [_V, _I64, _I32, _I32, ctypes.POINTER(IceScheme), _V, _V, _V, _V],
    "ice_rgb_to_hsv": [_V, _I64, _V, _V],
    "ice_conv_fprop": [_V, _I32, _V, _I32, _I32, _I32, _I32, _I32, _V, _V, _I32, _I32, _V, _V, _V, _V],
    "ice_conv_dgrad": [_V, _I32, _I32, _I32, _I32, _I32, _V, _I32, _I32, _V, _V, _V, _V, _V, _V, _V, _V, _I32,
                       _V, _V, _V, _V],
    "ice_halve_fprop": [_V, _I32, _I32, _I32, _I32, _V, _V, _I32, _V, _V],
    "ice_halve_dgrad": [_V, _I32, _I32, _I32, _I32, _V, _I32, _V, _V, _V, _V, _V],
    "ice_halve_wgrad": [_V, _I32, _V, _I32, _I32, _I32, _I32, _V, _V],
    "ice_stem_im2col": [_V, _I32, _I32, _I32, _V, _V],
    "ice_stem_im2col_f32": [_V, _I32, _I32, _I32, _V, _V],
    "ice_pad_weights": [_V, _I32, _I32, _V, _I32, _V],
    "ice_halve_prep": [_V, _I32, _I32, _V, _V],
    "ice_maxpool_fwd": [_V, _I32, _I32, _I32, _I32, _V, _V],
    "ice_maxpool_bwd": [_V, _V, _V, _V, _I32, _I32, _I32, _I32, _V, _V, _V],
    "ice_head_ce": [_V, _I64, _I32, _V, _V, _V, _V, _F32, _V, _V, _V, _V, _V, _V, _V],
    "ice_bias_grad": [_V, _I64, _I32, _V, _V],
    "ice_dropout_scale": [_I32, _F32, ctypes.c_uint64, _V, _V, _V],
    "ice_adam": [_V, _V, _V, _V, _I64, _I64, _V, _F32, _F32, _F32, _F32, _V, _V],
    "ice_counter_add": [_V, _I64, _V],
    "ice_cast_bf16": [_V, _I64, _V, _V],
    "ice_fill_f32": [_V, _I64, _F32, _V],
    "ice_conv_wgrad": [_V, _I32, _V, _I32, _V, _I32, _I32, _I32, _I32, _I32, _V, _V],
}

_lib = None


def load():
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                               f"g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _I32
        _lib = lib
    return _lib


class _Counter:
    """Launch accounting: every ice_* entry point enqueues exactly one kernel.  When
    `events` is a list, each call is bracketed by CUDA events on the current stream
    (bench.py's per-kernel breakdown); otherwise only the count is kept."""
    launches = 0
    events = None


counter = _Counter()


def call(name: str, *args) -> None:
    ev = counter.events
    if ev is not None:
        import torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = getattr(load(), name)(*args)
    if rc != ICE_OK:
        raise NativeError(name, rc)
    counter.launches += 1
    if ev is not None:
        e1.record()
        ev.append((name, args, e0, e1))


def ptr(t) -> int:
    """Device pointer of a torch tensor (must be CUDA and contiguous), or NULL for None."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (the B200 path has no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    load()
