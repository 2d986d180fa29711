"""ctypes binding of the C ABI in include/icelabel_b200.h (libicelabel_b200.so).

There is no CPU fallback: if the library is missing or no CUDA device is present, every
product call raises.  `load()` only needs the file (symbol checks work without a GPU).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ICE_LIB_PATH") or os.path.join(_HERE, "_C", "libicelabel_b200.so")

ICE_OK, ICE_EINVAL, ICE_EWINDOW, ICE_ETOOBIG, ICE_ENODRIVER, ICE_ESCRATCH = 0, -1, -2, -3, -4, -5
_ERRNAMES = {ICE_EINVAL: "ICE_EINVAL", ICE_EWINDOW: "ICE_EWINDOW", ICE_ETOOBIG: "ICE_ETOOBIG",
             ICE_ENODRIVER: "ICE_ENODRIVER", ICE_ESCRATCH: "ICE_ESCRATCH"}


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
_F64 = ctypes.c_double
_U64P = ctypes.POINTER(ctypes.c_uint64)
_S = [_V, _U64P]  # (scratch, scratch_bytes) before the stream: see include/icelabel_b200.h

# name -> argtypes (restype is always int32).  Kept in sync with include/icelabel_b200.h;
# tests/test_native_abi.py checks both directions.
SIGNATURES = {
    "ice_autolabel": [_V, _I64, _I32, _I32, ctypes.POINTER(IceFilterCfg), ctypes.POINTER(IceScheme),
                      _V, _V, _V, _V, _V, _V, _V],
    "ice_autolabel_set_path": [_I32],
    "ice_finish_defer": [_I32],
    "ice_finish_flush": [_V],
    "ice_grad_overwrite": [_I32],
    "ice_conv_reload_knobs": [],
    "ice_autolabel_scene": [_V, _I64, _I32, _I32, ctypes.POINTER(IceFilterCfg), ctypes.POINTER(IceScheme),
                            _V, _V, _V, _V, _V, _V, *_S, _V],
    "ice_cut_tiles": [_V, _I32, _I32, _I32, _I32, _V, _V],
    "ice_stitch_tiles": [_V, _I32, _I32, _I32, _I32, _I32, _V, _V],
    "ice_encode_labels": [_V, _I64, _V, _I32, _V, _V, _V],
    "ice_decode_labels": [_V, _I64, _V, _I32, _V, _V, _V],
    "ice_head_argmax": [_V, _I64, _V, _V, _V, _V],
    "ice_confusion": [_V, _V, _I64, _I32, _V, _V, _V],
    "ice_snap_labels": [_V, _I64, _V, _I32, _V, _V],
    "ice_ssim": [_V, _V, _I32, _I32, _V, ctypes.c_double, ctypes.c_double, _V, *_S, _V],
    "ice_segment": [_V, _I64, _I32, _I32, ctypes.POINTER(IceScheme), _V, _V, _V, _V],
    "ice_rgb_to_hsv": [_V, _I64, _V, _V],
    "ice_conv_fprop": [_V, _I32, _V, _I32, _I32, _I32, _I32, _I32, _V, _V, _I32, _I32, _V, _V, _V, *_S, _V],
    "ice_conv_dgrad": [_V, _I32, _I32, _I32, _I32, _I32, _V, _I32, _I32, _V, _V, _V, _V, _V, _V, _V, _V, _I32,
                       _V, _V, _V, *_S, _V],
    "ice_halve_fprop": [_V, _I32, _I32, _I32, _I32, _V, _V, _I32, _V, *_S, _V],
    "ice_halve_dgrad": [_V, _I32, _I32, _I32, _I32, _V, _I32, _V, _V, _V, _V, _V, *_S, _V],
    "ice_halve_wgrad": [_V, _I32, _V, _I32, _I32, _I32, _I32, _V, *_S, _V],
    "ice_stem_im2col": [_V, _I32, _I32, _I32, _V, _V],
    "ice_stem_fprop": [_V, _I32, _I32, _I32, _V, _V, _V, _V, _V],
    "ice_stem_wgrad": [_V, _I32, _I32, _I32, _V, _V, *_S, _V],
    "ice_stem_im2col_f32": [_V, _I32, _I32, _I32, _V, _V],
    "ice_pad_weights": [_V, _I32, _I32, _V, _I32, _V],
    "ice_halve_prep": [_V, _I32, _I32, _V, _V],
    "ice_maxpool_fwd": [_V, _I32, _I32, _I32, _I32, _V, _V],
    "ice_maxpool_bwd": [_V, _V, _V, _V, _I32, _I32, _I32, _I32, _V, _V, *_S, _V],
    "ice_head_ce": [_V, _I64, _I32, _V, _V, _V, _V, _F32, _V, _V, _V, _V, _V, _V, *_S, _V],
    "ice_bias_grad": [_V, _I64, _I32, _V, *_S, _V],
    "ice_dropout_scale": [_I32, _F32, ctypes.c_uint64, _V, _V, _V],
    "ice_adam": [_V, _V, _V, _V, _I64, _I64, _V, _F64, _F64, _F64, _F64, _I32, _V, _V],
    "ice_counter_add": [_V, _I64, _V],
    "ice_cast_bf16": [_V, _I64, _V, _V],
    "ice_fill_f32": [_V, _I64, _F32, _V],
    "ice_conv_wgrad": [_V, _I32, _V, _I32, _V, _I32, _I32, _I32, _I32, _I32, _V, *_S, _V],
}

# entry points taking caller scratch; `call` supplies it (the call sites pass the other args)
SCRATCH_FNS = frozenset(n for n, a in SIGNATURES.items() if len(a) >= 3 and a[-3:] == [*_S, _V])

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
        lib.ice_kernel_launches.argtypes = []
        lib.ice_kernel_launches.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def kernel_launches() -> int:
    """Kernels the library has launched in this process (counted at every launch site)."""
    return int(load().ice_kernel_launches())


class Scratch:
    """Caller-owned device scratch for the entry points in SCRATCH_FNS (the library never
    allocates): one uint8 buffer per device, shared by calls that are stream-ordered (the
    U-Net issues every scratch-using op on its compute stream; the gradient-bucket side
    stream runs only Adam), grown on an eager call to the largest
    size a call has asked for.  A buffer is never freed once replaced -- CUDA graphs captured
    earlier keep pointing at it -- and growing inside a stream capture is an error (run the
    step eagerly once first, as every warm-up does).  Sizes come from the library's own query
    mode (scratch == NULL), cached per call shape."""

    def __init__(self):
        self.bufs = {}
        self.retired = []
        self.sizes = {}
        self.bump = None  # bump mode: {dev: [chunk, offset, used_this_pass]}

    def begin_bump(self) -> None:
        """Every call until end_bump() gets its OWN slice (deferred finishers read the partial
        sums of earlier calls at flush time, so their scratch must not be reused)."""
        self.bump = {}

    def end_bump(self) -> None:
        """Leave bump mode; if a pass spilled into more than one chunk, the next pass gets a
        single chunk of the whole pass's size (steady state: one chunk, nothing allocated)."""
        import torch
        for dev, (chunk, _, used) in (self.bump or {}).items():
            base = self.bufs[("bump", dev)]
            if (chunk is not base or used > base.numel()) and not torch.cuda.is_current_stream_capturing():
                self.retired.append(base)
                self.bufs[("bump", dev)] = torch.empty(used, dtype=torch.uint8, device=dev)
        self.bump = None

    def _bump_get(self, nbytes: int):
        import torch
        dev = torch.cuda.current_device()
        st = self.bump.get(dev)
        if st is None:
            chunk = self.bufs.get(("bump", dev))
            if chunk is None:
                chunk = self.bufs[("bump", dev)] = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
            st = self.bump[dev] = [chunk, 0, 0]
        off = (st[1] + 255) & ~255
        if off + nbytes > st[0].numel():  # spill: a new chunk; earlier slices stay valid
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("bump scratch must grow inside a CUDA-graph capture: run the same "
                                   "step eagerly before capturing")
            self.retired.append(st[0])
            st[0] = torch.empty(max(nbytes, 2 * st[0].numel()), dtype=torch.uint8, device=dev)
            off = 0
        st[1] = off + nbytes
        st[2] += nbytes + 256
        return st[0][off:off + nbytes]

    def need(self, fn, name, core) -> int:
        key = (name,) + tuple(bool(a) if t is _V else (a if t in (_I32, _I64) else None)
                              for a, t in zip(core, SIGNATURES[name]))
        n = self.sizes.get(key)
        if n is None:
            q = ctypes.c_uint64(0)
            rc = fn(*core, None, ctypes.byref(q), None)
            if rc != ICE_OK:
                raise NativeError(name, rc)
            n = self.sizes[key] = int(q.value)
        return n

    def get(self, stream_handle, nbytes: int):
        import torch
        if self.bump is not None:
            return self._bump_get(nbytes)
        dev = torch.cuda.current_device()
        key = dev
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError(f"scratch must grow to {nbytes} B inside a CUDA-graph capture: "
                                   "run the same step eagerly before capturing")
            if buf is not None:
                self.retired.append(buf)
            size = max(nbytes, 2 * (buf.numel() if buf is not None else 0), 1 << 20)
            buf = torch.empty(size, dtype=torch.uint8, device=dev)
            self.bufs[key] = buf
        return buf


scratch = Scratch()


class _Counter:
    """Call accounting: `launches` counts ice_* entry-point calls (each enqueues one kernel,
    plus a fixed-order finishing kernel where it reduces partial sums; kernel_launches() is
    the library's own kernel count).  When `events` is a list, each call is bracketed by CUDA
    events on the current stream (bench.py's per-entry-point breakdown)."""
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
    fn = getattr(load(), name)
    if name in SCRATCH_FNS:
        core, stream = args[:-1], args[-1]
        need = scratch.need(fn, name, core)
        if need:
            buf = scratch.get(stream, need)
            cap = ctypes.c_uint64(buf.numel())
            rc = fn(*core, buf.data_ptr(), ctypes.byref(cap), stream)
        else:
            rc = fn(*core, None, None, stream)
    else:
        rc = fn(*args)
    if name in ("ice_autolabel_set_path", "ice_conv_reload_knobs"):
        scratch.sizes.clear()  # scratch needs depend on the path / the tiling switches
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
