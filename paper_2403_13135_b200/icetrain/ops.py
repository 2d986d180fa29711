"""Thin torch-tensor wrappers over the U-Net entry points of libicelabel_b200.so.

Activations are NHWC bf16 CUDA tensors, conv weights KRSC bf16 ([cout, k, k, cin]),
gradients of weights fp32.  Each wrapper checks shapes/dtypes, then calls the C ABI on
the current torch stream.  No CPU fallback exists.
"""

from __future__ import annotations

import torch

from .. import _native

BF16 = torch.bfloat16


def _c(t, dtype=None, what="tensor"):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{what}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous tensor")
    return t.data_ptr()


def conv_fprop(x1, wgt, bias=None, x2=None, relu=True, drop=None, ksize=3, out=None, relu_bits=None, stream=None):
    n, h, w, c1 = x1.shape
    c2 = 0 if x2 is None else x2.shape[3]
    cout = wgt.shape[0]
    if tuple(wgt.shape) != (cout, ksize, ksize, c1 + c2):
        raise ValueError(f"weight shape {tuple(wgt.shape)} != {(cout, ksize, ksize, c1 + c2)}")
    if out is None:
        out = torch.empty((n, h, w, cout), dtype=BF16, device=x1.device)
    _native.call("ice_conv_fprop", _c(x1, BF16, "x1"), c1, _c(x2, BF16, "x2"), c2, n, h, w, ksize,
                 _c(wgt, BF16, "wgt"), _c(bias, torch.float32, "bias"), cout, int(relu),
                 _c(drop, torch.float32, "drop"), _c(out, BF16, "out"), _c(relu_bits, torch.int32, "relu_bits"),
                 _native.stream_handle(stream))
    return out


def conv_dgrad(dy, wgt, c1, c2=0, ksize=3, out1=None, out2=None, ref1=None, ref2=None, drop1=None,
               drop2=None, add1=None, add2=None, want2=True, planes2=False, db1=None, db2=None,
               bits1=None, stream=None):
    n, h, w, cout = dy.shape
    if tuple(wgt.shape) != (cout, ksize, ksize, c1 + c2):
        raise ValueError(f"weight shape {tuple(wgt.shape)} != {(cout, ksize, ksize, c1 + c2)}")
    if out1 is None:
        out1 = torch.empty((n, h, w, c1), dtype=BF16, device=dy.device)
    if c2 and want2 and out2 is None:
        out2 = torch.empty((n, h, w, c2), dtype=BF16, device=dy.device)
    _native.call("ice_conv_dgrad", _c(dy, BF16, "dy"), cout, n, h, w, ksize, _c(wgt, BF16, "wgt"), c1, c2,
                 _c(out1, BF16), _c(ref1, BF16), _c(drop1, torch.float32), _c(add1, BF16),
                 _c(out2, BF16), _c(ref2, BF16), _c(drop2, torch.float32), _c(add2, BF16), int(planes2),
                 _c(db1, torch.float32), _c(db2, torch.float32), _c(bits1, torch.int32, "bits1"),
                 _native.stream_handle(stream))
    return out1, out2


def conv_wgrad(x1, dy, dw, x2=None, ksize=3, stream=None):
    n, h, w, c1 = x1.shape
    c2 = 0 if x2 is None else x2.shape[3]
    cout = dy.shape[3]
    if tuple(dw.shape) != (cout, ksize, ksize, c1 + c2) or dw.dtype != torch.float32:
        raise ValueError(f"dw must be fp32 {(cout, ksize, ksize, c1 + c2)}")
    _native.call("ice_conv_wgrad", _c(x1, BF16, "x1"), c1, _c(x2, BF16, "x2"), c2, _c(dy, BF16, "dy"), cout,
                 n, h, w, ksize, _c(dw, torch.float32, "dw"), _native.stream_handle(stream))
    return dw
