"""ctypes front end of the C auto-label oracle (oracle/autolabel_ref.c).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and bench.py's
CPU legs.  Restates `process_tile` (/root/reference/pkg/src/icelabel/engine.py:145-160)
and its callees; see the C file for per-function citations.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_autolabel.so")
_lib = None

ERR_WINDOW = {1: "noise_median_k", 2: "bg_dilate_k", 3: "bg_median_k"}
ERR_UNMATCHED = 4


class FilterCfg(ctypes.Structure):
    _fields_ = [("bg_dilate_k", ctypes.c_int), ("bg_median_k", ctypes.c_int),
                ("noise_median_k", ctypes.c_int), ("mask_mode_fixed", ctypes.c_int),
                ("fixed_t", ctypes.c_int), ("diff_truncate", ctypes.c_int),
                ("truncate_t", ctypes.c_int)]


class Scheme(ctypes.Structure):
    _fields_ = [("lo", (ctypes.c_uint8 * 3) * 3), ("hi", (ctypes.c_uint8 * 3) * 3),
                ("cls", ctypes.c_uint8 * 3)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.or_median_blur.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        L.or_dilate.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        L.or_minmax_normalize.argtypes = [u8p, ctypes.c_size_t, u8p]
        L.or_otsu_threshold.argtypes = [u8p, ctypes.c_size_t]
        L.or_otsu_threshold.restype = ctypes.c_int
        L.or_rgb_to_hsv.argtypes = [u8p, ctypes.c_size_t, u8p]
        L.or_segment.argtypes = [u8p, ctypes.c_size_t, ctypes.POINTER(Scheme), u8p]
        L.or_segment.restype = ctypes.c_long
        L.or_apply_filter.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(FilterCfg),
                                      u8p, u8p, ctypes.POINTER(ctypes.c_long)]
        L.or_process_tile.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(FilterCfg),
                                      ctypes.POINTER(Scheme), u8p, u8p,
                                      ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def make_cfg(bg_dilate_k=7, bg_median_k=21, noise_median_k=3, mask_mode="otsu",
             fixed_t=128, diff_truncate=False, truncate_t=16) -> FilterCfg:
    return FilterCfg(bg_dilate_k, bg_median_k, noise_median_k, int(mask_mode == "fixed"),
                     fixed_t, int(diff_truncate), truncate_t)


def make_scheme(ranges) -> Scheme:
    """ranges: iterable of (class_id, (h,s,v) lower, (h,s,v) upper); sorted by class id
    and hue-clamped to 179 like ColorRange/SegmentationScheme (segmentation.py:30-69)."""
    sc = Scheme()
    for k, (cls, lo, hi) in enumerate(sorted(ranges, key=lambda r: r[0])):
        lo = (min(lo[0], 179), lo[1], lo[2])
        hi = (min(hi[0], 179), hi[1], hi[2])
        for ch in range(3):
            sc.lo[k][ch] = lo[ch]
            sc.hi[k][ch] = hi[ch]
        sc.cls[k] = cls
    return sc


ROSS_SEA_SUMMER = ((0, (0, 0, 205), (179, 255, 255)),
                   (1, (0, 0, 31), (179, 255, 204)),
                   (2, (0, 0, 0), (179, 255, 30)))


def median_blur(img: np.ndarray, k: int) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(img)
    lib().or_median_blur(_p(img), img.shape[0], img.shape[1], k, _p(out))
    return out


def dilate(img: np.ndarray, k: int) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(img)
    lib().or_dilate(_p(img), img.shape[0], img.shape[1], k, _p(out))
    return out


def minmax_normalize(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(img)
    lib().or_minmax_normalize(_p(img), img.size, _p(out))
    return out


def otsu_threshold(img: np.ndarray) -> int:
    img = np.ascontiguousarray(img, np.uint8)
    return lib().or_otsu_threshold(_p(img), img.size)


def rgb_to_hsv(rgb: np.ndarray) -> np.ndarray:
    rgb = np.ascontiguousarray(rgb, np.uint8)
    out = np.empty_like(rgb)
    lib().or_rgb_to_hsv(_p(rgb), rgb.size // 3, _p(out))
    return out


def segment(rgb: np.ndarray, ranges=ROSS_SEA_SUMMER):
    """(label u8 HxW with 255 at unmatched pixels, first unmatched index or -1)"""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    label = np.empty(rgb.shape[:2], np.uint8)
    sc = make_scheme(ranges)
    first = lib().or_segment(_p(rgb), rgb.size // 3, ctypes.byref(sc), _p(label))
    return label, int(first)


def apply_filter(rgb: np.ndarray, cfg: FilterCfg | None = None):
    """(filtered, mask, affected_count) or raises ValueError with the reference text."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    cfg = cfg or make_cfg()
    h, w = rgb.shape[:2]
    filtered = np.empty_like(rgb)
    mask = np.empty((h, w), np.uint8)
    aff = ctypes.c_long(0)
    rc = lib().or_apply_filter(_p(rgb), h, w, ctypes.byref(cfg), _p(filtered), _p(mask),
                               ctypes.byref(aff))
    if rc:
        raise ValueError(f"window {getattr(cfg, ERR_WINDOW[rc])} exceeds image extent {(h, w)}")
    return filtered, mask, int(aff.value)


def process_tile(rgb: np.ndarray, cfg: FilterCfg | None = None, ranges=ROSS_SEA_SUMMER,
                 scheme_name: str = "ross-sea-summer"):
    """dict(label, filtered, affected_fraction, error) like TileResult (engine.py:118-160)."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    cfg = cfg or make_cfg()
    h, w = rgb.shape[:2]
    filtered = np.empty_like(rgb)
    label = np.empty((h, w), np.uint8)
    aff = ctypes.c_long(0)
    un = ctypes.c_long(-1)
    sc = make_scheme(ranges)
    rc = lib().or_process_tile(_p(rgb), h, w, ctypes.byref(cfg), ctypes.byref(sc),
                               _p(filtered), _p(label), ctypes.byref(aff), ctypes.byref(un))
    if rc in ERR_WINDOW:
        return dict(label=None, filtered=None, affected_fraction=0.0,
                    error=f"ValueError: window {getattr(cfg, ERR_WINDOW[rc])} "
                          f"exceeds image extent {(h, w)}")
    if rc == ERR_UNMATCHED:
        y, x = divmod(int(un.value), w)
        return dict(label=None, filtered=None, affected_fraction=0.0,
                    error=f"ValueError: scheme {scheme_name!r} matches no class at "
                          f"row={y}, col={x}")
    return dict(label=label, filtered=filtered, affected_fraction=aff.value / (h * w),
                error="")
