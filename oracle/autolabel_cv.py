"""TEST INFRASTRUCTURE / CPU BASELINE ONLY -- never imported by the product path.

A second CPU restatement of the reference labeler (engine.process_tile,
/root/reference/pkg/src/icelabel/engine.py:145-160) built on the same third-party calls
the reference makes -- OpenCV's medianBlur / dilate and NumPy float64 vector math -- so
that it runs at the reference's own CPU speed.  `bench.py` times it as the auto-label CPU
baseline (kind "port"); the exact-integer C restatement in oracle/autolabel_ref.c stays
the parity checker.  tests/test_oracle_golden.py pins this module to the reference's
golden digests too.

Third-party dependency: opencv-python-headless (reference pyproject: >=4.8; 4.13 here).
"""
from __future__ import annotations

import numpy as np

try:  # cv2 is part of the image; only the CPU baseline / its tests need it
    import cv2
except ImportError:  # pragma: no cover
    cv2 = None

ROSS_SEA_SUMMER = ((0, (0, 0, 205), (179, 255, 255)),
                   (1, (0, 0, 31), (179, 255, 204)),
                   (2, (0, 0, 0), (179, 255, 30)))


def _median_blur(img, k):  # kernels.py:42-46
    return cv2.medianBlur(img, k)


def _dilate(img, k):  # kernels.py:49-54
    return cv2.dilate(img, np.ones((k, k), np.uint8), borderType=cv2.BORDER_REPLICATE)


def _background(c, dil_k, med_k):  # cloudfilter.py:82-84
    return _median_blur(_dilate(c, dil_k), med_k)


def _minmax(img):  # kernels.py:66-74
    lo, hi = int(img.min()), int(img.max())
    if hi == lo:
        return np.zeros_like(img)
    return np.floor(255.0 * (img.astype(np.float64) - lo) / (hi - lo) + 0.5).astype(np.uint8)


def _otsu(img):  # kernels.py:77-110, exact integer comparison
    counts = [int(x) for x in np.bincount(img.ravel(), minlength=256)]
    n_total, s_total = sum(counts), sum(i * c for i, c in enumerate(counts))
    best_t, best_num, best_den, n0, s0 = 0, 0, 1, 0, 0
    for t in range(256):
        n0 += counts[t]
        s0 += t * counts[t]
        n1 = n_total - n0
        if n0 == 0 or n1 == 0:
            continue
        num = (s0 * n1 - (s_total - s0) * n0) ** 2
        den = n0 * n1
        if num * best_den > best_num * den:
            best_t, best_num, best_den = t, num, den
    return best_t


def apply_filter(rgb, dil_k=7, med_k=21, noise_k=3, fixed_t=None, truncate_t=None):
    """(filtered, mask, affected count) -- cloudfilter.py:87-117."""
    gray = rgb.max(axis=2)
    d = np.abs(_median_blur(gray, noise_k).astype(np.int16) -
               _background(gray, dil_k, med_k).astype(np.int16)).astype(np.uint8)
    if truncate_t is not None:
        d = np.minimum(d, np.uint8(truncate_t))
    d_n = _minmax(d)
    t = _otsu(d_n) if fixed_t is None else fixed_t
    affected = d_n > t
    out = rgb.copy()
    if affected.any():
        for ch in range(3):
            c = rgb[:, :, ch]
            bg = _background(c, dil_k, med_k).astype(np.int32)
            center = int(np.floor(float(np.median(c)) + 0.5))
            fixed = np.clip(c.astype(np.int32) - bg + center, 0, 255).astype(np.uint8)
            out[:, :, ch] = np.where(affected, fixed, c)
    return out, np.where(affected, np.uint8(255), np.uint8(0)), int(affected.sum())


def segment(rgb, ranges=ROSS_SEA_SUMMER):
    """(label with 255 where unmatched, first unmatched row-major index or -1) --
    segmentation.py:118-128 over raster.py:187-216 (float64, as the reference)."""
    f = rgb.astype(np.float64)
    r, g, b = f[..., 0], f[..., 1], f[..., 2]
    v = f.max(axis=-1)
    c = v - f.min(axis=-1)
    s = np.zeros_like(v)
    nz = v > 0
    s[nz] = np.floor(255.0 * c[nz] / v[nz] + 0.5)
    safe = np.where(c > 0, c, 1.0)
    hdeg = np.select([v == r, v == g], [np.mod(60.0 * (g - b) / safe, 360.0), 60.0 * (b - r) / safe + 120.0],
                     default=60.0 * (r - g) / safe + 240.0)
    half = np.floor(hdeg / 2.0 + 0.5)
    half[half == 180.0] = 0.0
    h = np.where(c > 0, half, 0.0)
    hsv = np.stack([h, s, v], axis=-1).astype(np.uint8)
    ordered = sorted(ranges, key=lambda x: x[0])
    conds = [np.logical_and(hsv >= np.asarray(lo, np.uint8), hsv <= np.asarray((min(hi[0], 179),) + tuple(hi[1:]),
                                                                                np.uint8)).all(axis=-1)
             for _, lo, hi in ordered]
    label = np.select(conds, [cls for cls, _, _ in ordered], default=255).astype(np.uint8)
    bad = np.flatnonzero(label == 255)
    return label, int(bad[0]) if bad.size else -1


def process_tile(rgb):
    """engine.process_tile with the default FilterConfig and the ross-sea-summer scheme."""
    f, _, a = apply_filter(rgb)
    lbl, first = segment(f)
    return f, lbl, a, first
