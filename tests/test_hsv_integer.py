"""The integer HSV restatement the kernels use equals the float64 reference on all 2^24 RGB.

SURVEY.md Appendix C; reference raster.py:187-216 restated in oracle/autolabel_ref.c.
"""
import numpy as np

from oracle import autolabel as orc


def integer_hsv(rgb):
    r, g, b = (rgb[..., i].astype(np.int64) for i in range(3))
    v = np.maximum(np.maximum(r, g), b)
    mn = np.minimum(np.minimum(r, g), b)
    c = v - mn
    s = np.where(v == 0, 0, (510 * c + v) // np.maximum(2 * v, 1))
    num = np.where(v == r, 60 * (g - b) + np.where(g < b, 360 * c, 0),
                   np.where(v == g, 60 * (b - r) + 120 * c, 60 * (r - g) + 240 * c))
    h = np.where(c > 0, (num + c) // np.maximum(2 * c, 1), 0)
    h = np.where(h == 180, 0, h)
    return np.stack([h, s, v], -1).astype(np.uint8)


def test_integer_hsv_exhaustive():
    allrgb = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(allrgb >> 16) & 255, (allrgb >> 8) & 255, allrgb & 255], -1).astype(np.uint8)
    rgb = rgb.reshape(4096, 4096, 3)
    want = orc.rgb_to_hsv(rgb)
    for lo in range(0, 4096, 512):
        assert np.array_equal(integer_hsv(rgb[lo:lo + 512]), want[lo:lo + 512])


def test_integer_minmax_exhaustive():
    # kernels.py:66-74 float64 stretch == (510 (x - lo) + (hi - lo)) // (2 (hi - lo))
    lo, hi, x = np.meshgrid(np.arange(256), np.arange(256), np.arange(256), indexing="ij")
    ok = (lo < hi) & (x >= lo) & (x <= hi)
    lo, hi, x = lo[ok], hi[ok], x[ok]
    ref = np.floor(255.0 * (x.astype(np.float64) - lo) / (hi - lo) + 0.5)
    assert np.array_equal(ref.astype(np.int64), (510 * (x - lo) + (hi - lo)) // (2 * (hi - lo)))
