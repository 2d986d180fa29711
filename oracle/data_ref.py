"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the data-path functions around the hot paths.

Checker for the GPU kernels in paper_2403_13135_b200/csrc/data_ops.cu; pinned to the
reference's own outputs by tests/test_data_oracle.py (tests/golden/data_golden.json, made by
tests/golden/make_data_golden.py from /root/reference).
"""
from __future__ import annotations

import numpy as np

CLASS_COLORS = ((255, 0, 0), (0, 0, 255), (0, 255, 0))  # icetrain/data.py:21


def cut_tiles(img, size):  # icetrain/data.py:55-66
    h, w = img.shape[:2]
    out = []
    for row, y in enumerate(range(0, h, size)):
        for col, x in enumerate(range(0, w, size)):
            tile = np.zeros((size, size) + img.shape[2:], img.dtype)
            piece = img[y:y + size, x:x + size]
            tile[:piece.shape[0], :piece.shape[1]] = piece
            out.append((tile, row, col))
    return out


def stitch_tiles(tiles, height, width):  # icetrain/data.py:69-80
    size = tiles[0][0].shape[0]
    rows = 1 + max(r for _, r, _ in tiles)
    cols = 1 + max(c for _, _, c in tiles)
    canvas = np.zeros((rows * size, cols * size) + tiles[0][0].shape[2:], tiles[0][0].dtype)
    for tile, r, c in tiles:
        canvas[r * size:(r + 1) * size, c * size:(c + 1) * size] = tile
    return canvas[:height, :width]


def encode_labels(mask):  # icetrain/data.py:47-52
    return np.asarray(CLASS_COLORS, np.uint8)[mask]


def decode_labels(img):  # icetrain/data.py:35-44 (returns -1 at unknown colours)
    mask = np.full(img.shape[:2], -1, np.int64)
    for idx, color in enumerate(CLASS_COLORS):
        mask[(img == np.asarray(color, np.uint8)).all(axis=-1)] = idx
    return mask


def confusion(pred, ref, n=3):  # icelabel/metrics.py:108-113
    return np.bincount(pred.astype(np.int64).ravel() * n + ref.ravel(), minlength=n * n).reshape(n, n)


def snap_labels(img):  # icelabel/segmentation.py:138-157 with snap=True
    colors = np.asarray(CLASS_COLORS, np.int64)
    flat = img.reshape(-1, 3).astype(np.int64)
    dist = ((flat[:, None, :] - colors[None, :, :]) ** 2).sum(axis=2)
    return dist.argmin(axis=1).reshape(img.shape[:2]).astype(np.uint8)


def ssim(a, b, window=11, sigma=1.5):  # icelabel/metrics.py:145-172
    from scipy.signal import convolve2d
    x = np.arange(window) - (window - 1) / 2
    g = np.exp(-(x ** 2) / (2 * sigma ** 2))
    k = np.outer(g, g)
    k = k / k.sum()
    c1, c2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2
    scores = []
    for ch in range(3):
        p, q = a[:, :, ch].astype(np.float64), b[:, :, ch].astype(np.float64)
        mx, my = convolve2d(p, k, mode="valid"), convolve2d(q, k, mode="valid")
        vx = convolve2d(p * p, k, mode="valid") - mx ** 2
        vy = convolve2d(q * q, k, mode="valid") - my ** 2
        cov = convolve2d(p * q, k, mode="valid") - mx * my
        scores.append(float(np.mean((2 * mx * my + c1) * (2 * cov + c2) / ((mx ** 2 + my ** 2 + c1) * (vx + vy + c2)))))
    return float(np.mean(scores))
