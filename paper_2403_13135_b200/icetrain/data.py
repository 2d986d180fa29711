"""File interface of the trainer (reference icetrain/data.py), with the byte work on the GPU.

Same functions, signatures and errors as the reference:
  * read_png / write_png (PIL; host file IO, data.py:24-32),
  * decode_labels / encode_labels: the label colour codec (data.py:35-52) -> ice_decode_labels /
    ice_encode_labels,
  * cut_tiles / stitch_tiles (data.py:55-80) -> ice_cut_tiles / ice_stitch_tiles,
  * scene_stems / load_pairs / load_run (data.py:83-122),
  * train_val_split (data.py:125-136).
`*_device` variants keep tiles and masks resident in HBM for the GPU pipeline (a run's
labels can go from K1 straight into training without a PNG round trip).  There is no CPU
fallback: the codec and cut/stitch calls need the CUDA library.
"""
from __future__ import annotations

import json
import os

import numpy as np

from .. import _native

CLASS_COLORS = ((255, 0, 0), (0, 0, 255), (0, 255, 0))
_NO_BAD = (1 << 64) - 1


def read_png(path: str) -> np.ndarray:
    from PIL import Image
    with Image.open(path) as img:
        return np.asarray(img.convert("RGB"), dtype=np.uint8)


def write_png(path: str, data: np.ndarray) -> None:
    from PIL import Image
    if data.dtype != np.uint8:
        raise ValueError(f"expected uint8 image data, got {data.dtype}")
    Image.fromarray(data, "RGB").save(path, "PNG")


def _dev(a):
    import torch
    _native.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.cuda().contiguous()
    host = torch.from_numpy(np.ascontiguousarray(a))
    return host.pin_memory().to("cuda", non_blocking=True)


def _colors_dev():
    import torch
    return torch.tensor(CLASS_COLORS, dtype=torch.uint8, device="cuda")


def _bad_flag():
    import torch
    return torch.full((1,), -1, dtype=torch.int64, device="cuda")  # all ones = UINT64_MAX


def decode_labels_device(img_dev):
    """u8 [h, w, 3] device colour image -> (u8 [h, w] class mask, first unknown index or -1)."""
    import torch
    h, w = img_dev.shape[:2]
    mask = torch.empty((h, w), dtype=torch.uint8, device=img_dev.device)
    bad = _bad_flag()
    _native.call("ice_decode_labels", img_dev.data_ptr(), h * w, _colors_dev().data_ptr(), len(CLASS_COLORS),
                 mask.data_ptr(), bad.data_ptr(), _native.stream_handle())
    first = int(bad.item())
    return mask, (-1 if first == -1 else first)


def decode_labels(img: np.ndarray, path: str = "") -> np.ndarray:
    """Color image -> int64 class-index mask. Unknown colors are loud (data.py:35-44)."""
    img = np.asarray(img)
    mask, first = decode_labels_device(_dev(img.astype(np.uint8, copy=False)))
    if first >= 0:
        y, x = divmod(first, img.shape[1])
        raise ValueError(f"{path or 'label image'}: unknown label color "
                         f"{tuple(int(v) for v in img[y, x])} at row {y}, col {x}")
    return mask.cpu().numpy().astype(np.int64)


def encode_labels_device(mask_dev):
    """u8 [..] device class mask -> (u8 [.., 3] colour image, first out-of-range index or -1)."""
    import torch
    rgb = torch.empty(tuple(mask_dev.shape) + (3,), dtype=torch.uint8, device=mask_dev.device)
    bad = _bad_flag()
    _native.call("ice_encode_labels", mask_dev.data_ptr(), mask_dev.numel(), _colors_dev().data_ptr(),
                 len(CLASS_COLORS), rgb.data_ptr(), bad.data_ptr(), _native.stream_handle())
    first = int(bad.item())
    return rgb, (-1 if first == -1 else first)


def encode_labels(mask: np.ndarray) -> np.ndarray:
    """Class-index mask -> color image, inverse of decode_labels (data.py:47-52)."""
    mask = np.asarray(mask)
    if mask.size and (mask.min() < 0 or mask.max() >= len(CLASS_COLORS)):
        raise ValueError(f"class index out of range: {int(mask.min())}..{int(mask.max())}")
    rgb, _ = encode_labels_device(_dev(mask.astype(np.uint8)))
    return rgb.cpu().numpy()


def cut_tiles_device(img_dev, size: int):
    """u8 [h, w(, c)] device image -> u8 [rows*cols, size, size(, c)] tiles (zero padded)."""
    import torch
    h, w = img_dev.shape[:2]
    c = img_dev.shape[2] if img_dev.ndim == 3 else 1
    rows, cols = -(-h // size), -(-w // size)
    shape = (rows * cols, size, size) + ((c,) if img_dev.ndim == 3 else ())
    tiles = torch.empty(shape, dtype=torch.uint8, device=img_dev.device)
    _native.call("ice_cut_tiles", img_dev.data_ptr(), h, w, c, size, tiles.data_ptr(), _native.stream_handle())
    return tiles, rows, cols


def stitch_tiles_device(tiles_dev, height: int, width: int, cols: int = 0):
    import torch
    size = tiles_dev.shape[1]
    c = tiles_dev.shape[3] if tiles_dev.ndim == 4 else 1
    out = torch.empty((height, width) + ((c,) if tiles_dev.ndim == 4 else ()), dtype=torch.uint8,
                      device=tiles_dev.device)
    _native.call("ice_stitch_tiles", tiles_dev.contiguous().data_ptr(), cols, size, c, height, width,
                 out.data_ptr(), _native.stream_handle())
    return out


def _check_byte_range(a: np.ndarray, who: str) -> None:
    """The GPU cut/stitch kernels move bytes: integer data in 0..255 round-trips exactly through
    them; anything else (float probabilities, wide integers) would be silently truncated, so it
    is refused instead (the reference keeps any dtype; labels and RGB tiles are all it cuts)."""
    if not (np.issubdtype(a.dtype, np.integer) or a.dtype == np.bool_):
        raise TypeError(f"{who}: integer data in 0..255 expected, got {a.dtype}")
    if a.size and (a.min() < 0 or a.max() > 255):
        raise ValueError(f"{who}: values outside 0..255")


def cut_tiles(img: np.ndarray, size: int) -> list:
    """(tile, row, col) squares covering the image, zero-padded at the ragged edges; works
    for (h, w, 3) images and (h, w) masks (data.py:55-66)."""
    img = np.asarray(img)
    if img.dtype != np.uint8:  # int64 class masks: values 0..2 travel as bytes
        _check_byte_range(img, "cut_tiles")
        tiles, rows, cols = cut_tiles_device(_dev(img.astype(np.uint8)), size)
        host = tiles.cpu().numpy().astype(img.dtype)
    else:
        tiles, rows, cols = cut_tiles_device(_dev(img), size)
        host = tiles.cpu().numpy()
    return [(host[t], t // cols, t % cols) for t in range(rows * cols)]


def stitch_tiles(tiles: list, height: int, width: int) -> np.ndarray:
    """Inverse of cut_tiles for (tile, row, col) lists; crops the padding (data.py:69-80)."""
    import torch
    if not tiles:
        raise ValueError("no tiles to stitch")
    size = tiles[0][0].shape[0]
    rows = 1 + max(r for _, r, _ in tiles)
    cols = 1 + max(c for _, _, c in tiles)
    dtype = tiles[0][0].dtype
    grid = np.zeros((rows * cols,) + tiles[0][0].shape, np.uint8)
    for tile, r, c in tiles:
        if dtype != np.uint8:
            _check_byte_range(np.asarray(tile), "stitch_tiles")
        grid[r * cols + c] = tile
    height, width = min(height, rows * size), min(width, cols * size)  # canvas[:height, :width]
    out = stitch_tiles_device(_dev(grid), height, width, cols)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(dtype)


def scene_stems(directory: str) -> list:
    return sorted(os.path.splitext(n)[0] for n in os.listdir(directory) if n.lower().endswith(".png"))


def load_pairs(images_dir: str, labels_dir: str, tile_size: int) -> list:
    """(image tile, class mask tile) pairs cut from every scene, paired by file stem
    (data.py:88-107).  PNG decode on the host; colour decode and cutting on the GPU."""
    pairs = []
    for stem in scene_stems(images_dir):
        image_path = os.path.join(images_dir, f"{stem}.png")
        label_path = os.path.join(labels_dir, f"{stem}.png")
        if not os.path.isfile(label_path):
            raise ValueError(f"no label image for scene {stem!r}: {label_path}")
        image = read_png(image_path)
        label_img = read_png(label_path)
        mask_dev, first = decode_labels_device(_dev(label_img))
        if first >= 0:
            y, x = divmod(first, label_img.shape[1])
            raise ValueError(f"{label_path}: unknown label color "
                             f"{tuple(int(v) for v in label_img[y, x])} at row {y}, col {x}")
        if image.shape[:2] != tuple(mask_dev.shape):
            raise ValueError(f"{stem}: image {image.shape[:2]} and label {tuple(mask_dev.shape)} sizes differ")
        itiles, rows, cols = cut_tiles_device(_dev(image), tile_size)
        mtiles, _, _ = cut_tiles_device(mask_dev, tile_size)
        ih, mh = itiles.cpu().numpy(), mtiles.cpu().numpy().astype(np.int64)
        pairs.extend((ih[t], mh[t]) for t in range(rows * cols))
    if not pairs:
        raise ValueError(f"no scenes under {images_dir}")
    return pairs


def load_run(run_dir: str, tile_size: int) -> list:
    """Pairs from a pipeline run directory, located via its manifest (data.py:110-122)."""
    manifest_path = os.path.join(run_dir, "manifest.json")
    outputs = {}
    if os.path.isfile(manifest_path):
        with open(manifest_path, "r", encoding="utf-8") as fh:
            outputs = json.load(fh).get("outputs", {})
    images_dir = os.path.join(run_dir, outputs.get("filtered", "filtered"))
    labels_dir = os.path.join(run_dir, outputs.get("labels", "labels"))
    for d in (images_dir, labels_dir):
        if not os.path.isdir(d):
            raise ValueError(f"run directory is missing {d}")
    return load_pairs(images_dir, labels_dir, tile_size)


def train_val_split(pairs: list, val_fraction: float, seed: int) -> tuple:
    """data.py:125-136: seeded permutation; validation = the first round(n * f) indices
    (never the whole corpus), training keeps the original order."""
    if not 0.0 <= val_fraction < 1.0:
        raise ValueError(f"val_fraction out of range: {val_fraction}")
    order = np.random.default_rng(seed).permutation(len(pairs))
    n_val = min(int(round(len(pairs) * val_fraction)), len(pairs) - 1)
    val_idx = set(order[:n_val].tolist())
    train = [pairs[i] for i in range(len(pairs)) if i not in val_idx]
    val = [pairs[i] for i in sorted(val_idx)]
    return train, val
