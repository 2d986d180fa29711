"""Label-mask colour rendering / parsing on the GPU (reference icelabel/segmentation.py:131-157).

render_labels paints class ids with the class colormap (ice_encode_labels); parse_labels
inverts it exactly (ice_decode_labels; an off-colormap pixel raises with the reference's
message naming its coordinates) or, with snap=True, takes the nearest colormap colour
(ice_snap_labels: squared RGB distance, ties to the earlier class).
"""
from __future__ import annotations

import numpy as np

from .. import _native
from .types import CLASS_COLORS, ClassId, LabelMask, SceneRaster

_COLORS = np.array([CLASS_COLORS[c] for c in ClassId], np.uint8)
_colors_dev_cache = {}


def _colors_dev():
    import torch
    dev = torch.cuda.current_device()
    if dev not in _colors_dev_cache:
        _colors_dev_cache[dev] = torch.from_numpy(_COLORS.copy()).cuda()
    return _colors_dev_cache[dev]


def render_labels_device(mask_dev):
    """u8 [..] device class ids (< 3) -> u8 [.., 3] device colour image."""
    import torch
    rgb = torch.empty(tuple(mask_dev.shape) + (3,), dtype=torch.uint8, device=mask_dev.device)
    bad = torch.full((1,), -1, dtype=torch.int64, device=mask_dev.device)
    _native.call("ice_encode_labels", _native.ptr(mask_dev.contiguous()), mask_dev.numel(), _colors_dev().data_ptr(),
                 len(_COLORS), rgb.data_ptr(), bad.data_ptr(), _native.stream_handle())
    return rgb


def parse_labels_device(rgb_dev, snap: bool = False):
    """u8 [h, w, 3] device colour image -> (u8 [h, w] class ids, first off-colormap pixel index
    or -1; always -1 with snap)."""
    import torch
    h, w = rgb_dev.shape[:2]
    mask = torch.empty((h, w), dtype=torch.uint8, device=rgb_dev.device)
    src = _native.ptr(rgb_dev.contiguous())
    if snap:
        _native.call("ice_snap_labels", src, h * w, _colors_dev().data_ptr(), len(_COLORS), mask.data_ptr(),
                     _native.stream_handle())
        return mask, -1
    bad = torch.full((1,), -1, dtype=torch.int64, device=rgb_dev.device)
    _native.call("ice_decode_labels", src, h * w, _colors_dev().data_ptr(), len(_COLORS), mask.data_ptr(),
                 bad.data_ptr(), _native.stream_handle())
    first = int(bad.item())
    return mask, first


def render_labels(mask: LabelMask) -> SceneRaster:
    """segmentation.py:131-135."""
    import torch
    return SceneRaster(render_labels_device(torch.from_numpy(np.ascontiguousarray(mask.data)).cuda()).cpu().numpy())


def parse_labels(raster: SceneRaster, snap: bool = False) -> LabelMask:
    """segmentation.py:138-157."""
    import torch
    mask, first = parse_labels_device(torch.from_numpy(np.ascontiguousarray(raster.data)).cuda(), snap)
    if first >= 0:
        y, x = divmod(first, raster.width)
        r, g, b = (int(v) for v in raster.data[y, x])
        raise ValueError(f"pixel at row={y}, col={x} is ({r}, {g}, {b}), not a colormap color")
    return LabelMask(mask.cpu().numpy())
