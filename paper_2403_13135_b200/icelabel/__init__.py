"""B200-native drop-in for the reference auto-labeler hot path (icelabel.process_tile)."""
from .types import (CLASS_COLORS, MASK_FIXED, MASK_OTSU, ROSS_SEA_SUMMER, ClassId, ColorRange,
                    FilterConfig, FilterOutput, LabelMask, SceneRaster, SegmentationScheme, Tile,
                    TileResult, get_preset)
from .ops import (apply_filter, autolabel, autolabel_sharded, check_windows, detect_mask, process_tile,
                  process_tiles, segment, segment_batch, shard_bounds)
from .labels import parse_labels, parse_labels_device, render_labels, render_labels_device
from .tiling import TileGrid, split_scene, split_scene_device, stitch_scene, stitch_scene_device

__all__ = ["CLASS_COLORS", "MASK_FIXED", "MASK_OTSU", "ROSS_SEA_SUMMER", "ClassId", "ColorRange",
           "FilterConfig", "FilterOutput", "LabelMask", "SceneRaster", "SegmentationScheme", "Tile",
           "TileResult", "get_preset", "apply_filter", "autolabel", "autolabel_sharded", "check_windows",
           "detect_mask", "process_tile", "process_tiles", "segment", "segment_batch", "shard_bounds",
           "parse_labels", "parse_labels_device", "render_labels", "render_labels_device", "TileGrid", "split_scene",
           "split_scene_device", "stitch_scene", "stitch_scene_device"]
