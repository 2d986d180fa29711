"""Scene tiling on the GPU (reference icelabel/tiling.py:33-103).

`split_scene` / `stitch_scene` keep the reference signatures and error messages; the byte
moves run in ice_cut_tiles / ice_stitch_tiles (csrc/data_ops.cu).  The `_device` variants keep
scenes and tiles resident in HBM, so a scene can go split -> K1 auto-label -> U-Net training
(icetrain.train_device) without a host round trip.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .. import _native
from .types import SceneRaster, Tile


@dataclass(frozen=True)
class TileGrid:
    """tiling.py:33-63: the scene extent and tile size; rows / cols derived."""
    scene_id: str
    scene_width: int
    scene_height: int
    tile_size: int = 256
    rows: int = field(init=False)
    cols: int = field(init=False)

    def __post_init__(self) -> None:
        if self.tile_size < 1:
            raise ValueError(f"tile_size must be >= 1, got {self.tile_size}")
        if self.scene_width < 1 or self.scene_height < 1:
            raise ValueError("scene extent must be positive")
        object.__setattr__(self, "rows", math.ceil(self.scene_height / self.tile_size))
        object.__setattr__(self, "cols", math.ceil(self.scene_width / self.tile_size))

    def to_dict(self) -> dict:
        return {"scene_id": self.scene_id, "scene_width": self.scene_width,
                "scene_height": self.scene_height, "tile_size": self.tile_size}

    @classmethod
    def from_dict(cls, data: dict) -> "TileGrid":
        try:
            return cls(data["scene_id"], data["scene_width"], data["scene_height"], data["tile_size"])
        except KeyError as exc:
            raise ValueError(f"tile grid missing field {exc}") from None


def split_scene_device(scene_dev, tile_size: int = 256):
    """u8 [h, w, 3] device scene -> (u8 [rows*cols, ts, ts, 3] device tiles, row-major,
    zero-padded at the ragged edges, (rows, cols))."""
    import torch
    if scene_dev.dtype != torch.uint8 or scene_dev.ndim != 3 or scene_dev.shape[2] != 3:
        raise ValueError(f"expected a uint8 (h, w, 3) device scene, got {tuple(scene_dev.shape)}")
    if tile_size < 1:
        raise ValueError(f"tile_size must be >= 1, got {tile_size}")
    h, w = scene_dev.shape[:2]
    rows, cols = math.ceil(h / tile_size), math.ceil(w / tile_size)
    tiles = torch.empty((rows * cols, tile_size, tile_size, 3), dtype=torch.uint8, device=scene_dev.device)
    _native.call("ice_cut_tiles", _native.ptr(scene_dev.contiguous()), h, w, 3, tile_size, tiles.data_ptr(),
                 _native.stream_handle())
    return tiles, (rows, cols)


def stitch_scene_device(tiles_dev, height: int, width: int, cols: int):
    """Inverse of split_scene_device: u8 [rows*cols, ts, ts, c] (or [.., ts, ts]) -> the
    height x width scene, edge padding cropped."""
    import torch
    ts = tiles_dev.shape[1]
    c = tiles_dev.shape[3] if tiles_dev.ndim == 4 else 1
    out = torch.empty((height, width) + ((c,) if tiles_dev.ndim == 4 else ()), dtype=torch.uint8,
                      device=tiles_dev.device)
    _native.call("ice_stitch_tiles", _native.ptr(tiles_dev.contiguous()), cols, ts, c, height, width,
                 out.data_ptr(), _native.stream_handle())
    return out


def split_scene(scene: SceneRaster, tile_size: int = 256) -> tuple:
    """tiling.py:66-81: row-major tiles, zero-padded at the ragged edges, and the grid."""
    import torch
    grid = TileGrid(scene.scene_id, scene.width, scene.height, tile_size)
    tiles_dev, (rows, cols) = split_scene_device(torch.from_numpy(np.ascontiguousarray(scene.data)).cuda(),
                                                 tile_size)
    host = tiles_dev.cpu().numpy()
    tiles = [Tile(SceneRaster(host[r * cols + c], scene.scene_id), scene.scene_id, r, c)
             for r in range(rows) for c in range(cols)]
    return tiles, grid


def stitch_scene(tiles: list, grid: TileGrid) -> SceneRaster:
    """tiling.py:84-103: reassemble, cropping the edge padding; the reference's checks and
    messages (outside the grid, duplicates, wrong size, missing tiles)."""
    import torch
    ts = grid.tile_size
    seen = {}
    for tile in tiles:
        key = (tile.grid_row, tile.grid_col)
        if not (0 <= tile.grid_row < grid.rows and 0 <= tile.grid_col < grid.cols):
            raise ValueError(f"tile ({tile.grid_row},{tile.grid_col}) outside {grid.rows}x{grid.cols} grid")
        if key in seen:
            raise ValueError(f"duplicate tile ({tile.grid_row},{tile.grid_col})")
        if tile.raster.data.shape != (ts, ts, 3):
            raise ValueError(f"tile ({tile.grid_row},{tile.grid_col}) is not {ts}x{ts}")
        seen[key] = tile
    missing = [(r, c) for r in range(grid.rows) for c in range(grid.cols) if (r, c) not in seen]
    if missing:
        raise ValueError("missing tile " + ", ".join(f"({r},{c})" for r, c in missing))
    stack = np.stack([seen[(r, c)].raster.data for r in range(grid.rows) for c in range(grid.cols)])
    out = stitch_scene_device(torch.from_numpy(stack).cuda(), grid.scene_height, grid.scene_width, grid.cols)
    return SceneRaster(out.cpu().numpy(), grid.scene_id)
