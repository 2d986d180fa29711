"""Reference-facing value types of the labeling path.

Same names, fields and validation messages as the reference
(raster.py:28-142, cloudfilter.py:23-79, segmentation.py:21-110, engine.py:118-133) so
callers and tests written against `icelabel` work unchanged.  No arithmetic lives here.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np


class ClassId(enum.IntEnum):
    THICK_ICE = 0
    THIN_ICE = 1
    OPEN_WATER = 2


CLASS_COLORS = {ClassId.THICK_ICE: (255, 0, 0), ClassId.THIN_ICE: (0, 0, 255),
                ClassId.OPEN_WATER: (0, 255, 0)}


def _check_hwc(data, what="(h, w, 3)"):
    data = np.asarray(data)
    if data.ndim != 3 or data.shape[2] != 3:
        raise ValueError(f"expected {what} array, got shape {data.shape}")
    if data.dtype != np.uint8:
        raise ValueError(f"expected uint8 samples, got {data.dtype}")
    return data


@dataclass(eq=False)
class SceneRaster:
    data: np.ndarray
    scene_id: str = ""

    def __post_init__(self):
        self.data = _check_hwc(self.data)
        if self.data.shape[0] == 0 or self.data.shape[1] == 0:
            raise ValueError("empty raster")

    @property
    def height(self):
        return self.data.shape[0]

    @property
    def width(self):
        return self.data.shape[1]

    def same_pixels(self, other):
        return np.array_equal(self.data, other.data)


@dataclass(eq=False)
class Tile:
    raster: SceneRaster
    scene_id: str
    grid_row: int
    grid_col: int

    def __post_init__(self):
        if self.raster.width != self.raster.height:
            raise ValueError(f"tile raster must be square, got {self.raster.width}x{self.raster.height}")
        if self.grid_row < 0 or self.grid_col < 0:
            raise ValueError("grid position must be nonnegative")


@dataclass(eq=False)
class LabelMask:
    data: np.ndarray

    def __post_init__(self):
        self.data = np.asarray(self.data)
        if self.data.ndim != 2:
            raise ValueError(f"expected 2-d array, got shape {self.data.shape}")
        if self.data.dtype != np.uint8:
            raise ValueError(f"expected uint8 class ids, got {self.data.dtype}")
        if self.data.max(initial=0) > max(ClassId):
            raise ValueError("class id out of range")

    @property
    def height(self):
        return self.data.shape[0]

    @property
    def width(self):
        return self.data.shape[1]

    def same_labels(self, other):
        return np.array_equal(self.data, other.data)


MASK_OTSU = "otsu"
MASK_FIXED = "fixed"


@dataclass(frozen=True)
class FilterConfig:
    bg_dilate_k: int = 7
    bg_median_k: int = 21
    noise_median_k: int = 3
    mask_mode: str = MASK_OTSU
    fixed_t: int = 128
    diff_truncate: bool = False
    truncate_t: int = 16

    def __post_init__(self):
        for name in ("bg_dilate_k", "bg_median_k", "noise_median_k"):
            k = getattr(self, name)
            if not (isinstance(k, int) and k >= 3 and k % 2 == 1):
                raise ValueError(f"{name} must be an odd int >= 3, got {k!r}")
        if self.mask_mode not in (MASK_OTSU, MASK_FIXED):
            raise ValueError(f"mask_mode must be {MASK_OTSU!r} or {MASK_FIXED!r}")
        for name in ("fixed_t", "truncate_t"):
            t = getattr(self, name)
            if not 0 <= t <= 255:
                raise ValueError(f"{name} out of range: {t}")

    def to_dict(self):
        return {f: getattr(self, f) for f in self.__dataclass_fields__}

    @classmethod
    def from_dict(cls, data):
        return cls(**{f: data[f] for f in cls.__dataclass_fields__ if f in data})


@dataclass(frozen=True)
class FilterOutput:
    filtered: SceneRaster
    cloud_shadow_mask: np.ndarray
    affected_fraction: float

    def __post_init__(self):
        if self.cloud_shadow_mask.shape != self.filtered.data.shape[:2]:
            raise ValueError("mask dimensions must match the raster")
        if not 0.0 <= self.affected_fraction <= 1.0:
            raise ValueError(f"affected_fraction out of range: {self.affected_fraction}")


HSV_MAX = (179, 255, 255)


@dataclass(frozen=True)
class ColorRange:
    class_id: ClassId
    lower: tuple
    upper: tuple

    def __post_init__(self):
        lo = tuple(int(v) for v in self.lower)
        up = tuple(int(v) for v in self.upper)
        if len(lo) != 3 or len(up) != 3:
            raise ValueError("lower and upper must be (h, s, v) triples")
        lo = (min(lo[0], 179), lo[1], lo[2])
        up = (min(up[0], 179), up[1], up[2])
        for name, (a, b), cap in zip(("h", "s", "v"), zip(lo, up), HSV_MAX):
            if not (0 <= a <= b <= cap):
                raise ValueError(f"{name} bounds [{a}, {b}] invalid, need 0 <= lower <= upper <= {cap}")
        object.__setattr__(self, "lower", lo)
        object.__setattr__(self, "upper", up)
        object.__setattr__(self, "class_id", ClassId(self.class_id))


@dataclass(frozen=True)
class SegmentationScheme:
    name: str
    ranges: tuple

    def __post_init__(self):
        ranges = tuple(self.ranges)
        if {r.class_id for r in ranges} != set(ClassId) or len(ranges) != len(ClassId):
            raise ValueError("scheme needs exactly one range per class")
        ranges = tuple(sorted(ranges, key=lambda r: r.class_id))
        covered = np.zeros(256, bool)
        for r in ranges:
            covered[r.lower[2]: r.upper[2] + 1] = True
        if not covered.all():
            gap = int(np.flatnonzero(~covered)[0])
            raise ValueError(f"V intervals leave a gap: value {gap} belongs to no class")
        object.__setattr__(self, "ranges", ranges)

    def to_dict(self):
        return {"name": self.name,
                "ranges": [{"class": r.class_id.name, "lower": list(r.lower), "upper": list(r.upper)}
                           for r in self.ranges]}

    @classmethod
    def from_dict(cls, data):
        try:
            ranges = tuple(ColorRange(ClassId[r["class"]], tuple(r["lower"]), tuple(r["upper"]))
                           for r in data["ranges"])
            return cls(str(data["name"]), ranges)
        except KeyError as exc:
            raise ValueError(f"scheme dict missing field {exc}") from exc


ROSS_SEA_SUMMER = SegmentationScheme("ross-sea-summer", (
    ColorRange(ClassId.THICK_ICE, (0, 0, 205), (179, 255, 255)),
    ColorRange(ClassId.THIN_ICE, (0, 0, 31), (179, 255, 204)),
    ColorRange(ClassId.OPEN_WATER, (0, 0, 0), (179, 255, 30)),
))
PRESETS = {ROSS_SEA_SUMMER.name: ROSS_SEA_SUMMER}


def get_preset(name):
    try:
        return PRESETS[name]
    except KeyError:
        raise ValueError(f"unknown scheme preset {name!r}, have {sorted(PRESETS)}") from None


@dataclass
class TileResult:
    scene_id: str
    row: int
    col: int
    label: Optional[np.ndarray] = None
    filtered: Optional[np.ndarray] = None
    affected_fraction: float = 0.0
    seconds: float = 0.0
    error: str = ""

    @property
    def ok(self):
        return self.error == ""
