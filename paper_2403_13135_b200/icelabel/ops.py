"""Reference-signature labeling entry points backed by the sm_100a kernels.

Drop-in for the hot path of the reference labeler:
  * process_tile(tile, config, scheme, delay_s=0.0) -> TileResult   (engine.py:145-160)
  * apply_filter(raster, cfg=None) -> FilterOutput                   (cloudfilter.py:99-117)
  * detect_mask(raster, cfg) -> np.ndarray                           (cloudfilter.py:87-96)
  * segment(raster, scheme) -> LabelMask                             (segmentation.py:118-128)
plus the batched device API the GPU pipeline uses:
  * autolabel(rgb_dev, cfg, scheme) -> dict of device tensors  (ice_autolabel, K1)
  * segment_batch(rgb_dev, scheme) -> dict                     (ice_segment, K1s)
Every call goes through libicelabel_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import time

import numpy as np

from .. import _native
from .types import (FilterConfig, FilterOutput, LabelMask, SceneRaster, SegmentationScheme, Tile,
                    TileResult, ROSS_SEA_SUMMER)


def native_cfg(cfg: FilterConfig) -> _native.IceFilterCfg:
    return _native.IceFilterCfg(cfg.bg_dilate_k, cfg.bg_median_k, cfg.noise_median_k,
                                int(cfg.mask_mode == "fixed"), cfg.fixed_t, int(bool(cfg.diff_truncate)),
                                cfg.truncate_t)


def native_scheme(scheme: SegmentationScheme) -> _native.IceScheme:
    sc = _native.IceScheme()
    for k, r in enumerate(scheme.ranges):  # already in precedence order (segmentation.py:62)
        for ch in range(3):
            sc.lo[k][ch] = r.lower[ch]
            sc.hi[k][ch] = r.upper[ch]
        sc.cls[k] = int(r.class_id)
    return sc


def check_windows(cfg: FilterConfig, h: int, w: int) -> None:
    """kernels.py:35-39 in the order detect_mask/estimate_background reach them."""
    for k in (cfg.noise_median_k, cfg.bg_dilate_k, cfg.bg_median_k):
        if k > min(h, w):
            raise ValueError(f"window {k} exceeds image extent {(h, w)}")


def autolabel(rgb, cfg: FilterConfig | None = None, scheme: SegmentationScheme = ROSS_SEA_SUMMER,
              want_mask: bool = False, out=None, stream=None):
    """Fused filter + segmentation for a device batch rgb u8 [n, h, w, 3] (K1), any extent."""
    import torch
    cfg = cfg or FilterConfig()
    if rgb.dtype != torch.uint8 or rgb.ndim != 4 or rgb.shape[3] != 3:
        raise ValueError(f"expected uint8 (n, h, w, 3) device tensor, got {tuple(rgb.shape)} {rgb.dtype}")
    n, h, w, _ = rgb.shape
    check_windows(cfg, h, w)
    dev = rgb.device
    if out is None:
        out = dict(filtered=torch.empty_like(rgb),
                   label=torch.empty((n, h, w), dtype=torch.uint8, device=dev),
                   affected=torch.empty(n, dtype=torch.int32, device=dev),
                   counts=torch.empty((n, 3), dtype=torch.int32, device=dev),
                   unmatched=torch.empty(n, dtype=torch.int32, device=dev))
        out["mask"] = torch.empty((n, h, w), dtype=torch.uint8, device=dev) if want_mask else None
    c = native_cfg(cfg)
    s = native_scheme(scheme)
    # ice_autolabel_scene: one CTA per tile up to 256 x 256 (ice_autolabel), the multi-CTA
    # region path beyond (whole scenes, 512^2 tiles) with caller scratch
    _native.call("ice_autolabel_scene", _native.ptr(rgb.contiguous()), n, h, w, c, s,
                 _native.ptr(out["filtered"]), _native.ptr(out["label"]), _native.ptr(out.get("mask")),
                 _native.ptr(out["affected"]), _native.ptr(out["counts"]), _native.ptr(out["unmatched"]),
                 _native.stream_handle(stream))
    return out


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Contiguous tile range [lo, hi) of `rank` when n tiles are split over `world` ranks
    (tiles are independent -- no data-path collective)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} world={world} rank={rank}")
    return (n * rank) // world, (n * (rank + 1)) // world


def autolabel_sharded(rgb_all, cfg: FilterConfig | None = None, scheme: SegmentationScheme = ROSS_SEA_SUMMER,
                      group=None):
    """Auto-label a corpus split over the ranks of torch.distributed (one GPU each): this rank
    runs K1 on its contiguous shard of ``rgb_all`` (u8 [n, h, w, 3], host or device) and the
    per-class pixel counts / masked-pixel totals of the whole corpus are summed with ONE small
    all-reduce at the end.  Returns (this rank's K1 outputs, (lo, hi), totals) where totals is a
    device int64 tensor [class0, class1, class2, masked, unmatched tiles]."""
    import torch
    import torch.distributed as tdist
    dist_on = tdist.is_available() and tdist.is_initialized()
    world = tdist.get_world_size(group) if dist_on else 1
    rank = tdist.get_rank(group) if dist_on else 0
    lo, hi = shard_bounds(len(rgb_all), world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    local = rgb_all[lo:hi]
    local = local.to(dev, non_blocking=True) if local.device != dev else local
    totals = torch.zeros(5, dtype=torch.int64, device=dev)
    out = None
    if hi > lo:
        out = autolabel(local.contiguous(), cfg, scheme)
        totals[:3] = out["counts"].to(torch.int64).sum(0)
        totals[3] = out["affected"].to(torch.int64).sum()
        totals[4] = (out["unmatched"] >= 0).sum()
    if dist_on and world > 1:
        tdist.all_reduce(totals, group=group)
    return out, (lo, hi), totals


def segment_batch(rgb, scheme: SegmentationScheme = ROSS_SEA_SUMMER, out=None, stream=None):
    """Segment-only labeling of a device batch (K1s)."""
    import torch
    n, h, w, _ = rgb.shape
    dev = rgb.device
    if out is None:
        out = dict(label=torch.empty((n, h, w), dtype=torch.uint8, device=dev),
                   counts=torch.empty((n, 3), dtype=torch.int32, device=dev),
                   unmatched=torch.empty(n, dtype=torch.int32, device=dev))
    s = native_scheme(scheme)
    _native.call("ice_segment", _native.ptr(rgb.contiguous()), n, h, w, s, _native.ptr(out["label"]),
                 _native.ptr(out["counts"]), _native.ptr(out["unmatched"]), _native.stream_handle(stream))
    return out


def _unmatched_message(scheme: SegmentationScheme, index: int, w: int) -> str:
    y, x = divmod(int(index), w)
    return f"scheme {scheme.name!r} matches no class at row={y}, col={x}"


def _device_batch(arrays):
    import torch
    _native.require_cuda()
    host = torch.from_numpy(np.ascontiguousarray(np.stack(arrays))).pin_memory()
    return host.to("cuda", non_blocking=True)


def apply_filter(raster: SceneRaster, cfg: FilterConfig | None = None) -> FilterOutput:
    cfg = cfg or FilterConfig()
    h, w = raster.data.shape[:2]
    check_windows(cfg, h, w)
    res = autolabel(_device_batch([raster.data]), cfg, ROSS_SEA_SUMMER, want_mask=True)
    filtered = res["filtered"][0].cpu().numpy()
    mask = res["mask"][0].cpu().numpy()
    aff = int(res["affected"][0].item())
    return FilterOutput(SceneRaster(filtered, raster.scene_id), mask, float(aff) / (h * w))


def detect_mask(raster: SceneRaster, cfg: FilterConfig) -> np.ndarray:
    return apply_filter(raster, cfg).cloud_shadow_mask


def segment(raster: SceneRaster, scheme: SegmentationScheme) -> LabelMask:
    res = segment_batch(_device_batch([raster.data]), scheme)
    first = int(res["unmatched"][0].item())
    if first >= 0:
        raise ValueError(_unmatched_message(scheme, first, raster.data.shape[1]))
    return LabelMask(res["label"][0].cpu().numpy())


def process_tiles(tiles, config: FilterConfig, scheme: SegmentationScheme) -> list:
    """Batched process_tile: one kernel launch per group of equally-sized tiles."""
    started = time.perf_counter()
    results = [None] * len(tiles)
    groups = {}
    for i, t in enumerate(tiles):
        groups.setdefault(t.raster.data.shape, []).append(i)
    for shape, idx in groups.items():
        h, w = shape[:2]
        try:
            check_windows(config, h, w)
        except ValueError as exc:
            for i in idx:
                t = tiles[i]
                results[i] = TileResult(t.scene_id, t.grid_row, t.grid_col, error=f"ValueError: {exc}")
            continue
        res = autolabel(_device_batch([tiles[i].raster.data for i in idx]), config, scheme)
        filtered = res["filtered"].cpu().numpy()
        label = res["label"].cpu().numpy()
        aff = res["affected"].cpu().numpy()
        un = res["unmatched"].cpu().numpy()
        for j, i in enumerate(idx):
            t = tiles[i]
            if un[j] >= 0:
                results[i] = TileResult(t.scene_id, t.grid_row, t.grid_col,
                                        error="ValueError: " + _unmatched_message(scheme, un[j], w))
            else:
                results[i] = TileResult(t.scene_id, t.grid_row, t.grid_col, label=label[j],
                                        filtered=filtered[j], affected_fraction=float(aff[j]) / (h * w))
    elapsed = time.perf_counter() - started
    for r in results:
        r.seconds = elapsed / max(1, len(tiles))
    return results


def process_tile(tile: Tile, config: FilterConfig, scheme: SegmentationScheme,
                 delay_s: float = 0.0) -> TileResult:
    """engine.py:145-160: never raises; errors become "Type: message" strings."""
    started = time.perf_counter()
    try:
        if delay_s:
            time.sleep(delay_s)
        res = process_tiles([tile], config, scheme)[0]
        res.seconds = time.perf_counter() - started
        return res
    except Exception as exc:  # the reference's catch-all contract
        return TileResult(tile.scene_id, tile.grid_row, tile.grid_col,
                          seconds=time.perf_counter() - started, error=f"{type(exc).__name__}: {exc}")
