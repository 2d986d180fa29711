"""GPU executor for the reference labeling engine.

The reference engine (pkg/src/icelabel/engine.py) maps `process_tile` over tiles in three
places: `run_sequential` (:204-214), the `run_local` pool children (:217-224) and the TCP
worker's TASK handler (:778-786, one ThreadPoolExecutor call per tile).  On a GPU box the
unit of work is the whole chunk: `process_chunk` labels a TASK's tiles with one fused K1
launch per tile shape and returns the TileResults in input order, with the reference's
per-tile error contract (never raises; errors become "Type: message" strings).  The wire
format (engine.py:398-442) is untouched: TileResult keeps the reference fields.

`install(engine)` points a reference engine module at this executor: its `process_tile`
(the seam the reference's own tests monkeypatch, test_engine.py:168,234) becomes the GPU one
and `run_sequential` labels in chunks; INTEGRATION.md shows the 3-line TASK-handler change
that sends a whole TASK through `process_chunk`.
"""
from __future__ import annotations

import time

from .ops import process_tile, process_tiles
from .types import FilterConfig, SegmentationScheme, TileResult, get_preset

DEFAULT_CHUNK = 256


def process_chunk(tiles: list, config: FilterConfig = None, scheme: SegmentationScheme = None,
                  delay_s: float = 0.0) -> list:
    """One TASK's tiles -> TileResults in input order (engine.py:778-786 semantics)."""
    config = config or FilterConfig()
    scheme = scheme or get_preset("ross-sea-summer")
    started = time.perf_counter()
    if delay_s:
        time.sleep(delay_s * len(tiles))  # the reference sleeps delay_s per tile
    try:
        results = process_tiles(tiles, config, scheme)
    except Exception as exc:  # the reference's catch-all, per tile
        elapsed = time.perf_counter() - started
        return [TileResult(t.scene_id, t.grid_row, t.grid_col, seconds=elapsed / max(1, len(tiles)),
                           error=f"{type(exc).__name__}: {exc}") for t in tiles]
    return results


def run_tiles(tiles: list, config: FilterConfig = None, scheme: SegmentationScheme = None,
              chunk_size: int = DEFAULT_CHUNK, delay_s: float = 0.0) -> tuple:
    """`run_sequential`'s map phase on the GPU: chunks of `chunk_size` tiles, results in input
    order.  Returns (results, {"map_s", "tiles_processed", "chunks"})."""
    if chunk_size < 1:
        raise ValueError(f"chunk_size must be >= 1, got {chunk_size}")
    t0 = time.perf_counter()
    results = []
    for lo in range(0, len(tiles), chunk_size):
        results += process_chunk(tiles[lo:lo + chunk_size], config, scheme, delay_s)
    return results, {"map_s": time.perf_counter() - t0, "tiles_processed": sum(r.ok for r in results),
                     "chunks": -(-len(tiles) // chunk_size)}


def install(engine, chunk_size: int = DEFAULT_CHUNK):
    """Point a reference `icelabel.engine` module (or any namespace with the same names) at the
    GPU executor: `process_tile` becomes the GPU drop-in and `run_sequential(job)` labels the
    job's tiles in chunks.  Returns the replaced attributes, for `uninstall`."""
    missing = object()
    saved = {n: getattr(engine, n, missing) for n in ("process_tile", "run_sequential")}
    saved = {n: (v is not missing, None if v is missing else v) for n, v in saved.items()}
    engine.process_tile = process_tile
    load_tiles, timing_cls, outcome_cls = (getattr(engine, n, None) for n in ("load_tiles", "PhaseTiming",
                                                                               "RunOutcome"))

    def run_sequential(job):
        t0 = time.perf_counter()
        tiles = load_tiles(job, parallel=False)
        t1 = time.perf_counter()
        results, _ = run_tiles(tiles, job.filter_config, job.scheme, chunk_size, job.tile_delay_s)
        t2 = time.perf_counter()
        timing = timing_cls(t1 - t0, t2 - t1, time.perf_counter() - t2,
                            tiles_processed=sum(r.ok for r in results), workers=1)
        return outcome_cls(results, timing)

    if load_tiles is not None and timing_cls is not None and outcome_cls is not None:
        engine.run_sequential = run_sequential
    return saved


def uninstall(engine, saved: dict) -> None:
    """Restore what `install` replaced (attributes it created are removed)."""
    for name, (present, value) in saved.items():
        if present:
            setattr(engine, name, value)
        elif hasattr(engine, name):
            delattr(engine, name)
