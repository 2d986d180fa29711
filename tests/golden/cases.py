"""Auto-label golden cases: how each input is built (shared by make_golden.py and tests).

Inputs come from our own generators so they can be rebuilt on the GPU box; the
golden JSON stores each input's sha256 as produced by the reference's generator.
"""

from __future__ import annotations

import numpy as np

from tests.fixtures import synth


def _gray(seed, count, haze, i, size=256):
    flags = synth.haze_flags(seed, count, haze)
    return synth.scene(seed, i, size, bool(flags[i]))[0]


def _rand(seed, shape):
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


def _flat(v, size):
    return np.full((size, size, 3), v, np.uint8)


def _swath_tile(base, delta, seed, size=256, radius=88, width=24):
    rng = np.random.default_rng(seed)
    v, _ = synth.swath(np.full((size, size), base, np.uint8), rng, (size // 2, size // 2),
                       radius, delta, ring=width)
    return np.repeat(v[:, :, None], 3, axis=2)


def _edge(size=256):
    v = np.full((size, size), 230, np.uint8)
    v[:, : size // 2] = 10
    return np.repeat(v[:, :, None], 3, axis=2)


def all_cases():
    cases = []
    # T-gray: the SURVEY's 64-tile parity/measurement set (generate_corpus(101, 64, 0.3))
    for i in range(64):
        cases.append(dict(name=f"tgray_{i}", op="process_tile",
                          make=lambda i=i: _gray(101, 64, 0.3, i)))
    # T-tint: unequal channels exercise H/S and per-channel backgrounds
    for i in range(12):
        cases.append(dict(name=f"ttint_{i}", op="process_tile",
                          make=lambda i=i: synth.tint(_gray(101, 64, 0.3, i), 101, i)))
    # T-rand: adversarial, ~40% masked
    for i in range(6):
        cases.append(dict(name=f"trand_{i}", op="process_tile",
                          make=lambda i=i: synth.random_tile(i)))
    # sizes, including the window-extent errors and ragged (non multiple of 4) extents
    for size in (2, 5, 16, 21, 22, 23, 24, 31, 33, 64, 100, 128, 255):
        cases.append(dict(name=f"rand_size_{size}", op="process_tile",
                          make=lambda s=size: _rand(1000 + s, (s, s, 3))))
    # configuration variants
    variants = [
        dict(mask_mode="fixed", fixed_t=50),
        dict(mask_mode="fixed", fixed_t=0),
        dict(mask_mode="fixed", fixed_t=255),
        dict(diff_truncate=True, truncate_t=16),
        dict(diff_truncate=True, truncate_t=0),
        dict(bg_median_k=15),
        dict(bg_median_k=3, bg_dilate_k=3),
        dict(noise_median_k=5),
        dict(noise_median_k=7, bg_dilate_k=9, bg_median_k=31),
    ]
    for j, cfg in enumerate(variants):
        cases.append(dict(name=f"cfg_{j}_gray", op="process_tile", cfg=cfg,
                          make=lambda: _gray(101, 64, 0.3, 3)))
        cases.append(dict(name=f"cfg_{j}_rand", op="process_tile", cfg=cfg,
                          make=lambda j=j: _rand(2000 + j, (64, 64, 3))))
    # structured scenes from the reference filter tests (test_filter.py:51-150)
    cases.append(dict(name="flat_140", op="process_tile", make=lambda: _flat(140, 64)))
    cases.append(dict(name="flat_0", op="process_tile", make=lambda: _flat(0, 32)))
    cases.append(dict(name="flat_255", op="process_tile", make=lambda: _flat(255, 32)))
    cases.append(dict(name="haze_blob", op="process_tile", make=lambda: _swath_tile(160, 40, 0)))
    cases.append(dict(name="shadow_ice", op="process_tile", make=lambda: _swath_tile(230, -60, 3)))
    cases.append(dict(name="wide_haze", op="process_tile",
                      make=lambda: _swath_tile(200, 40, 7, radius=110, width=64)))
    cases.append(dict(name="edge", op="process_tile", make=_edge))
    # apply_filter on non-square rasters (the filter itself is not tile-bound)
    for shp in ((64, 48, 3), (48, 64, 3), (30, 97, 3)):
        cases.append(dict(name=f"filter_{shp[0]}x{shp[1]}", op="apply_filter",
                          make=lambda s=shp: _rand(3000 + s[0] + s[1], s)))
    # segment only: V fences, precedence, unmatched-pixel error
    for v in (0, 30, 31, 100, 204, 205, 255):
        cases.append(dict(name=f"seg_v{v}", op="segment", make=lambda v=v: _flat(v, 16)))
    cases.append(dict(name="seg_rand", op="segment", make=lambda: _rand(7, (37, 53, 3))))
    cases.append(dict(name="seg_satonly_gray", op="segment", scheme="sat-only",
                      make=lambda: _flat(100, 16)))
    cases.append(dict(name="seg_satonly_rand", op="segment", scheme="sat-only",
                      make=lambda: _rand(8, (40, 40, 3))))
    cases.append(dict(name="pt_satonly_rand", op="process_tile", scheme="sat-only",
                      make=lambda: _rand(9, (64, 64, 3))))
    # beyond one 256 x 256 CTA (round 2): whole-scene apply_filter and 512^2 tiles run the
    # multi-CTA region path; 1024^2 and 2048^2 also need Otsu's > 128-bit exact compare
    for i in range(4):
        cases.append(dict(name=f"large_gray_512_{i}", op="process_tile",
                          make=lambda i=i: synth.scene(101, i, 512, i % 2 == 0)[0]))
    for i in range(2):
        cases.append(dict(name=f"large_tint_512_{i}", op="process_tile",
                          make=lambda i=i: synth.tint(synth.scene(101, i, 512, True)[0], 101, i)))
    cases.append(dict(name="large_rand_512", op="process_tile", make=lambda: synth.random_tile(3, 512)))
    cases.append(dict(name="large_flat_512", op="process_tile", make=lambda: _flat(140, 512)))
    cases.append(dict(name="large_edge_512", op="process_tile", make=lambda: _edge(512)))
    for shp in ((300, 517, 3), (40, 700, 3), (257, 256, 3), (700, 33, 3)):
        cases.append(dict(name=f"large_filter_{shp[0]}x{shp[1]}", op="apply_filter",
                          make=lambda s=shp: _rand(4000 + s[0] + s[1], s)))
    cases.append(dict(name="large_scene_1024", op="apply_filter",
                      make=lambda: synth.scene(7, 0, 1024, True)[0]))
    cases.append(dict(name="large_scene_2048", op="apply_filter",
                      make=lambda: synth.scene(7, 1, 2048, True)[0]))
    for j, cfg in enumerate(variants):
        cases.append(dict(name=f"large_cfg_{j}", op="apply_filter", cfg=cfg,
                          make=lambda j=j: synth.scene(11, j, 384, True)[0][:320]))
    return cases
