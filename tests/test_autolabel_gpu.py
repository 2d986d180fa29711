"""K1 / K1s on the GPU, bit-exact against the reference (golden digests) and the oracle.

Golden digests were produced by the reference itself (tests/golden/make_golden.py); the
oracle (oracle/autolabel_ref.c, pinned by tests/test_oracle_golden.py) covers inputs
beyond the golden set.  Calls go through the C ABI (libicelabel_b200.so).
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import autolabel as orc
from paper_2403_13135_b200 import icelabel as il
from tests.fixtures import synth
from tests.golden.cases import all_cases

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "autolabel_golden.json")))
CASES = {c["name"]: c for c in all_cases()}
SAT_ONLY = il.SegmentationScheme("sat-only", (
    il.ColorRange(il.ClassId.THICK_ICE, (0, 100, 205), (179, 255, 255)),
    il.ColorRange(il.ClassId.THIN_ICE, (0, 100, 31), (179, 255, 204)),
    il.ColorRange(il.ClassId.OPEN_WATER, (0, 100, 0), (179, 255, 30))))
SCHEMES = {"ross-sea-summer": il.ROSS_SEA_SUMMER, "sat-only": SAT_ONLY}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("rec", GOLDEN["cases"], ids=lambda r: r["name"])
def test_matches_reference_golden(rec):
    rgb = CASES[rec["name"]]["make"]()
    cfg = il.FilterConfig(**rec.get("cfg", {}))
    scheme = SCHEMES[rec.get("scheme", "ross-sea-summer")]
    if rec["op"] == "process_tile":
        res = il.process_tile(il.Tile(il.SceneRaster(rgb, "t"), "t", 0, 0), cfg, scheme)
        assert res.error == rec["error"]
        if not rec["error"]:
            assert sha(res.label) == rec["label_sha"]
            assert sha(res.filtered) == rec["filtered_sha"]
            assert res.affected_fraction == rec["affected_fraction"]
    elif rec["op"] == "apply_filter":
        try:
            fo = il.apply_filter(il.SceneRaster(rgb), cfg)
            err = ""
        except ValueError as exc:
            err = f"ValueError: {exc}"
        assert err == rec["error"]
        if not err:
            assert sha(fo.filtered.data) == rec["filtered_sha"]
            assert sha(fo.cloud_shadow_mask) == rec["mask_sha"]
            assert fo.affected_fraction == rec["affected_fraction"]
    else:
        try:
            lm = il.segment(il.SceneRaster(rgb), scheme)
            err = ""
        except ValueError as exc:
            err = f"ValueError: {exc}"
        assert err == rec["error"]
        if not err:
            assert sha(lm.data) == rec["label_sha"]


def _batch_vs_oracle(tiles, cfg=None):
    cfg = cfg or il.FilterConfig()
    dev = torch.from_numpy(np.stack(tiles)).cuda()
    res = il.autolabel(dev, cfg, want_mask=True)
    filt = res["filtered"].cpu().numpy()
    lab = res["label"].cpu().numpy()
    mask = res["mask"].cpu().numpy()
    aff = res["affected"].cpu().numpy()
    cnt = res["counts"].cpu().numpy()
    un = res["unmatched"].cpu().numpy()
    ocfg = orc.make_cfg(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    for i, t in enumerate(tiles):
        f, m, a = orc.apply_filter(t, ocfg)
        lbl, first = orc.segment(f)
        assert np.array_equal(filt[i], f), i
        assert np.array_equal(mask[i], m), i
        assert aff[i] == a, i
        assert np.array_equal(lab[i], lbl), i
        assert un[i] == first, i
        assert cnt[i].tolist() == np.bincount(lbl.ravel(), minlength=256)[:3].tolist(), i


def test_batch_tgray_tint_rand_vs_oracle():
    tiles = [rgb for rgb, _ in synth.corpus(7, 24, 0.5)]
    tiles += [synth.tint(t, 7, i) for i, t in enumerate(tiles[:8])]
    tiles += [synth.random_tile(100 + i) for i in range(4)]
    _batch_vs_oracle(tiles)


@pytest.mark.parametrize("size", [21, 37, 64, 129])
def test_ragged_sizes_vs_oracle(size):
    rng = np.random.default_rng(size)
    smooth = np.repeat(np.repeat(rng.integers(0, 256, (size // 8 + 1, size // 8 + 1, 3)), 8, 0), 8, 1)
    tiles = [rng.integers(0, 256, (size, size, 3), dtype=np.uint8),
             smooth[:size, :size].astype(np.uint8)]
    _batch_vs_oracle(tiles)


def test_config_variants_vs_oracle():
    tiles = [rgb for rgb, _ in synth.corpus(11, 4, 1.0, size=96)]
    tiles.append(synth.random_tile(5, size=96))
    for cfg in (il.FilterConfig(noise_median_k=5), il.FilterConfig(bg_median_k=9, bg_dilate_k=5),
                il.FilterConfig(mask_mode="fixed", fixed_t=20), il.FilterConfig(diff_truncate=True)):
        _batch_vs_oracle(tiles, cfg)


def test_hsv_exhaustive_vs_oracle():
    allrgb = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(allrgb >> 16) & 255, (allrgb >> 8) & 255, allrgb & 255], -1).astype(np.uint8)
    dev = torch.from_numpy(rgb).cuda()
    out = torch.empty_like(dev)
    from paper_2403_13135_b200 import _native
    _native.call("ice_rgb_to_hsv", dev.data_ptr(), 1 << 24, out.data_ptr(), _native.stream_handle())
    assert np.array_equal(out.cpu().numpy(), orc.rgb_to_hsv(rgb))


def test_segment_batch_counts_and_unmatched():
    rng = np.random.default_rng(3)
    tiles = rng.integers(0, 256, (8, 33, 47, 3), dtype=np.uint8)
    res = il.segment_batch(torch.from_numpy(tiles).cuda(), SAT_ONLY)
    lab = res["label"].cpu().numpy()
    for i in range(8):
        want, first = orc.segment(tiles[i], ((0, (0, 100, 205), (179, 255, 255)),
                                             (1, (0, 100, 31), (179, 255, 204)),
                                             (2, (0, 100, 0), (179, 255, 30))))
        assert np.array_equal(lab[i], want)
        assert int(res["unmatched"][i]) == first
        assert res["counts"][i].tolist() == np.bincount(want.ravel(), minlength=256)[:3].tolist()


HUE_ONLY = il.SegmentationScheme("hue-only", (
    il.ColorRange(il.ClassId.THICK_ICE, (20, 0, 205), (150, 255, 255)),
    il.ColorRange(il.ClassId.THIN_ICE, (0, 0, 31), (179, 255, 204)),
    il.ColorRange(il.ClassId.OPEN_WATER, (40, 0, 0), (179, 255, 30))))
HUE_SAT = il.SegmentationScheme("hue-sat", (
    il.ColorRange(il.ClassId.THICK_ICE, (20, 10, 205), (150, 255, 255)),
    il.ColorRange(il.ClassId.THIN_ICE, (0, 0, 31), (170, 240, 204)),
    il.ColorRange(il.ClassId.OPEN_WATER, (0, 30, 0), (179, 255, 30))))


def _ranges(scheme):
    return tuple((int(r.class_id), tuple(r.lower), tuple(r.upper)) for r in scheme.ranges)


@pytest.mark.parametrize("scheme", [il.ROSS_SEA_SUMMER, SAT_ONLY, HUE_ONLY, HUE_SAT], ids=lambda s: s.name)
@pytest.mark.parametrize("shape", [(5, 64, 64), (3, 16, 48), (2, 256, 256)])
def test_segment_vec_variants_vs_oracle(scheme, shape):
    """K1s vectorised kernel (npx % 16 == 0): one template variant per scheme kind."""
    rng = np.random.default_rng(shape[1] * 7 + len(scheme.name))
    tiles = rng.integers(0, 256, shape + (3,), dtype=np.uint8)
    tiles[0] = 0
    tiles[-1, ::2] = 255
    res = il.segment_batch(torch.from_numpy(tiles).cuda(), scheme)
    lab = res["label"].cpu().numpy()
    for i in range(shape[0]):
        want, first = orc.segment(tiles[i], _ranges(scheme))
        assert np.array_equal(lab[i], want), i
        assert int(res["unmatched"][i]) == first, i
        assert res["counts"][i].tolist() == np.bincount(want.ravel(), minlength=256)[:3].tolist(), i


def test_segment_vec_raw_scheme_gaps_and_overlaps():
    """C ABI with a raw IceScheme the Python types would reject: V gaps (unmatched pixels),
    overlapping ranges (first wins) and a class id outside 0..2 (labelled, never counted)."""
    from paper_2403_13135_b200 import _native
    ranges = ((0, (0, 0, 200), (179, 255, 250)), (2, (0, 0, 10), (179, 255, 60)),
              (7, (0, 0, 40), (179, 255, 220)))  # class-id order, as the oracle applies them
    sc = _native.IceScheme()
    for k, (c, lo, hi) in enumerate(ranges):
        for ch in range(3):
            sc.lo[k][ch], sc.hi[k][ch] = lo[ch], hi[ch]
        sc.cls[k] = c
    rng = np.random.default_rng(9)
    tiles = rng.integers(0, 256, (6, 32, 64, 3), dtype=np.uint8)
    tiles[1] = 255  # all unmatched from pixel 0
    tiles[2] = 5
    dev = torch.from_numpy(tiles).cuda()
    n, h, w, _ = tiles.shape
    label = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
    counts = torch.empty((n, 3), dtype=torch.int32, device="cuda")
    unmatched = torch.empty(n, dtype=torch.int32, device="cuda")
    _native.call("ice_segment", dev.data_ptr(), n, h, w, sc, label.data_ptr(), counts.data_ptr(),
                 unmatched.data_ptr(), _native.stream_handle())
    lab = label.cpu().numpy()
    for i in range(n):
        want, first = orc.segment(tiles[i], ranges)
        assert np.array_equal(lab[i], want), i
        assert int(unmatched[i]) == first, i
        assert counts[i].tolist() == np.bincount(want.ravel(), minlength=256)[:3].tolist(), i


def test_empty_batch_and_window_errors():
    out = il.autolabel(torch.empty((0, 32, 32, 3), dtype=torch.uint8, device="cuda"))
    assert out["label"].shape == (0, 32, 32)
    with pytest.raises(ValueError, match=r"window 21 exceeds image extent \(16, 16\)"):
        il.autolabel(torch.zeros((1, 16, 16, 3), dtype=torch.uint8, device="cuda"))
    res = il.process_tile(il.Tile(il.SceneRaster(np.zeros((5, 5, 3), np.uint8)), "s", 0, 0),
                          il.FilterConfig(), il.ROSS_SEA_SUMMER)
    assert res.error == "ValueError: window 7 exceeds image extent (5, 5)"


def _edge_tiles():
    """Hand-made 256 x 256 tiles for the SWAR kernel's corner cases."""
    rng = np.random.default_rng(2024)
    const = np.full((256, 256, 3), 97, np.uint8)
    white = np.full((256, 256, 3), 255, np.uint8)
    black = np.zeros((256, 256, 3), np.uint8)
    two = np.where(rng.random((256, 256, 1)) < 0.5, 20, 230).astype(np.uint8).repeat(3, 2)
    stripes = np.zeros((256, 256, 3), np.uint8)
    stripes[:, ::7] = 255
    stripes[::5] = 128
    corner = np.full((256, 256, 3), 200, np.uint8)
    corner[:11, :11] = 3        # exercises the replicated border weights of the 21 x 21 window
    corner[-11:, -11:] = 250
    ramp = np.broadcast_to(np.arange(256, dtype=np.uint8)[None, :, None], (256, 256, 3)).copy()
    return [const, white, black, two, stripes, corner, ramp, ramp.transpose(1, 0, 2).copy()]


def _run_path(tiles, mode, cfg=None, scheme=il.ROSS_SEA_SUMMER):
    from paper_2403_13135_b200 import _native
    _native.call("ice_autolabel_set_path", mode)
    try:
        dev = torch.from_numpy(np.stack(tiles)).cuda()
        res = il.autolabel(dev, cfg or il.FilterConfig(), scheme, want_mask=True)
        torch.cuda.synchronize()
        return {k: v.cpu().numpy() for k, v in res.items() if v is not None}
    finally:
        _native.call("ice_autolabel_set_path", 0)


@pytest.mark.parametrize("cfg", [il.FilterConfig(), il.FilterConfig(mask_mode="fixed", fixed_t=40),
                                 il.FilterConfig(diff_truncate=True, truncate_t=9)],
                         ids=["default", "fixed40", "trunc9"])
def test_swar_kernel_matches_generic_kernel(cfg):
    """The SWAR 256 x 256 kernel and the generic kernel agree on every output."""
    tiles = [rgb for rgb, _ in synth.corpus(13, 12, 0.5)]
    tiles += [synth.tint(t, 13, i) for i, t in enumerate(tiles[:4])]
    tiles += [synth.random_tile(300 + i) for i in range(3)] + _edge_tiles()
    fast = _run_path(tiles, 2, cfg)
    gen = _run_path(tiles, 1, cfg)
    for k in gen:
        for i in range(len(tiles)):
            assert np.array_equal(fast[k][i], gen[k][i]), (k, i)


def test_swar_kernel_vs_oracle_hsv_scheme():
    """SWAR kernel with a hue/saturation scheme (per-pixel HSV classify) against the oracle."""
    tiles = [synth.tint(rgb, 17, i) for i, (rgb, _) in enumerate(synth.corpus(17, 4, 1.0))]
    tiles += [synth.random_tile(900), _edge_tiles()[3]]
    out = _run_path(tiles, 2, None, SAT_ONLY)
    for i, t in enumerate(tiles):
        f, m, a = orc.apply_filter(t)
        assert np.array_equal(out["filtered"][i], f), i
        assert np.array_equal(out["mask"][i], m), i
        assert out["affected"][i] == a, i
        lbl, first = orc.segment(f, _ranges(SAT_ONLY))
        assert np.array_equal(out["label"][i], lbl), i
        assert out["unmatched"][i] == first, i


def test_swar_kernel_edge_tiles_vs_oracle():
    tiles = _edge_tiles()
    out = _run_path(tiles, 2)
    for i, t in enumerate(tiles):
        f, m, a = orc.apply_filter(t)
        lbl, first = orc.segment(f)
        assert np.array_equal(out["filtered"][i], f), i
        assert np.array_equal(out["mask"][i], m), i
        assert out["affected"][i] == a, i
        assert np.array_equal(out["label"][i], lbl), i
        assert out["unmatched"][i] == first, i
        assert out["counts"][i].tolist() == np.bincount(lbl.ravel(), minlength=256)[:3].tolist(), i


def test_autolabel_sharded_single_rank_totals():
    """autolabel_sharded on one rank labels the whole corpus and totals its counts."""
    tiles = np.stack([rgb for rgb, _ in synth.corpus(21, 6, 0.5)])
    out, (lo, hi), totals = il.autolabel_sharded(torch.from_numpy(tiles))
    assert (lo, hi) == (0, 6)
    ref = il.autolabel(torch.from_numpy(tiles).cuda())
    assert totals[:3].tolist() == ref["counts"].to(torch.int64).sum(0).tolist()
    assert int(totals[3]) == int(ref["affected"].sum())
    assert torch.equal(out["label"], ref["label"])


# ---- region path (ice_autolabel_scene): extents beyond one CTA's 256 x 256 planes ----------

def _oracle_check(out, tiles, cfg=None):
    ocfg = None
    if cfg is not None:
        ocfg = orc.make_cfg(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    for i, t in enumerate(tiles):
        f, m, a = orc.apply_filter(t, ocfg) if ocfg is not None else orc.apply_filter(t)
        lbl, first = orc.segment(f)
        assert np.array_equal(out["filtered"][i], f), i
        assert np.array_equal(out["mask"][i], m), i
        assert out["affected"][i] == a, i
        assert np.array_equal(out["label"][i], lbl), i
        assert out["unmatched"][i] == first, i
        assert out["counts"][i].tolist() == np.bincount(lbl.ravel(), minlength=256)[:3].tolist(), i


@pytest.mark.parametrize("cfg", [il.FilterConfig(), il.FilterConfig(mask_mode="fixed", fixed_t=40),
                                 il.FilterConfig(diff_truncate=True, truncate_t=9),
                                 il.FilterConfig(noise_median_k=5, bg_median_k=9, bg_dilate_k=5)],
                         ids=["default", "fixed40", "trunc9", "windows"])
def test_region_path_forced_matches_one_cta_kernels(cfg):
    """Mode 3 cuts even 256^2 tiles into <= 40 x 40 cores with halos: every core border is
    interior, so the halo logic is exercised everywhere; outputs equal the one-CTA kernels."""
    tiles = [rgb for rgb, _ in synth.corpus(13, 6, 0.5)]
    tiles += [synth.tint(t, 13, i) for i, t in enumerate(tiles[:3])]
    tiles += [synth.random_tile(310)] + _edge_tiles()
    one = _run_path(tiles, 0, cfg)
    reg = _run_path(tiles, 3, cfg)
    for k in one:
        for i in range(len(tiles)):
            assert np.array_equal(one[k][i], reg[k][i]), (k, i)


@pytest.mark.parametrize("shape", [(100, 37), (37, 100), (129, 131), (64, 300)])
def test_region_path_ragged_vs_oracle(shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    h, w = shape
    smooth = np.repeat(np.repeat(rng.integers(0, 256, (h // 8 + 1, w // 8 + 1, 3)), 8, 0), 8, 1)
    tiles = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8), smooth[:h, :w].astype(np.uint8)]
    _oracle_check(_run_path(tiles, 3), tiles)


def test_region_path_512_tiles_vs_oracle():
    """BASELINE configs[4] geometry: 512^2 T-gray / T-tint / T-rand tiles (3 x 3 regions)."""
    tiles = [synth.scene(31, i, 512, i % 2 == 0)[0] for i in range(4)]
    tiles += [synth.tint(tiles[0], 31, 0), synth.random_tile(41, 512)]
    _oracle_check(_run_path(tiles, 0), tiles)


def test_region_path_hsv_scheme_and_scene_size():
    """Whole-scene apply_filter (1000 x 1400, no tiling) and a hue/saturation scheme."""
    scene = synth.tint(np.ascontiguousarray(synth.scene(5, 2, 1400, True)[0][:1000]), 5, 2)
    out = _run_path([scene], 0, None, SAT_ONLY)
    f, m, a = orc.apply_filter(scene)
    assert np.array_equal(out["filtered"][0], f)
    assert np.array_equal(out["mask"][0], m)
    assert out["affected"][0] == a
    lbl, first = orc.segment(f, _ranges(SAT_ONLY))
    assert np.array_equal(out["label"][0], lbl)
    assert out["unmatched"][0] == first


@pytest.mark.parametrize("shape", [(512, 512), (600, 768), (257, 256), (256, 1024)], ids=str)
def test_region_swar_windows_match_generic_region_path(shape):
    """The SWAR 256 x 256-window region path (default windows, w % 16 == 0) equals the generic
    region path (mode 1) on T-gray, T-tint and T-rand content, every output."""
    h, w = shape
    base = np.ascontiguousarray(synth.scene(3, 1, max(h, w), True)[0][:h, :w])
    rng = np.random.default_rng(h * w)
    tiles = [base, synth.tint(base, 3, 1), rng.integers(0, 256, (h, w, 3), dtype=np.uint8)]
    sw = _run_path(tiles, 0)
    gen = _run_path(tiles, 1)
    for k in gen:
        for i in range(len(tiles)):
            assert np.array_equal(sw[k][i], gen[k][i]), (k, i)
