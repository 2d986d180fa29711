"""SURVEY.md 8(f) rows on the GPU against the reference's own outputs
(tests/golden/data_golden.json, generator tests/golden/make_data_golden.py):

  row 1  icelabel split_scene / stitch_scene (tiling.py:66-103), render_labels / parse_labels
         (segmentation.py:131-157), and the K1 -> training device hand-off (train_device);
  row 3  ssim (metrics.py:145-172);
  row 4  the GPU TASK executor under the engine's map phase (engine.py:204-214, 778-786).
"""
import hashlib
import json
import os
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from tests.golden import data_cases as dc  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "data_golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_split_and_stitch_scene_match_reference():
    from paper_2403_13135_b200.icelabel import SceneRaster, TileGrid, split_scene, stitch_scene
    for rec in GOLDEN["split_scene"]:
        scene = SceneRaster(dc.scene(rec["h"], rec["w"]), f"sc{rec['h']}x{rec['w']}")
        tiles, grid = split_scene(scene, rec["tile_size"])
        assert grid.to_dict() == rec["grid"] and (grid.rows, grid.cols) == (rec["rows"], rec["cols"])
        assert [[sha(t.raster.data), t.grid_row, t.grid_col, t.scene_id] for t in tiles] == rec["tiles"]
        back = stitch_scene(tiles[::-1], TileGrid.from_dict(grid.to_dict()))  # any order
        assert sha(back.data) == rec["stitch"] and back.scene_id == scene.scene_id
    tiles, grid = split_scene(SceneRaster(dc.scene(300, 517), "e"), 256)
    with pytest.raises(ValueError, match=GOLDEN["stitch_errors"]["missing"].replace("(", r"\(").replace(")", r"\)")):
        stitch_scene(tiles[:-1], grid)
    with pytest.raises(ValueError, match=r"duplicate tile \(0,0\)"):
        stitch_scene(tiles + tiles[:1], grid)
    with pytest.raises(ValueError, match="tile_size"):
        TileGrid("x", 10, 10, 0)


def test_render_and_parse_labels_match_reference():
    from paper_2403_13135_b200.icelabel import LabelMask, SceneRaster, parse_labels, render_labels
    rendered = render_labels(LabelMask(dc.mask(17, 40)))
    assert sha(rendered.data) == GOLDEN["render"]
    assert sha(parse_labels(rendered).data) == GOLDEN["parse"]
    noisy = SceneRaster(dc.noisy_colors(64, 48))
    assert sha(parse_labels(noisy, snap=True).data) == GOLDEN["parse_snap"]
    with pytest.raises(ValueError) as exc:
        parse_labels(noisy)
    assert str(exc.value) == GOLDEN["parse_error"]


def test_ssim_matches_reference():
    from paper_2403_13135_b200.icelabel import SceneRaster
    from paper_2403_13135_b200.icelabel.metrics import report, ssim
    for rec, (name, a, b) in zip(GOLDEN["ssim"], dc.ssim_pairs()):
        got = ssim(SceneRaster(a), SceneRaster(b))
        assert abs(got - rec["value"]) <= 1e-10, (name, got, rec["value"])
        assert got == ssim(SceneRaster(a), SceneRaster(b))  # fixed-order sums: run-to-run identical
    with pytest.raises(ValueError, match="window"):
        ssim(SceneRaster(dc.scene(10, 40)), SceneRaster(dc.scene(10, 40)))
    with pytest.raises(ValueError, match="shape mismatch"):
        ssim(SceneRaster(dc.scene(20, 40)), SceneRaster(dc.scene(20, 41)))
    from paper_2403_13135_b200.icelabel.metrics import confusion
    from paper_2403_13135_b200.icelabel import LabelMask
    pred, ref = dc.pred_ref()
    rep = report(confusion(LabelMask(pred), LabelMask(ref)), 0.5)
    assert rep.ssim == 0.5


def test_gpu_task_executor_matches_per_tile_process_tile():
    from paper_2403_13135_b200.icelabel import FilterConfig, SceneRaster, Tile, get_preset, process_tile
    from paper_2403_13135_b200.icelabel import engine
    from tests.fixtures import synth
    scheme, cfg = get_preset("ross-sea-summer"), FilterConfig()
    tiles = [Tile(SceneRaster(t, f"s{i}"), f"s{i}", i // 3, i % 3) for i, (t, _) in enumerate(synth.corpus(101, 9, 0.5))]
    tiles.insert(4, Tile(SceneRaster(np.zeros((16, 16, 3), np.uint8), "tiny"), "tiny", 7, 7))  # window error
    chunk = engine.process_chunk(tiles, cfg, scheme)
    assert [(r.scene_id, r.row, r.col) for r in chunk] == [(t.scene_id, t.grid_row, t.grid_col) for t in tiles]
    for t, r in zip(tiles, chunk):
        one = process_tile(t, cfg, scheme)
        assert r.error == one.error
        if r.ok:
            assert np.array_equal(r.label, one.label) and np.array_equal(r.filtered, one.filtered)
            assert r.affected_fraction == one.affected_fraction
    assert chunk[4].error == "ValueError: window 21 exceeds image extent (16, 16)"
    results, info = engine.run_tiles(tiles, cfg, scheme, chunk_size=4)
    assert info["chunks"] == 3 and info["tiles_processed"] == 9
    assert all(a.error == b.error for a, b in zip(results, chunk))
    # install() on an engine-shaped namespace (the reference module's names)
    job = types.SimpleNamespace(filter_config=cfg, scheme=scheme, tile_delay_s=0.0)
    ns = types.SimpleNamespace(process_tile=None, run_sequential=None,
                               load_tiles=lambda j, parallel: tiles,
                               PhaseTiming=lambda *a, **k: ("timing", a, k),
                               RunOutcome=lambda results, timing: (results, timing))
    saved = engine.install(ns, chunk_size=5)
    assert ns.process_tile is process_tile
    out, timing = ns.run_sequential(job)
    assert [r.error for r in out] == [r.error for r in chunk] and timing[2]["tiles_processed"] == 9
    engine.uninstall(ns, saved)
    assert ns.process_tile is None


def test_scene_to_training_stays_on_device():
    """split_scene_device -> K1 labels -> train_device: the same history as train() on the
    host pairs (same split / shuffle / steps; the step is bit-reproducible)."""
    from paper_2403_13135_b200 import icelabel as il
    from paper_2403_13135_b200.icelabel.tiling import split_scene_device, stitch_scene_device
    from paper_2403_13135_b200.icetrain import TrainConfig, UNetSpec, train, train_device
    from tests.fixtures import synth
    scene = np.concatenate([np.concatenate([t for t, _ in synth.corpus(101, 6, 0.5)[r * 3:(r + 1) * 3]], axis=1)
                            for r in range(2)], axis=0)[:, :700]  # 512 x 700: a ragged right edge
    sd = torch.from_numpy(np.ascontiguousarray(scene)).cuda()
    tiles, (rows, cols) = split_scene_device(sd, 256)
    assert (rows, cols) == (2, 3)
    assert torch.equal(stitch_scene_device(tiles, 512, 700, cols), sd)
    lab = il.autolabel(tiles)
    assert int((lab["unmatched"] >= 0).sum()) == 0
    spec = UNetSpec(input_size=256, base_channels=8, depth=4, dropout=0.0)
    cfg = TrainConfig(batch_size=2, epochs=2, seed=4, val_fraction=0.34)
    dev_result, row = train_device(tiles, lab["label"], spec, cfg)
    host_pairs = [(t, l.astype(np.int64)) for t, l in zip(tiles.cpu().numpy(), lab["label"].cpu().numpy())]
    host_result = train(host_pairs, spec, cfg)
    assert dev_result.history == host_result.history
    assert row["devices"] == 1
    with pytest.raises(ValueError, match="do not match"):
        train_device(tiles, lab["label"][:, :10], spec, cfg)
