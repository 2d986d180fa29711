"""Pin oracle/data_ref.py to the reference's data-path outputs (tests/golden/data_golden.json)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import data_ref as orc
from tests.golden import data_cases as dc

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "data_golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_cut_stitch_oracle_matches_reference():
    for rec in GOLDEN["cut"]:
        img = dc.scene(rec["h"], rec["w"])
        tiles = orc.cut_tiles(img, dc.TILE)
        assert [[sha(t), r, c] for t, r, c in tiles] == rec["tiles"]
        assert sha(orc.stitch_tiles(tiles, rec["h"], rec["w"])) == rec["stitch"]
        mt = orc.cut_tiles(dc.mask(rec["h"], rec["w"]).astype(np.int64), dc.TILE)
        assert [[sha(t), str(t.dtype)] for t, _, _ in mt] == rec["mask_tiles"]


def test_codec_oracle_matches_reference():
    for rec in GOLDEN["codec"]:
        m = dc.mask(rec["h"], rec["w"]).astype(np.int64)
        enc = orc.encode_labels(m)
        assert sha(enc) == rec["encode"]
        assert sha(orc.decode_labels(enc)) == rec["decode"]


def test_confusion_oracle_matches_reference():
    pred, ref = dc.pred_ref()
    assert orc.confusion(pred, ref).tolist() == GOLDEN["confusion"]


def test_train_val_split_matches_reference():
    """trainer data.py:125-136 on the BASELINE corpus size and edge cases (tiny corpora keep
    at least one training pair; val_fraction 0 gives an empty validation side)."""
    from paper_2403_13135_b200.icetrain.data import train_val_split
    for rec in GOLDEN["train_val_split"]:
        tr, va = train_val_split(list(range(rec["n"])), rec["frac"], rec["seed"])
        assert len(va) == rec["n_val"] and len(tr) + len(va) == rec["n"]
        assert sha(np.array(tr, np.int64)) == rec["train"] and sha(np.array(va, np.int64)) == rec["val"], rec["n"]
    import pytest
    with pytest.raises(ValueError, match="val_fraction"):
        train_val_split([1, 2], 1.0, 0)


def test_snap_and_ssim_oracle_match_reference():
    assert sha(orc.snap_labels(dc.noisy_colors(64, 48))) == GOLDEN["parse_snap"]
    for rec, (name, a, b) in zip(GOLDEN["ssim"], dc.ssim_pairs()):
        assert rec["case"] == name
        assert abs(orc.ssim(a, b) - rec["value"]) <= 1e-12, name


def test_split_scene_oracle_matches_reference():
    for rec in GOLDEN["split_scene"]:
        tiles = orc.cut_tiles(dc.scene(rec["h"], rec["w"]), rec["tile_size"])
        assert [[sha(t), r, c] for t, r, c in tiles] == [x[:3] for x in rec["tiles"]]
        assert (rec["rows"], rec["cols"]) == (1 + tiles[-1][1], 1 + tiles[-1][2])


def test_cut_stitch_refuse_non_byte_data():
    """The GPU cut / stitch kernels move bytes; float or out-of-range data is refused before any
    device work (it would otherwise be silently truncated)."""
    from paper_2403_13135_b200.icetrain import data as D
    with pytest.raises(TypeError, match="cut_tiles: integer data"):
        D.cut_tiles(np.zeros((8, 8), np.float32), 4)
    with pytest.raises(ValueError, match="cut_tiles: values outside"):
        D.cut_tiles(np.full((8, 8), 300, np.int64), 4)
    with pytest.raises(TypeError, match="stitch_tiles: integer data"):
        D.stitch_tiles([(np.zeros((4, 4), np.float64), 0, 0)], 4, 4)
    with pytest.raises(ValueError, match="stitch_tiles: values outside"):
        D.stitch_tiles([(np.full((4, 4), -1, np.int64), 0, 0)], 4, 4)
