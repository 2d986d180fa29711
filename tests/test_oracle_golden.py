"""Pin the CPU oracle (oracle/autolabel_ref.c) to the reference's own outputs.

tests/golden/autolabel_golden.json holds sha256 digests produced by the reference
(`process_tile`, `apply_filter`, `segment`; generator tests/golden/make_golden.py).
Inputs are rebuilt by our generators; their digests must match the reference's too.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import autolabel as orc
from tests.fixtures import synth
from tests.golden.cases import all_cases

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "autolabel_golden.json")))
SAT_ONLY = ((0, (0, 100, 205), (179, 255, 255)), (1, (0, 100, 31), (179, 255, 204)),
            (2, (0, 100, 0), (179, 255, 30)))
SCHEMES = {"ross-sea-summer": orc.ROSS_SEA_SUMMER, "sat-only": SAT_ONLY}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_synth_port_matches_reference_corpus():
    ours = [sha(rgb) for rgb, _ in synth.corpus(101, 64, 0.3)]
    assert ours == GOLDEN["corpus_101_64_0.3"]


CASES = {c["name"]: c for c in all_cases()}


@pytest.mark.parametrize("rec", GOLDEN["cases"], ids=lambda r: r["name"])
def test_oracle_matches_reference(rec):
    rgb = CASES[rec["name"]]["make"]()
    assert sha(rgb) == rec["input_sha"]
    cfg = orc.make_cfg(**rec.get("cfg", {}))
    ranges = SCHEMES[rec.get("scheme", "ross-sea-summer")]
    name = rec.get("scheme", "ross-sea-summer")
    if rec["op"] == "process_tile":
        res = orc.process_tile(rgb, cfg, ranges, name)
        assert res["error"] == rec["error"]
        if not rec["error"]:
            assert sha(res["label"]) == rec["label_sha"]
            assert sha(res["filtered"]) == rec["filtered_sha"]
            assert res["affected_fraction"] == rec["affected_fraction"]
            assert np.bincount(res["label"].ravel(), minlength=3).tolist() == rec["counts"]
    elif rec["op"] == "apply_filter":
        try:
            filtered, mask, aff = orc.apply_filter(rgb, cfg)
            err = ""
        except ValueError as exc:
            err = f"ValueError: {exc}"
        assert err == rec["error"]
        if not err:
            assert sha(filtered) == rec["filtered_sha"]
            assert sha(mask) == rec["mask_sha"]
            assert aff / (rgb.shape[0] * rgb.shape[1]) == rec["affected_fraction"]
    else:
        label, first = orc.segment(rgb, ranges)
        if rec["error"]:
            y, x = divmod(first, rgb.shape[1])
            assert rec["error"] == (f"ValueError: scheme {name!r} matches no class at "
                                    f"row={y}, col={x}")
        else:
            assert first == -1
            assert sha(label) == rec["label_sha"]


def test_hsv_known_answers():
    # test_raster.py:29-32
    px = np.array([[[255, 255, 255], [0, 0, 0], [0, 255, 0]]], np.uint8)
    assert orc.rgb_to_hsv(px).reshape(-1, 3).tolist() == [[0, 0, 255], [0, 0, 0], [60, 255, 255]]


def test_minmax_and_otsu_known_answers():
    # test_kernels.py:72-77, 94-101
    assert orc.minmax_normalize(np.array([[10, 20, 30]], np.uint8)).tolist() == [[0, 128, 255]]
    assert orc.otsu_threshold(np.full((8, 8), 77, np.uint8)) == 0
    bimodal = np.array([[20] * 8 + [200] * 8] * 4, np.uint8)
    t = orc.otsu_threshold(bimodal)
    assert 20 <= t < 200


@pytest.mark.parametrize("rec", [r for r in GOLDEN["cases"] if r["op"] == "process_tile" and not r["error"]
                                 and not r.get("cfg") and r.get("scheme", "ross-sea-summer") == "ross-sea-summer"],
                         ids=lambda r: r["name"])
def test_cv_baseline_port_matches_reference(rec):
    """oracle/autolabel_cv.py (the auto-label CPU baseline bench.py times) reproduces the
    reference's process_tile digests with the default config."""
    cv = pytest.importorskip("oracle.autolabel_cv")
    if cv.cv2 is None:
        pytest.skip("cv2 unavailable")
    rgb = CASES[rec["name"]]["make"]()
    if min(rgb.shape[:2]) < 21:
        pytest.skip("window larger than the tile")
    f, lbl, a, first = cv.process_tile(rgb)
    assert sha(f) == rec["filtered_sha"]
    assert sha(lbl) == rec["label_sha"]
    assert a / (rgb.shape[0] * rgb.shape[1]) == rec["affected_fraction"]
