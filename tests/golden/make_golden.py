"""Generate tests/golden/autolabel_golden.json from the REFERENCE implementation.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference read-only via PYTHONPATH-style sys.path insertion and
records, for every case, sha256 digests of the input tile and of the reference's
`process_tile` / `apply_filter` / `segment` outputs, plus the affected fraction and
the error string.  Inputs are rebuilt at test time by our own generators
(paper_2403_13135_b200.icelabel.synth), and the input digest pins that those
generators reproduce the reference corpus byte for byte.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from icelabel.cloudfilter import FilterConfig, apply_filter  # noqa: E402  (reference)
from icelabel.engine import process_tile  # noqa: E402
from icelabel.raster import ClassId, SceneRaster, Tile  # noqa: E402
from icelabel.segmentation import ROSS_SEA_SUMMER, ColorRange, SegmentationScheme, segment  # noqa: E402
from icelabel.synth import generate_corpus  # noqa: E402

from tests.golden.cases import all_cases  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


SAT_ONLY = SegmentationScheme("sat-only", (
    ColorRange(ClassId.THICK_ICE, (0, 100, 205), (179, 255, 255)),
    ColorRange(ClassId.THIN_ICE, (0, 100, 31), (179, 255, 204)),
    ColorRange(ClassId.OPEN_WATER, (0, 100, 0), (179, 255, 30))))
SCHEMES = {"ross-sea-summer": ROSS_SEA_SUMMER, "sat-only": SAT_ONLY}


def main() -> None:
    # cross-check: our T-gray generator equals the reference generate_corpus
    ref_corpus = generate_corpus(101, 64, 0.3)
    out = {"corpus_101_64_0.3": [sha(s.raster.data) for s in ref_corpus],
           "cases": []}
    for case in all_cases():
        rgb = case["make"]()
        cfg = FilterConfig(**case.get("cfg", {}))
        scheme = SCHEMES[case.get("scheme", "ross-sea-summer")]
        rec = {k: v for k, v in case.items() if k != "make"}
        rec["input_sha"] = sha(rgb)
        if case["op"] == "process_tile":
            res = process_tile(Tile(SceneRaster(rgb, "t"), "t", 0, 0), cfg, scheme)
            rec["error"] = res.error
            if res.ok:
                rec["label_sha"] = sha(res.label)
                rec["filtered_sha"] = sha(res.filtered)
                rec["affected_fraction"] = res.affected_fraction
                rec["counts"] = np.bincount(res.label.ravel(), minlength=3).tolist()
        elif case["op"] == "apply_filter":
            try:
                fo = apply_filter(SceneRaster(rgb), cfg)
                rec["error"] = ""
                rec["filtered_sha"] = sha(fo.filtered.data)
                rec["mask_sha"] = sha(fo.cloud_shadow_mask)
                rec["affected_fraction"] = fo.affected_fraction
            except ValueError as exc:
                rec["error"] = f"ValueError: {exc}"
        elif case["op"] == "segment":
            try:
                lm = segment(SceneRaster(rgb), scheme)
                rec["error"] = ""
                rec["label_sha"] = sha(lm.data)
                rec["counts"] = np.bincount(lm.data.ravel(), minlength=3).tolist()
            except ValueError as exc:
                rec["error"] = f"ValueError: {exc}"
        out["cases"].append(rec)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "autolabel_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {len(out['cases'])} cases to {path}")


if __name__ == "__main__":
    main()
