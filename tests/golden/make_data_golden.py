"""Generate tests/golden/data_golden.json from the REFERENCE (run where /root/reference exists).

    python tests/golden/make_data_golden.py

Records sha256 digests of the reference's cut_tiles / stitch_tiles / encode_labels /
decode_labels (pkg/trainer/src/icetrain/data.py:35-80) outputs, and its confusion counts and
report (pkg/src/icelabel/metrics.py:108-142), and its train_val_split (data.py:125-136), on the
seeded inputs of tests/golden/data_cases.py.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/trainer/src")

from icetrain.data import cut_tiles, decode_labels, encode_labels, stitch_tiles, train_val_split  # noqa: E402  (reference)
from icelabel.metrics import confusion, report, ssim  # noqa: E402
from icelabel.raster import LabelMask, SceneRaster  # noqa: E402
from icelabel.segmentation import parse_labels, render_labels  # noqa: E402
from icelabel.tiling import split_scene, stitch_scene  # noqa: E402

from tests.golden import data_cases as dc  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


out = {"cut": [], "codec": []}
for h, w in dc.SIZES:
    img = dc.scene(h, w)
    tiles = cut_tiles(img, dc.TILE)
    rec = {"h": h, "w": w, "n_tiles": len(tiles), "tiles": [[sha(t), r, c] for t, r, c in tiles]}
    m = dc.mask(h, w)
    mt = cut_tiles(m.astype(np.int64), dc.TILE)
    rec["mask_tiles"] = [[sha(t), str(t.dtype)] for t, _, _ in mt]
    rec["stitch"] = sha(stitch_tiles(tiles, h, w))
    out["cut"].append(rec)
    enc = encode_labels(m.astype(np.int64))
    dec = decode_labels(enc)
    out["codec"].append({"h": h, "w": w, "encode": sha(enc), "decode": sha(dec), "decode_dtype": str(dec.dtype)})
bad = encode_labels(dc.mask(17, 40).astype(np.int64))
bad[3, 5] = (1, 2, 3)
try:
    decode_labels(bad, "x.png")
except ValueError as exc:
    out["decode_error"] = str(exc)
try:
    encode_labels(np.array([[0, 3]]))
except ValueError as exc:
    out["encode_error"] = str(exc)
pred, ref = dc.pred_ref()
cm = confusion(LabelMask(pred), LabelMask(ref))
out["confusion"] = cm.counts.tolist()
out["report"] = report(cm, 0.5).to_dict()
out["report_csv"] = report(cm).to_csv()
out["train_val_split"] = []
for n, frac, seed in dc.SPLITS:
    tr, va = train_val_split(list(range(n)), frac, seed)
    out["train_val_split"].append({"n": n, "frac": frac, "seed": seed, "train": sha(np.array(tr, np.int64)),
                                   "val": sha(np.array(va, np.int64)), "n_val": len(va)})
# icelabel tiling (tiling.py:66-103)
out["split_scene"] = []
for h, w in dc.SIZES:
    scene = SceneRaster(dc.scene(h, w), f"sc{h}x{w}")
    for ts in (dc.TILE, 100):
        tiles, grid = split_scene(scene, ts)
        rec = {"h": h, "w": w, "tile_size": ts, "grid": grid.to_dict(), "rows": grid.rows, "cols": grid.cols,
               "tiles": [[sha(t.raster.data), t.grid_row, t.grid_col, t.scene_id] for t in tiles],
               "stitch": sha(stitch_scene(tiles, grid).data)}
        out["split_scene"].append(rec)
errs = {}
tiles, grid = split_scene(SceneRaster(dc.scene(300, 517), "e"), 256)
for name, bad in (("missing", tiles[:-1]), ("duplicate", tiles + tiles[:1])):
    try:
        stitch_scene(bad, grid)
    except ValueError as exc:
        errs[name] = str(exc)
out["stitch_errors"] = errs
# label colour rendering / parsing (segmentation.py:131-157)
m = dc.mask(17, 40)
rendered = render_labels(LabelMask(m)).data
out["render"] = sha(rendered)
out["parse"] = sha(parse_labels(SceneRaster(rendered)).data)
noisy = dc.noisy_colors(64, 48)
out["parse_snap"] = sha(parse_labels(SceneRaster(noisy), snap=True).data)
try:
    parse_labels(SceneRaster(noisy))
except ValueError as exc:
    out["parse_error"] = str(exc)
# SSIM (metrics.py:153-172)
out["ssim"] = [{"case": name, "value": ssim(SceneRaster(a), SceneRaster(b))} for name, a, b in dc.ssim_pairs()]
json.dump(out, open(os.path.join(os.path.dirname(__file__), "data_golden.json"), "w"), indent=1)
print("ok")
