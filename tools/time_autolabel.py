"""Time K1 paths over resident T-gray / T-rand tiles (CUDA events).  Dev tool, not the bench.

    python tools/time_autolabel.py [--tiles 14800] [--kind tgray|trand|tint] [--path 0|1|2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402
from paper_2403_13135_b200 import icelabel as il  # noqa: E402
from tests.fixtures import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tiles", type=int, default=14800)
ap.add_argument("--uniq", type=int, default=296)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kind", default="tgray")
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--prof", action="store_true", help="needs ICE_LIB_PATH=.../_C/prof/libicelabel_b200.so")
a = ap.parse_args()
if a.kind == "trand":
    u = np.stack([synth.random_tile(i, a.size) for i in range(a.uniq)])
elif a.kind == "tint":
    u = np.stack([synth.tint(t, 101, i) for i, (t, _) in enumerate(synth.corpus(101, a.uniq, 0.3, a.size))])
else:
    u = np.stack([t for t, _ in synth.corpus(101, a.uniq, 0.3, a.size)])
x = torch.from_numpy(u).cuda()[torch.arange(a.tiles) % a.uniq]
_native.call("ice_autolabel_set_path", a.path)
out = il.autolabel(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    il.autolabel(x, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
if a.prof:
    import ctypes
    lib = _native.load()
    buf = (ctypes.c_ulonglong * 16)()
    lib.ice_al_prof_read(buf, 1)
    il.autolabel(x, out=out)
    torch.cuda.synchronize()
    lib.ice_al_prof_read(buf, 1)
    tot = sum(buf[:8]) or 1
    print("phase cycles per tile:", [round(buf[i] / a.tiles) for i in range(8)],
          "share:", [round(buf[i] / tot, 3) for i in range(8)])
    print("per tile: distinct values %.1f, passes %.1f, active col blocks/pass %.1f" %
          (buf[8] / a.tiles, buf[9] / a.tiles, buf[10] / max(1, buf[9])))
px = a.tiles * a.size * a.size
print(f"{a.kind} {a.size}^2 path={a.path} tiles={a.tiles}: {ms:.2f} ms  {px / ms / 1e6:.1f} Gpx/s  "
      f"{px * 7 / ms / 1e6:.1f} GB/s  us/tile/SM={ms * 1000 * 148 / a.tiles:.1f}")
