"""Run K1 (autolabel) and K1s (segment) a few times over resident tiles, for ncu.

    python tools/profile_autolabel.py [--tiles 4224] [--reps 2] [--kind tgray|trand]
No timing is reported: numbers taken under a profiler are not bench values.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_13135_b200 import icelabel as il  # noqa: E402
from tests.fixtures import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tiles", type=int, default=1184)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kind", default="tgray")
a = ap.parse_args()
if a.kind == "trand":
    tiles = np.stack([synth.random_tile(i) for i in range(a.tiles)])
else:
    tiles = np.stack([t for t, _ in synth.corpus(101, a.tiles, 0.3)])
x = torch.from_numpy(tiles).cuda()
out = il.autolabel(x)
for _ in range(a.reps):
    il.autolabel(x, out=out)
seg = il.segment_batch(x)
for _ in range(a.reps):
    il.segment_batch(x, out=seg)
torch.cuda.synchronize()
print("done")
