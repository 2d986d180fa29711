"""Run a few paper-spec U-Net train steps (batch 32, 256^2) for profilers (ncu).

    python tools/profile_step.py [--steps 3] [--batch 32]
No timing is reported: numbers taken under a profiler are not bench values.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from tests.fixtures import synth  # noqa: E402
from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec  # noqa: E402
from paper_2403_13135_b200.icetrain.train import device_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--batch", type=int, default=32)
a = ap.parse_args()
dev = torch.device("cuda")
x = torch.stack([torch.from_numpy(synth.random_tile(i)) for i in range(a.batch)]).to(dev)
y = torch.randint(0, 3, (a.batch, 256, 256), dtype=torch.uint8, device=dev)
torch.manual_seed(0)
model = UNet(UNetSpec(), dev)
opt = Adam(model.parameters())
for _ in range(a.steps):
    device_step(model, opt, x, y, a.batch)
torch.cuda.synchronize()
print("done")
