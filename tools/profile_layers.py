"""Per-launch breakdown of one eager train step (CUDA events per C-ABI call).

    python tools/profile_layers.py [--batch 32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_13135_b200 import _native  # noqa: E402
from tests.fixtures import synth  # noqa: E402
from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec  # noqa: E402
from paper_2403_13135_b200.icetrain.train import GradBucketer, device_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
a = ap.parse_args()
dev = torch.device("cuda")
x = torch.stack([torch.from_numpy(synth.random_tile(i)) for i in range(a.batch)]).to(dev)
y = torch.randint(0, 3, (a.batch, 256, 256), dtype=torch.uint8, device=dev)
torch.manual_seed(0)
model = UNet(UNetSpec(), dev)
opt = Adam(model.parameters())
from paper_2403_13135_b200.icetrain.train import SINGLE_GPU_BUCKET  # noqa: E402
bucketer = GradBucketer(model.engine, bucket_bytes=SINGLE_GPU_BUCKET, optimizer=opt)
for _ in range(3):
    device_step(model, opt, x, y, a.batch, bucketer)
torch.cuda.synchronize()
_native.counter.events = []
device_step(model, opt, x, y, a.batch, bucketer)
torch.cuda.synchronize()
evs, _native.counter.events = _native.counter.events, None
tot = 0.0
rows = []
for name, args, e0, e1 in evs:
    ms = e0.elapsed_time(e1)
    fl = bench.conv_flops(name, args)
    tot += ms
    rows.append((ms, name, args, fl))
for ms, name, args, fl in rows:
    tf = fl / (ms / 1e3) / 1e12 if fl else 0
    print(f"{name:18s} {ms:7.3f} ms {tf:7.1f} TF/s  {[a_ if isinstance(a_, int) else '' for a_ in args][:12]}")
print(f"total {tot:.3f} ms")
