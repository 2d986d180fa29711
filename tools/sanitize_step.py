"""Two small U-Net train steps (batch 2, 256^2: every halo kind, row pairs, staged plane stores,
the deep GEMM tiles) for compute-sanitizer.  Dev tool.

    compute-sanitizer --tool memcheck python tools/sanitize_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from tests.fixtures import synth  # noqa: E402
from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec  # noqa: E402
from paper_2403_13135_b200.icetrain.train import device_step  # noqa: E402

dev = torch.device("cuda")
b = int(sys.argv[1]) if len(sys.argv) > 1 else 2
x = torch.stack([torch.from_numpy(synth.random_tile(i)) for i in range(b)]).to(dev)
y = torch.randint(0, 3, (b, 256, 256), dtype=torch.uint8, device=dev)
torch.manual_seed(0)
model = UNet(UNetSpec(), dev)
opt = Adam(model.parameters())
for _ in range(2):
    device_step(model, opt, x, y, b)
torch.cuda.synchronize()
print("done")
