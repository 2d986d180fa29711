"""Gradient overwrite mode vs zero + accumulate: the same backward must give bit-identical
gradients (every element has exactly one producer).  Dev tool (GPU): lists differing tensors."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402
from paper_2403_13135_b200.icetrain import UNet, UNetSpec  # noqa: E402

for spec in (UNetSpec(256, base_channels=16, dropout=0.0), UNetSpec(dropout=0.1)):
    rng = np.random.default_rng(3)
    n = 8 if spec.base_channels == 16 else 4
    x = torch.from_numpy(rng.integers(0, 256, (n, 256, 256, 3), dtype=np.uint8)).cuda()
    y = torch.from_numpy(rng.integers(0, 3, (n, 256, 256), dtype=np.uint8)).cuda()
    torch.manual_seed(0)
    model = UNet(spec)
    eng = model.engine
    out = []
    for ow in (False, True):
        eng.grads.fill_(0.0 if not ow else 123.0)  # overwrite mode must not read the stale values
        eng.grads_stale = ow  # (head + backward)
        A = eng.forward(x, train=True, seed=5)
        dz = eng.head(A, y, train=True, grad_scale=1.0 / y.numel())
        eng.backward(A, dz)
        torch.cuda.synchronize()
        out.append({k: v.clone() for k, v in eng.grad_dict().items()})
    bad = [k for k in out[0] if not torch.equal(out[0][k], out[1][k])]
    print(spec, "differing tensors:", bad)
    for k in bad[:10]:
        a, b = out[0][k], out[1][k]
        print("  ", k, float((a - b).abs().max()), int((a != b).sum()), a.numel())
    # physical buffer: elements no producer writes (alignment gaps between tensors: never read)
    print("  unwritten flat-buffer elements:", int((eng.grads == 123.0).sum()))
