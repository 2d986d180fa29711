"""Time single conv calls (CUDA events, 20 reps) for given shapes.  Dev tool.

    python tools/time_conv.py fprop|dgrad|wgrad n h w c1 c2 cout [--ref]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_13135_b200.icetrain import ops  # noqa: E402

kind = sys.argv[1]
n, h, w, c1, c2, cout = map(int, sys.argv[2:8])
ref = "--ref" in sys.argv
bf = torch.bfloat16
x1 = torch.randn(n, h, w, c1, device="cuda").to(bf)
x2 = torch.randn(n, h, w, c2, device="cuda").to(bf) if c2 else None
wt = (torch.randn(cout, 3, 3, c1 + c2, device="cuda") * 0.05).to(bf)
dy = torch.randn(n, h, w, cout, device="cuda").to(bf)
b = torch.randn(cout, device="cuda")
dw = torch.zeros(cout, 3, 3, c1 + c2, device="cuda")
r1 = torch.relu(x1) if ref else None


def run():
    if kind == "fprop":
        ops.conv_fprop(x1, wt, b, x2)
    elif kind == "dgrad":
        ops.conv_dgrad(dy, wt, c1, c2, ref1=r1)
    else:
        ops.conv_wgrad(x1, dy, dw, x2)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
fl = 2.0 * n * h * w * cout * 9 * (c1 + c2)
print(f"{kind} {sys.argv[2:8]} {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s")
