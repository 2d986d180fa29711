"""Time the halving-conv fprop (ice_halve_fprop) at one U-Net level.  Dev tool.

    python tools/time_halve.py n h w c cout     (h, w = input size; output is 2h x 2w)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402

n, h, w, c, cout = map(int, sys.argv[1:6])
bf = torch.bfloat16
x = torch.randn(n, h, w, c, device="cuda").to(bf)
wc = (torch.randn(cout, 9, c, device="cuda") * 0.05).to(bf)
b = torch.randn(cout, device="cuda")
y = torch.empty(n, 2 * h, 2 * w, cout, device="cuda", dtype=bf)
st = _native.stream_handle()


def run():
    _native.call("ice_halve_fprop", x.data_ptr(), c, n, h, w, wc.data_ptr(), b.data_ptr(), cout, y.data_ptr(), st)


reps = int(os.environ.get("REPS", "20"))
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
mb = (x.numel() + y.numel()) * 2 / 1e6
print(f"halve_fprop {sys.argv[1:6]} {ms:.3f} ms  {mb / ms / 1e3:.0f} GB/s (x + y)")
