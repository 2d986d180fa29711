"""Time the fused head (ice_head_ce: 1x1 conv 64 -> 3 + cross-entropy + backward) at the bench
shape (batch 32, 256^2).  Dev tool.

    python tools/time_head.py [n_img]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
hw = 65536
npx = n * hw
h = torch.randn(npx, 64, device="cuda").clamp_min(0).to(torch.bfloat16)
y = torch.randint(0, 3, (npx,), device="cuda", dtype=torch.uint8)
w = torch.randn(3, 64, device="cuda") * 0.2
b = torch.randn(3, device="cuda") * 0.1
drop = torch.ones(n, 64, device="cuda")
dz = torch.empty(npx, 64, dtype=torch.bfloat16, device="cuda")
dw, db, stats, dzb = (torch.zeros(3, 64, device="cuda"), torch.zeros(3, device="cuda"), torch.zeros(2, device="cuda"),
                      torch.zeros(64, device="cuda"))
st = _native.stream_handle()


def run():
    _native.call("ice_head_ce", h.data_ptr(), npx, hw, y.data_ptr(), w.data_ptr(), b.data_ptr(), drop.data_ptr(),
                 1.0 / npx, dz.data_ptr(), dw.data_ptr(), db.data_ptr(), stats.data_ptr(), None, dzb.data_ptr(), st)


for _ in range(3):
    run()
torch.cuda.synchronize()
reps = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = npx * (64 * 2 * 2 + 1)
print(f"head_ce n={n}: {ms * 1e3:.1f} us/call, {alg / ms / 1e6:.0f} GB/s algorithmic (h read + dz write + labels)")
