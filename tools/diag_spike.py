"""Diagnostic: replay the (bit-reproducible) desk-config trajectory to step K, then compare
the B200 forward/loss on batch K with torch fp32 on the same weights.

    python tools/diag_spike.py [--step 174]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import unet_ref  # noqa: E402
from paper_2403_13135_b200 import icelabel as il  # noqa: E402
from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec, synchronized_step  # noqa: E402
from tests.fixtures import synth  # noqa: E402
from tests.golden.desk_trajectory_data import N_TILES, SEED, SPEC, batch_order  # noqa: E402

K = int(sys.argv[sys.argv.index("--step") + 1]) if "--step" in sys.argv else 174
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
tiles = np.stack([t for t, _ in synth.corpus(101, N_TILES, 0.3)])
x = torch.from_numpy(tiles).cuda()
y = il.autolabel(x)["label"]
torch.manual_seed(SEED)
spec = UNetSpec(**SPEC)
model = UNet(spec)
opt = Adam(model.parameters(), lr=1e-3)
order = batch_order()
for k in range(K):
    synchronized_step([model], [opt], [(x[order[k].cuda()], y[order[k].cuda()])])
idx = order[K].cuda()
xb, yb = x[idx], y[idx]
ref = unet_ref.RefUNet(spec).cuda()
ref.load_state_dict({k: v.cuda() for k, v in model.state_dict().items()})
with torch.no_grad():
    lr_ = ref(xb.permute(0, 3, 1, 2).float() / 255.0)
    loss_ref = float(torch.nn.functional.cross_entropy(lr_, yb.long()))
model.eval()
lo = model(xb.permute(0, 3, 1, 2).float() / 255.0)
loss_ours = float(torch.nn.functional.cross_entropy(lo, yb.long()))
print(f"step {K}: loss ours {loss_ours:.4f} torch-fp32(same weights) {loss_ref:.4f}")
print("logit rel err", float((lo.double() - lr_.double()).norm() / lr_.double().norm()))
print("logit absmax ours", float(lo.abs().max()), "ref", float(lr_.abs().max()))
# per-layer activation magnitudes of the reference forward
acts = {}
hooks = [m.register_forward_hook(lambda mod, i, o, n=n: acts.__setitem__(n, float(o.abs().max())))
         for n, m in ref.named_modules() if isinstance(m, torch.nn.Conv2d)]
with torch.no_grad():
    ref(xb.permute(0, 3, 1, 2).float() / 255.0)
print({k: round(v, 1) for k, v in acts.items()})
pn = {k: round(float(v.norm()), 2) for k, v in model.state_dict().items() if k.endswith("weight")}
print(pn)
