"""Diagnostic: the desk-config 200-step trajectory of the B200 engine next to torch on the same
GPU (the oracle module, fp32 with TF32 off, and bf16 autocast), all from the reference's
initial weights, corpus and batch order (tests/golden/desk_trajectory.pt).

    python tools/diag_traj.py [--which ours,fp32,bf16]
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

which = sys.argv[sys.argv.index("--which") + 1].split(",") if "--which" in sys.argv else ["ours", "fp32", "bf16"]
gold = torch.load("tests/golden/desk_trajectory.pt")
tiles = np.stack([t for t, _ in synth.corpus(101, N_TILES, 0.3)])
x = torch.from_numpy(tiles).cuda()
y = il.autolabel(x)["label"]
xf = x.permute(0, 3, 1, 2).float() / 255.0
yl = y.long()
out = {"ref": gold["losses"]}
if "ours" in which:
    torch.manual_seed(SEED)
    model = UNet(UNetSpec(**SPEC))
    opt = Adam(model.parameters(), lr=1e-3)
    out["ours"] = [synchronized_step([model], [opt], [(x[i.cuda()], y[i.cuda()])])[0] for i in batch_order()]
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
for mode in ("fp32", "bf16"):
    if mode not in which:
        continue
    torch.manual_seed(SEED)
    m = unet_ref.RefUNet(UNetSpec(**SPEC)).cuda()
    opt = torch.optim.Adam(m.parameters(), lr=1e-3)
    ls = []
    for i in batch_order():
        i = i.cuda()
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=mode == "bf16"):
            logits = m(xf[i])
        loss = torch.nn.functional.cross_entropy(logits.float(), yl[i])
        loss.backward()
        opt.step()
        ls.append(float(loss))
    out[mode] = ls
keys = list(out)
print("step " + " ".join(f"{k:>9s}" for k in keys))
for s in range(200):
    print(f"{s:4d} " + " ".join(f"{out[k][s]:9.4f}" for k in keys))
late = {k: float(np.mean(v[-50:])) for k, v in out.items()}
print("late50", late)
print("max", {k: float(np.max(v)) for k, v in out.items()})
