"""Diagnostic: desk-config trajectories at a given lr -- torch fp32 on the GPU (from the
reference's initial weights and from 1e-6-perturbed ones) and the B200 engine.

    python tools/diag_lr.py --lr 1e-4 [--pert 2]
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

lr = float(sys.argv[sys.argv.index("--lr") + 1]) if "--lr" in sys.argv else 1e-4
npert = int(sys.argv[sys.argv.index("--pert") + 1]) if "--pert" in sys.argv else 2
ours_pert = int(sys.argv[sys.argv.index("--ours-pert") + 1]) if "--ours-pert" in sys.argv else 0
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
tiles = np.stack([t for t, _ in synth.corpus(101, N_TILES, 0.3)])
x = torch.from_numpy(tiles).cuda()
y = il.autolabel(x)["label"]
xf, yl = x.permute(0, 3, 1, 2).float() / 255.0, y.long()
spec = UNetSpec(**SPEC)


def perturb(sd, seed):
    g = torch.Generator().manual_seed(seed)
    return {k: v * (1 + 1e-6 * torch.randn(v.shape, generator=g)) for k, v in sd.items()}


def torch_run(sd, amp=False):
    m = unet_ref.RefUNet(spec).cuda()
    m.load_state_dict({k: v.cuda() for k, v in sd.items()})
    opt = torch.optim.Adam(m.parameters(), lr=lr)
    ls = []
    for i in batch_order():
        i = i.cuda()
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=amp):
            out = m(xf[i])
        loss = torch.nn.functional.cross_entropy(out.float(), yl[i])
        loss.backward()
        opt.step()
        ls.append(float(loss))
    return ls


def ours_run(sd):
    m = UNet(spec)
    m.load_state_dict(sd)
    opt = Adam(m.parameters(), lr=lr)
    return [synchronized_step([m], [opt], [(x[i.cuda()], y[i.cuda()])])[0] for i in batch_order()]


torch.manual_seed(SEED)
sd0 = unet_ref.RefUNet(spec).state_dict()
runs = {"fp32": torch_run(sd0), "bf16amp": torch_run(sd0, amp=True), "ours": ours_run(sd0)}
for k in range(npert):
    runs[f"fp32_p{k}"] = torch_run(perturb(sd0, 1000 + k))
for k in range(ours_pert):
    runs[f"ours_p{k}"] = ours_run(perturb(sd0, 1000 + k))
base = np.array(runs["fp32"])
for name, ls in runs.items():
    a = np.array(ls)
    rel = np.abs(a - base) / base
    first = int(np.argmax(rel > 0.02)) if (rel > 0.02).any() else 200
    print(f"{name:10s} step200 {a[-1]:.4f} mean_last20 {a[-20:].mean():.4f} median_last50 {np.median(a[-50:]):.4f} "
          f"max {a.max():.3f} first>2% {first} maxrel {rel.max():.3f}")
