"""Diagnostic: per-tensor gradient error of one B200 train step vs torch fp32 (TF32 off) and
torch bf16 autocast on the same GPU, at a given spec / batch.

    python tools/diag_grads.py [--base 16] [--batch 8] [--size 256] [--steps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import unet_ref  # noqa: E402
from paper_2403_13135_b200.icetrain import UNet, UNetSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--base", type=int, default=16)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
spec = UNetSpec(input_size=a.size, base_channels=a.base, dropout=0.0)
rng = np.random.default_rng(a.seed)
imgs = torch.from_numpy(rng.integers(0, 256, (a.batch, a.size, a.size, 3), dtype=np.uint8))
labels = torch.from_numpy(rng.integers(0, 3, (a.batch, a.size, a.size)))
torch.manual_seed(0)
model = UNet(spec)
eng = model.engine
x = imgs.cuda()
A = eng.forward(x, train=False)
A.stats.zero_()
eng.zero_grad()
dz = eng.head(A, labels.to(torch.uint8).cuda(), train=True, grad_scale=1.0 / labels.numel())
eng.backward(A, dz)
torch.cuda.synchronize()
ours = eng.grad_dict()
ref = unet_ref.RefUNet(spec).cuda()
ref.load_state_dict({k: v.cuda() for k, v in model.state_dict().items()})
xf = unet_ref.images_to_input(imgs).cuda()
res = {}
for mode in ("fp32", "bf16"):
    ref.zero_grad(set_to_none=True)
    with torch.autocast("cuda", dtype=torch.bfloat16, enabled=mode == "bf16"):
        out = ref(xf)
    torch.nn.functional.cross_entropy(out.float(), labels.cuda()).backward()
    res[mode] = {k: p.grad.detach().clone() for k, p in ref.named_parameters()}
print(f"loss ours {float(A.stats[0]) / labels.numel():.6f}")
print(f"{'tensor':28s} {'ours':>9s} {'bf16':>9s}  (rel err vs fp32)")
for k in ours:
    g = res["fp32"][k].double().cpu()
    e_o = float((ours[k].double() - g).norm() / g.norm().clamp_min(1e-30))
    e_b = float((res["bf16"][k].double().cpu() - g).norm() / g.norm().clamp_min(1e-30))
    flag = "  <<<" if e_o > max(0.02, 2 * e_b) else ""
    print(f"{k:28s} {e_o:9.2e} {e_b:9.2e}{flag}")
