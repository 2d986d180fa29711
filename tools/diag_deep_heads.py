"""Per-tensor gradient errors of the deep-spec golden (norm, leading values, random sample) for
the engine and for torch bf16 autocast.  Dev tool (GPU)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from tests.test_unet_gpu import GOLD, UNet, UNetSpec, engine_grads, autocast_bf16_grads, unet_ref, rel
g = GOLD["deep"]
spec = UNetSpec(**g["spec"])
torch.manual_seed(0)
model = UNet(spec)
loss, grads = engine_grads(model, g["images"], g["labels"])
torch.manual_seed(0)
base = autocast_bf16_grads(spec, unet_ref.RefUNet(spec).state_dict(), g["images"], g["labels"])
for k, v in grads.items():
    ref = g["grads"][k]
    head, idx = ref["head"], ref["idx"].long()
    print(f"{k:32s} norm_err {abs(float(v.norm()) - ref['norm']) / ref['norm']:.4f} ac {abs(float(base[k].norm()) - ref['norm']) / ref['norm']:.4f}"
          f"  head_err {rel(v.reshape(-1)[:head.numel()], head):.4f} ac {rel(base[k].reshape(-1)[:head.numel()], head):.4f}"
          f"  sample_err {rel(v.reshape(-1)[idx], ref['sample']):.4f} ac {rel(base[k].reshape(-1)[idx], ref['sample']):.4f}")
