"""Generate tests/golden/unet_golden.pt from the REFERENCE trainer (run in the build
container, where /root/reference exists):

    python tests/golden/make_unet_golden.py

Records, for a desk-scale spec at dropout 0 (the reference's own parity setting,
trainer/tests/conftest.py:6): the seeded initial state_dict digest, logits, loss and
every parameter gradient of one step on fixed synthetic tiles, and the losses of 5
synchronized_step calls (Adam, lr 1e-3) on a fixed batch order.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/trainer/src")

from icetrain.model import UNet, UNetSpec  # noqa: E402  (reference)
from icetrain.train import synchronized_step  # noqa: E402

from tests.fixtures import synth  # noqa: E402


def corpus(n, size):
    tiles = synth.corpus(5, n, 0.5, size=size)
    x = np.stack([t for t, _ in tiles])
    y = np.stack([l for _, l in tiles]).astype(np.int64)
    return x, y


def digest(sd):
    h = hashlib.sha256()
    for k, v in sd.items():
        h.update(k.encode())
        h.update(v.detach().contiguous().numpy().tobytes())
    return h.hexdigest()


def compact(tensors, full):
    """full tensors for the desk spec; otherwise (size cap) norms, the leading 256 values, and
    the values at 1024 seeded random positions of each tensor ("idx" / "sample": an unbiased
    element sample, so a per-tensor relative error is measured on the whole tensor)."""
    if full:
        return {k: v.detach().clone() for k, v in tensors.items()}
    out = {}
    for pos, (k, v) in enumerate(tensors.items()):
        flat = v.detach().reshape(-1)
        idx = torch.randperm(flat.numel(), generator=torch.Generator().manual_seed(1000 + pos))[:1024]
        out[k] = {"norm": float(v.norm()), "head": flat[:256].clone(), "idx": idx.to(torch.int32),
                  "sample": flat[idx].clone()}
    return out


def main():
    torch.set_num_threads(8)
    out = {}
    for name, spec_kw, n in (("desk", dict(input_size=32, base_channels=8, depth=2, dropout=0.0), 4),
                             ("deep", dict(input_size=64, base_channels=16, depth=5, dropout=0.0), 2)):
        spec = UNetSpec(**spec_kw)
        torch.manual_seed(0)
        model = UNet(spec)
        x_u8, y = corpus(n, spec.input_size)
        x = torch.from_numpy(x_u8).permute(0, 3, 1, 2).float() / 255.0
        yt = torch.from_numpy(y)
        logits = model(x)
        loss = torch.nn.CrossEntropyLoss()(logits, yt)
        loss.backward()
        full = name == "desk"
        rec = {"spec": spec_kw, "images": torch.from_numpy(x_u8), "labels": yt.to(torch.uint8),
               "init_digest": digest(model.state_dict()),
               "logits": logits.detach().clone(), "loss": float(loss.detach()),
               "grads": compact({k: p.grad for k, p in model.named_parameters()}, full)}
        # 5 Adam steps, fixed batch order, union batch split over 2 replicas
        torch.manual_seed(0)
        m0 = UNet(spec)
        m1 = UNet(spec)
        m1.load_state_dict(m0.state_dict())
        opts = [torch.optim.Adam(m.parameters(), lr=1e-3) for m in (m0, m1)]
        losses = []
        for step in range(5):
            perm = torch.randperm(n, generator=torch.Generator().manual_seed(step))
            pieces = torch.tensor_split(perm, 2)
            shards = [(x[p], yt[p]) for p in pieces]
            losses.append(synchronized_step([m0, m1], opts, shards)[0])
        rec["step_losses"] = losses
        rec["final_state"] = compact(m0.state_dict(), full)
        out[name] = rec
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "unet_golden.pt")
    torch.save(out, path)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
