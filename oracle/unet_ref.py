"""CPU fp32 restatement of the reference U-Net train step (TEST INFRASTRUCTURE).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.  Restates
  * icetrain.model.UNet / _DoubleConv / _HalvingConv  (pkg/trainer/src/icetrain/model.py:64-134)
  * icetrain.train.synchronized_step                  (pkg/trainer/src/icetrain/train.py:85-120)
with plain torch CPU modules; the module tree (and so the nn.Conv2d construction order,
the RNG draws of the default init, and the state_dict keys) is the reference's.  It is
pinned against vectors produced by the reference itself (tests/golden/unet_golden.pt,
generator tests/golden/make_unet_golden.py).
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn


class DoubleConv(nn.Module):  # model.py:64-76
    def __init__(self, cin, cout, dropout):
        super().__init__()
        layers = [nn.Conv2d(cin, cout, 3, padding=1), nn.ReLU(inplace=True),
                  nn.Conv2d(cout, cout, 3, padding=1), nn.ReLU(inplace=True)]
        if dropout > 0:
            layers.append(nn.Dropout2d(dropout))
        self.block = nn.Sequential(*layers)

    def forward(self, x):
        return self.block(x)


class HalvingConv(nn.Module):  # model.py:79-88
    def __init__(self, cin):
        super().__init__()
        self.conv = nn.Conv2d(cin, cin // 2, 2)

    def forward(self, x):
        return self.conv(F.pad(x, (0, 1, 0, 1)))


class RefUNet(nn.Module):  # model.py:91-130
    def __init__(self, spec):
        super().__init__()
        self.spec = spec
        chans = [spec.base_channels * (2 ** i) for i in range(spec.depth + 1)]
        self.down = nn.ModuleList()
        cin = spec.in_channels
        for c in chans[:-1]:
            self.down.append(DoubleConv(cin, c, spec.dropout))
            cin = c
        self.pool = nn.MaxPool2d(2)
        self.bottleneck = DoubleConv(chans[-2], chans[-1], spec.dropout)
        self.upsample = nn.Upsample(scale_factor=2, mode="nearest")
        self.halve = nn.ModuleList(HalvingConv(c) for c in reversed(chans[1:]))
        self.up = nn.ModuleList(DoubleConv(c, c // 2, spec.dropout) for c in reversed(chans[1:]))
        self.out = nn.Conv2d(chans[0], spec.classes, 1)

    def forward(self, x):
        skips = []
        for block in self.down:
            x = block(x)
            skips.append(x)
            x = self.pool(x)
        x = self.bottleneck(x)
        for halve, block, skip in zip(self.halve, self.up, reversed(skips)):
            x = halve(self.upsample(x))
            x = block(torch.cat([skip, x], dim=1))
        return self.out(x)


def images_to_input(images_u8):
    """train.py:60-65: uint8 NHWC -> float32 NCHW / 255."""
    return torch.as_tensor(images_u8).permute(0, 3, 1, 2).float() / 255.0


def loss_and_grads(model: RefUNet, x, y):
    """CrossEntropyLoss (mean) forward + backward (train.py:89-99); returns
    (loss, logits, {name: grad})."""
    model.zero_grad(set_to_none=True)
    logits = model(x)
    loss = nn.CrossEntropyLoss()(logits, y)
    loss.backward()
    return float(loss.detach()), logits.detach(), {k: p.grad.detach().clone() for k, p in model.named_parameters()}


def synchronized_step(models, optimizers, shards):
    """train.py:85-120 without the thread pool: shard-size-weighted gradient average,
    identical Adam step on every replica; returns (union mean loss, count)."""
    outcomes = []
    for model, (x, y) in zip(models, shards):
        if len(x) == 0:
            outcomes.append(([torch.zeros_like(p) for p in model.parameters()], 0, 0.0))
            continue
        loss, _, grads = loss_and_grads(model, x, y)
        outcomes.append((list(grads.values()), len(x), loss))
    total = sum(n for _, n, _ in outcomes)
    if total == 0:
        raise ValueError("synchronized step got only empty shards")
    averaged = [sum(n * g[k] for g, n, _ in outcomes) / total for k in range(len(outcomes[0][0]))]
    for model, opt in zip(models, optimizers):
        for p, g in zip(model.parameters(), averaged):
            p.grad = g.clone()
        opt.step()
    return sum(n * l for _, n, l in outcomes) / total, total
