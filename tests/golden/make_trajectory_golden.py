"""tests/golden/unet_trajectory.pt: the reference trainer's loss over 200 synchronized_step
calls (north_star: "loss after 200 steps on the same seed and batch order must agree within
2%").  Run in the build container (/root/reference present):

    python tests/golden/make_trajectory_golden.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/trainer/src")

from icetrain.model import UNet, UNetSpec  # noqa: E402  (reference)
from icetrain.train import synchronized_step  # noqa: E402

from tests.golden.trajectory_data import SEED, SPEC, batch_order, corpus  # noqa: E402


def main():
    torch.set_num_threads(8)
    x_u8, y = corpus()
    x = torch.from_numpy(x_u8).permute(0, 3, 1, 2).float() / 255.0
    yt = torch.from_numpy(y)
    torch.manual_seed(SEED)
    model = UNet(UNetSpec(**SPEC))
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    losses = []
    for idx in batch_order():
        losses.append(synchronized_step([model], [opt], [(x[idx], yt[idx])])[0])
    model.eval()
    with torch.no_grad():  # loss of the trained model over the whole corpus (eval mode)
        eval_loss = float(torch.nn.CrossEntropyLoss()(model(x), yt))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "unet_trajectory.pt")
    torch.save({"spec": SPEC, "losses": losses, "eval_loss": eval_loss}, path)
    print("eval loss after 200 steps", eval_loss)
    print("wrote", path, "first", losses[0], "last", losses[-1])


if __name__ == "__main__":
    main()
