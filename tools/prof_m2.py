"""MMA-thread wait accounting of conv_gemm_m2 over one warm train step (debug build with
-DICE_CONV_PROF: ICE_LIB_PATH=.../_C/prof2/libicelabel_b200.so).  Dev tool."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402
from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec  # noqa: E402
from paper_2403_13135_b200.icetrain.train import device_step  # noqa: E402
from tests.fixtures import synth  # noqa: E402

dev = torch.device("cuda")
x = torch.stack([torch.from_numpy(synth.random_tile(i)) for i in range(32)]).to(dev)
y = torch.randint(0, 3, (32, 256, 256), dtype=torch.uint8, device=dev)
torch.manual_seed(0)
model = UNet(UNetSpec(), dev)
opt = Adam(model.parameters())
for _ in range(2):
    device_step(model, opt, x, y, 32)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_ulonglong * 8)()
lib.ice_conv_prof_read(buf, 1)
device_step(model, opt, x, y, 32)
torch.cuda.synchronize()
lib.ice_conv_prof_read(buf, 1)
tiles, kbs = max(1, buf[3]), max(1, buf[4])
print(f"m2 MMA thread: tiles {buf[3]}, K-blocks {buf[4]}; wait for epilogue {buf[0] / 1e6:.2f} Mcyc "
      f"({buf[0] / tiles:.0f}/tile); wait for TMA {buf[1] / 1e6:.2f} Mcyc ({buf[1] / kbs:.0f}/K-block)")
