"""tcgen05 implicit-GEMM convolutions vs a plain PyTorch fp32 reference of the same op.

Inputs are rounded to bf16 first, so the reference sees exactly the kernel's operands;
remaining differences are fp32 accumulation order and the bf16 output rounding.
"""
import pytest

torch = pytest.importorskip("torch")
import torch.nn.functional as F

from paper_2403_13135_b200.icetrain import ops

pytestmark = pytest.mark.gpu
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def rnd(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def nchw(t):
    return t.permute(0, 3, 1, 2).float()


def krsc_to_oihw(w):
    return w.permute(0, 3, 1, 2).float()


SHAPES = [  # n, h, w, c1, c2, cout, ksize
    (2, 16, 16, 64, 0, 64, 3),
    (2, 8, 8, 64, 64, 128, 3),
    (3, 32, 32, 128, 0, 256, 3),
    (1, 4, 4, 64, 0, 64, 3),
    (2, 64, 64, 64, 0, 128, 3),
    (4, 256, 256, 64, 0, 64, 3),
    (2, 16, 16, 64, 0, 64, 1),
    (33, 8, 8, 128, 128, 512, 3),
]


@pytest.mark.parametrize("shape", SHAPES, ids=str)
def test_fprop(shape):
    n, h, w, c1, c2, cout, k = shape
    torch.manual_seed(0)
    x1 = rnd(n, h, w, c1)
    x2 = rnd(n, h, w, c2) if c2 else None
    wt = rnd(cout, k, k, c1 + c2, scale=0.05)
    b = torch.randn(cout, device="cuda")
    drop = (torch.rand(n, cout, device="cuda") > 0.3).float() / 0.7
    y = ops.conv_fprop(x1, wt, b, x2, relu=True, drop=drop, ksize=k)
    xin = nchw(x1) if x2 is None else torch.cat([nchw(x1), nchw(x2)], 1)
    ref = F.relu(F.conv2d(xin, krsc_to_oihw(wt), b, padding=k // 2)) * drop[:, :, None, None]
    assert rel(nchw(y), ref) < 1e-2


@pytest.mark.parametrize("shape", SHAPES, ids=str)
def test_dgrad(shape):
    n, h, w, c1, c2, cout, k = shape
    torch.manual_seed(1)
    dy = rnd(n, h, w, cout)
    wt = rnd(cout, k, k, c1 + c2, scale=0.05)
    ref1 = torch.relu(rnd(n, h, w, c1))
    add1 = rnd(n, h, w, c1)
    drop1 = (torch.rand(n, c1, device="cuda") > 0.2).float() / 0.8
    d1, d2 = ops.conv_dgrad(dy, wt, c1, c2, ksize=k, ref1=ref1, add1=add1, drop1=drop1)
    xin = torch.zeros(n, c1 + c2, h, w, device="cuda", requires_grad=True)
    out = F.conv2d(xin, krsc_to_oihw(wt), padding=k // 2)
    out.backward(nchw(dy))
    g = xin.grad
    want1 = (g[:, :c1] + nchw(add1)) * drop1[:, :, None, None] * (nchw(ref1) > 0)
    assert rel(nchw(d1), want1) < 1e-2
    if c2:
        assert rel(nchw(d2), g[:, c1:]) < 1e-2


@pytest.mark.parametrize("shape", SHAPES, ids=str)
def test_wgrad(shape):
    n, h, w, c1, c2, cout, k = shape
    torch.manual_seed(2)
    x1 = rnd(n, h, w, c1)
    x2 = rnd(n, h, w, c2) if c2 else None
    dy = rnd(n, h, w, cout)
    dw = torch.zeros(cout, k, k, c1 + c2, device="cuda")
    ops.conv_wgrad(x1, dy, dw, x2, ksize=k)
    xin = nchw(x1) if x2 is None else torch.cat([nchw(x1), nchw(x2)], 1)
    wref = torch.zeros(cout, c1 + c2, k, k, device="cuda", requires_grad=True)
    F.conv2d(xin, wref, padding=k // 2).backward(nchw(dy))
    assert rel(dw.permute(0, 3, 1, 2), wref.grad) < 1e-3
