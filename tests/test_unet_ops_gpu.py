"""The U-Net's non-conv kernels in isolation, against plain PyTorch fp32 references of the same
ops (unet_ops.cu): the 2x2 max-pool forward / fused backward (with the ties bf16 makes common:
routed to the first maximum in window order, like torch's CPU max_pool2d the reference uses),
the fused softmax-cross-entropy head (loss, hits, logits, dW, db, dZ and the bias gradient of
the conv below) and the fused Adam step (torch.optim.Adam, train.py:149)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.nn.functional as F  # noqa: E402

from paper_2403_13135_b200 import _native  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def tied(shape, seed, levels=5):
    """bf16 NHWC with few distinct values (many ties inside 2x2 windows) and zeros (ReLU)."""
    g = torch.Generator().manual_seed(seed)
    v = torch.randint(-1, levels, shape, generator=g).float() * 0.25
    return v.clamp_min(0).to(torch.bfloat16).cuda()


def first_max_route(x, dpool):
    """maxpool backward with ties to the first max in (dy, dx) raster order, NHWC."""
    n, h, w, c = x.shape
    win = x.float().view(n, h // 2, 2, w // 2, 2, c).permute(0, 1, 3, 5, 2, 4).reshape(n, h // 2, w // 2, c, 4)
    arg = win.argmax(-1)  # torch.argmax: first occurrence of the maximum
    first = torch.zeros_like(win)
    first.scatter_(-1, arg.unsqueeze(-1), 1.0)
    # verify torch's argmax picks the first max (the routing rule itself)
    assert bool((win.gather(-1, arg.unsqueeze(-1)).squeeze(-1) == win.max(-1).values).all())
    out = first * dpool.float().unsqueeze(-1)
    return out.view(n, h // 2, w // 2, c, 2, 2).permute(0, 1, 4, 2, 5, 3).reshape(n, h, w, c)


@pytest.mark.parametrize("shape", [(2, 8, 8, 64), (3, 16, 32, 128), (1, 64, 64, 64), (4, 4, 4, 256)], ids=str)
def test_maxpool_fwd_bwd_with_ties(shape):
    n, h, w, c = shape
    st = _native.stream_handle()
    x = tied(shape, 1)
    y = torch.empty(n, h // 2, w // 2, c, dtype=torch.bfloat16, device="cuda")
    _native.call("ice_maxpool_fwd", x.data_ptr(), n, h, w, c, y.data_ptr(), st)
    ref = F.max_pool2d(x.float().permute(0, 3, 1, 2), 2).permute(0, 2, 3, 1)
    assert torch.equal(y.float(), ref)
    g = torch.Generator().manual_seed(2)
    dpool = (torch.randn(n, h // 2, w // 2, c, generator=g)).to(torch.bfloat16).cuda()
    add = (torch.randn(n, h, w, c, generator=g)).to(torch.bfloat16).cuda()
    drop = ((torch.rand(n, c, generator=g) > 0.1).float() / 0.9).cuda()
    dz = torch.empty_like(x)
    db = torch.full((c,), 0.5, device="cuda")
    _native.call("ice_maxpool_bwd", x.data_ptr(), dpool.data_ptr(), add.data_ptr(), drop.data_ptr(), n, h, w, c,
                 dz.data_ptr(), db.data_ptr(), st)
    torch.cuda.synchronize()
    want = (add.float() + first_max_route(x, dpool)) * drop.view(n, 1, 1, c) * (x.float() > 0)
    assert torch.equal(dz, want.to(torch.bfloat16))  # one rounding of an exactly-computed value
    assert rel(db - 0.5, want.double().sum((0, 1, 2))) < 1e-5  # the bias sum uses the unrounded values
    # no add / no drop / no bias
    dz2 = torch.empty_like(x)
    _native.call("ice_maxpool_bwd", x.data_ptr(), dpool.data_ptr(), None, None, n, h, w, c, dz2.data_ptr(), None, st)
    torch.cuda.synchronize()
    assert torch.equal(dz2, (first_max_route(x, dpool) * (x.float() > 0)).to(torch.bfloat16))


@pytest.mark.parametrize("npx,hw", [(4 * 4096, 4096), (3 * 100, 100), (2 * 65536, 65536)], ids=str)
def test_head_ce_against_torch(npx, hw):
    """ice_head_ce: 1x1 conv 64 -> 3 + CrossEntropyLoss, fused with its backward."""
    g = torch.Generator().manual_seed(7)
    h = (torch.randn(npx, 64, generator=g)).clamp_min(0).to(torch.bfloat16).cuda()
    y = torch.randint(0, 3, (npx,), generator=g, dtype=torch.uint8).cuda()
    w = (torch.randn(3, 64, generator=g) * 0.2).cuda()
    b = (torch.randn(3, generator=g) * 0.1).cuda()
    n_img = npx // hw
    drop = ((torch.rand(n_img, 64, generator=g) > 0.1).float() / 0.9).cuda()
    scale = 1.0 / npx
    dz = torch.empty(npx, 64, dtype=torch.bfloat16, device="cuda")
    dw = torch.full((3, 64), 0.25, device="cuda")
    db = torch.full((3,), 0.25, device="cuda")
    stats = torch.zeros(2, device="cuda")
    logits = torch.empty(npx, 3, device="cuda")
    dzb = torch.full((64,), 0.25, device="cuda")
    _native.call("ice_head_ce", h.data_ptr(), npx, hw, y.data_ptr(), w.data_ptr(), b.data_ptr(), drop.data_ptr(),
                 scale, dz.data_ptr(), dw.data_ptr(), db.data_ptr(), stats.data_ptr(), logits.data_ptr(),
                 dzb.data_ptr(), _native.stream_handle())
    torch.cuda.synchronize()
    hd = h.double()
    lg = hd @ w.double().t() + b.double()
    yl = y.long()
    assert rel(logits, lg) < 1e-5
    loss = F.cross_entropy(lg, yl, reduction="sum")
    assert abs(float(stats[0]) - float(loss)) / float(loss) < 1e-5
    assert float(stats[1]) == float((lg.argmax(1) == yl).sum())
    dl = (torch.softmax(lg, 1) - F.one_hot(yl, 3).double()) * scale
    assert rel(dw - 0.25, dl.t() @ hd) < 1e-5
    assert rel(db - 0.25, dl.sum(0)) < 1e-5
    img = torch.arange(npx, device="cuda") // hw
    want_dz = (dl @ w.double()) * drop.double()[img] * (hd > 0)
    assert rel(dz, want_dz) < 5e-3
    assert rel(dzb - 0.25, dz.double().sum(0)) < 1e-5
    # eval: stats only
    stats2 = torch.zeros(2, device="cuda")
    _native.call("ice_head_ce", h.data_ptr(), npx, hw, y.data_ptr(), w.data_ptr(), b.data_ptr(), None, 0.0, None,
                 None, None, stats2.data_ptr(), None, None, _native.stream_handle())
    torch.cuda.synchronize()
    assert torch.equal(stats2, stats)


def test_adam_matches_torch_optim():
    """ice_adam == torch.optim.Adam (defaults of train.py:149) for several steps, plus the bf16
    working copy and the gradient zeroing."""
    n = 1 << 20
    g = torch.Generator().manual_seed(3)
    p0 = torch.randn(n, generator=g)
    p = p0.clone().cuda()
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    wb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ref = torch.nn.Parameter(p0.clone().cuda())
    opt = torch.optim.Adam([ref], lr=1e-3)
    for step in range(1, 6):
        grad = (torch.randn(n, generator=g) * 10 ** (-step)).cuda()
        gk = grad.clone()
        _native.call("ice_adam", p.data_ptr(), gk.data_ptr(), m.data_ptr(), v.data_ptr(), n, step, None, 1e-3, 0.9,
                     0.999, 1e-8, 1, wb.data_ptr(), _native.stream_handle())
        ref.grad = grad
        opt.step()
        torch.cuda.synchronize()
        assert float(gk.abs().max()) == 0.0
        assert rel(p, ref.detach()) < 1e-6, step
        assert torch.equal(wb, p.to(torch.bfloat16))
    st = opt.state[ref]
    assert rel(m, st["exp_avg"]) < 1e-5 and rel(v, st["exp_avg_sq"]) < 1e-5
