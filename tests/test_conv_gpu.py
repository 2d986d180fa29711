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
    (2, 128, 128, 128, 0, 128, 3),   # row-halo path (W % 128 == 0)
    (1, 4, 256, 64, 64, 64, 3),      # row-halo, concat input, 2 tiles per row
    (3, 128, 128, 64, 0, 64, 3),
    (32, 8, 8, 1024, 0, 2048, 3),    # bottleneck: 256-wide tiles; dgrad splits K (64 tiles)
    (8, 8, 8, 256, 256, 512, 3),     # 8 tiles: fprop and dgrad both split K, concat input
    (3, 8, 256, 128, 128, 128, 3),   # row-pair halo tiles (128-wide), concat input, 2 tiles per row
    (2, 1, 128, 64, 64, 128, 3),     # one-row images: 128-wide halo tiles without pairing
    (3, 2, 256, 64, 64, 128, 3),     # one row pair per image column: pair slabs cover both borders
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
    db1 = torch.zeros(c1, device="cuda")
    d1, d2 = ops.conv_dgrad(dy, wt, c1, c2, ksize=k, ref1=ref1, add1=add1, drop1=drop1, db1=db1)
    xin = torch.zeros(n, c1 + c2, h, w, device="cuda", requires_grad=True)
    out = F.conv2d(xin, krsc_to_oihw(wt), padding=k // 2)
    out.backward(nchw(dy))
    g = xin.grad
    want1 = (g[:, :c1] + nchw(add1)) * drop1[:, :, None, None] * (nchw(ref1) > 0)
    assert rel(nchw(d1), want1) < 1e-2
    assert rel(db1, want1.sum((0, 2, 3))) < 1e-2  # fused bias gradient
    if c2:
        assert rel(nchw(d2), g[:, c1:]) < 1e-2


# 256-row tiles (conv_gemm_m2) forced on, including shapes the size rule would not pick:
# ragged image counts (padding rows in the second M half), concat inputs, 8x8 levels
M2_SHAPES = [(33, 8, 8, 128, 128, 512, 3), (8, 8, 8, 256, 256, 512, 3), (6, 16, 16, 256, 0, 512, 3),
             (3, 32, 32, 128, 0, 256, 3), (5, 16, 16, 512, 512, 512, 3)]


@pytest.fixture
def conv_knobs(monkeypatch):
    """Set tiling switches (read by the library at load and on ice_conv_reload_knobs) for one
    test; the defaults come back afterwards."""
    from paper_2403_13135_b200 import _native

    def set_knobs(**kv):
        for k, v in kv.items():
            monkeypatch.setenv(k, v)
        _native.call("ice_conv_reload_knobs")

    yield set_knobs
    monkeypatch.undo()
    _native.call("ice_conv_reload_knobs")


@pytest.mark.parametrize("shape", M2_SHAPES, ids=str)
def test_m2_tiles_forced(shape, conv_knobs):
    conv_knobs(ICE_CONV_M2="1", ICE_WG_M2="1", ICE_NO_SPLITK="1")  # the 256-row path runs unsplit
    test_fprop(shape)
    test_dgrad(shape)
    test_wgrad(shape)


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


HALVE = [(2, 8, 8, 128, 64), (3, 4, 4, 256, 128), (2, 16, 16, 64, 64), (1, 2, 2, 512, 256),
         (2, 64, 64, 128, 64), (1, 32, 128, 64, 64)]  # the last two take the halo weight-gradient path


def _halve_ref(x_nchw, w_oihw, b):
    up = F.interpolate(x_nchw, scale_factor=2, mode="nearest")
    return F.conv2d(F.pad(up, (0, 1, 0, 1)), w_oihw, b)


def _planes(t):  # [n][2h][2w][c] -> [4][n][h][w][c], plane 2*(y&1)+(x&1)
    return torch.stack([t[:, cy::2, cx::2, :] for cy in (0, 1) for cx in (0, 1)]).contiguous()


@pytest.mark.parametrize("shape", HALVE, ids=str)
def test_halve_fprop_dgrad_wgrad(shape):
    """model.py:79-88,105,128: Upsample(x2, nearest) -> pad(0,1,0,1) -> Conv2d(k=2)."""
    from paper_2403_13135_b200 import _native
    n, h, w, c, cout = shape
    torch.manual_seed(4)
    x = rnd(n, h, w, c)
    w32 = (torch.randn(cout, 2, 2, c, device="cuda") * 0.05)
    wc = torch.empty(cout, 9, c, dtype=torch.bfloat16, device="cuda")
    st = _native.stream_handle()
    _native.call("ice_halve_prep", w32.data_ptr(), cout, c, wc.data_ptr(), st)
    b = torch.randn(cout, device="cuda")
    y = torch.empty(n, 2 * h, 2 * w, cout, dtype=torch.bfloat16, device="cuda")
    _native.call("ice_halve_fprop", x.data_ptr(), c, n, h, w, wc.data_ptr(), b.data_ptr(), cout, y.data_ptr(), st)
    w_oihw = w32.permute(0, 3, 1, 2).contiguous()
    ref = _halve_ref(nchw(x), w_oihw, b)
    assert rel(nchw(y), ref) < 1e-2
    # backward
    dy = rnd(n, 2 * h, 2 * w, cout)
    ref_relu = torch.relu(rnd(n, h, w, c))
    dx = torch.empty(n, h, w, c, dtype=torch.bfloat16, device="cuda")
    dyp = _planes(dy)
    dbx = torch.zeros(c, device="cuda")
    _native.call("ice_halve_dgrad", dyp.data_ptr(), cout, n, h, w, wc.data_ptr(), c, dx.data_ptr(),
                 ref_relu.data_ptr(), None, None, dbx.data_ptr(), st)
    # the same through the packed ReLU mask (bit j of word k = channel 32 k + j > 0): identical
    pos = (ref_relu.view(-1, c).float() > 0).to(torch.int64)
    words = torch.stack([(pos[:, 32 * k:32 * k + 32] << torch.arange(32, device="cuda")).sum(1)
                         for k in range(c // 32)])
    bits = ((words + 2 ** 31) % 2 ** 32 - 2 ** 31).to(torch.int32).contiguous()
    dx_b = torch.empty_like(dx)
    dbx_b = torch.zeros(c, device="cuda")
    _native.call("ice_halve_dgrad", dyp.data_ptr(), cout, n, h, w, wc.data_ptr(), c, dx_b.data_ptr(),
                 None, bits.data_ptr(), None, dbx_b.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(dx_b, dx) and torch.equal(dbx_b, dbx)
    dw = torch.zeros(cout, 2, 2, c, device="cuda")
    _native.call("ice_halve_wgrad", x.data_ptr(), c, dyp.data_ptr(), cout, n, h, w, dw.data_ptr(), st)
    xin = nchw(x).requires_grad_(True)
    wref = w_oihw.clone().requires_grad_(True)
    _halve_ref(xin, wref, b).backward(nchw(dy))
    assert rel(nchw(dx), xin.grad * (nchw(ref_relu) > 0)) < 1e-2
    assert rel(dbx, (xin.grad * (nchw(ref_relu) > 0)).sum((0, 2, 3))) < 1e-2
    assert rel(dw.permute(0, 3, 1, 2), wref.grad) < 1e-2


@pytest.mark.parametrize("shape", [(4, 8, 8, 256, 256, 512), (2, 4, 256, 64, 64, 64), (2, 4, 128, 128, 128, 128)],
                         ids=str)
def test_dgrad_split_k_planes_and_both_outputs(shape):
    """dx1 / dx2 split at c1, sub-pixel planes for dx2, gradient sums, ReLU-backward masks,
    Dropout2d scales and both bias gradients: through the split-K finisher (8x8) and the
    128-wide halo tiles with staged plane stores (unpaired K = 64, row pairs K = 128)."""
    n, h, w, c1, c2, cout = shape
    torch.manual_seed(7)
    dy = rnd(n, h, w, cout)
    wt = rnd(cout, 3, 3, c1 + c2, scale=0.05)
    ref1, ref2 = torch.relu(rnd(n, h, w, c1)), torch.relu(rnd(n, h, w, c2))
    add1 = rnd(n, h, w, c1)
    add2p = rnd(4, n, h // 2, w // 2, c2)
    drop1 = (torch.rand(n, c1, device="cuda") > 0.2).float() / 0.8
    drop2 = (torch.rand(n, c2, device="cuda") > 0.5).float() / 0.5
    db1 = torch.zeros(c1, device="cuda")
    db2 = torch.zeros(c2, device="cuda")
    out2 = torch.empty(4, n, h // 2, w // 2, c2, dtype=torch.bfloat16, device="cuda")
    ref2p = _planes(ref2)
    d1, d2 = ops.conv_dgrad(dy, wt, c1, c2, ref1=ref1, add1=add1, drop1=drop1, db1=db1, out2=out2,
                            ref2=ref2p, add2=add2p, drop2=drop2, db2=db2, planes2=True)
    xin = torch.zeros(n, c1 + c2, h, w, device="cuda", requires_grad=True)
    F.conv2d(xin, krsc_to_oihw(wt), padding=1).backward(nchw(dy))
    g = xin.grad
    want1 = (g[:, :c1] + nchw(add1)) * drop1[:, :, None, None] * (nchw(ref1) > 0)
    add2 = torch.empty(n, h, w, c2, dtype=torch.bfloat16, device="cuda")
    for p_, (cy, cx) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
        add2[:, cy::2, cx::2] = add2p[p_]
    want2 = (g[:, c1:] + nchw(add2)) * drop2[:, :, None, None] * (nchw(ref2) > 0)
    got2 = torch.empty(n, h, w, c2, dtype=torch.bfloat16, device="cuda")
    for p_, (cy, cx) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
        got2[:, cy::2, cx::2] = d2[p_]
    assert rel(nchw(d1), want1) < 1e-2
    assert rel(nchw(got2), want2) < 1e-2
    assert rel(db1, want1.sum((0, 2, 3))) < 1e-2
    assert rel(db2, want2.sum((0, 2, 3))) < 1e-2


@pytest.mark.parametrize("shape", [(2, 16, 16, 64, 0, 64, 3), (4, 256, 256, 64, 0, 64, 3), (2, 128, 128, 128, 0, 128, 3),
                                   (2, 128, 128, 64, 64, 64, 3), (33, 8, 8, 128, 128, 512, 3), (32, 8, 8, 1024, 0, 2048, 3)],
                         ids=str)
def test_relu_bits_roundtrip(shape):
    """fprop's packed ReLU mask equals (y > 0); dgrad with that mask equals dgrad with the bf16
    ReLU reference (all kernels: halo BN 64/128, generic, split-K)."""
    n, h, w, c1, c2, cout, k = shape
    torch.manual_seed(3)
    x1 = rnd(n, h, w, c1)
    x2 = rnd(n, h, w, c2) if c2 else None
    wt = rnd(cout, k, k, c1 + c2, scale=0.05)
    b = torch.randn(cout, device="cuda") * 0.1
    bits = torch.empty(cout // 32, n * h * w, dtype=torch.int32, device="cuda")
    y = ops.conv_fprop(x1, wt, b, x2, relu=True, relu_bits=bits)
    pos = (y.float() > 0).reshape(n * h * w, cout // 32, 32)
    weights = (2 ** torch.arange(32, device="cuda", dtype=torch.int64))
    want = (pos.long() * weights).sum(-1).t()  # [cout/32][npx] as unsigned
    got = bits.long() & 0xFFFFFFFF
    assert torch.equal(got, want)
    # dgrad of a conv whose input is y: mask by bits == mask by the bf16 reference
    wt2 = rnd(64, k, k, cout, scale=0.05)
    dy = rnd(n, h, w, 64)
    db_a, db_b = torch.zeros(cout, device="cuda"), torch.zeros(cout, device="cuda")
    da, _ = ops.conv_dgrad(dy, wt2, cout, ref1=y, db1=db_a)
    dbb, _ = ops.conv_dgrad(dy, wt2, cout, bits1=bits, db1=db_b)
    assert rel(da, dbb) < 1e-6 or torch.equal(da, dbb)
    assert rel(db_a, db_b) < 1e-5


# every tiling switch off in turn (the alternate paths they select stay correct): a halo shape
# with a concat input, a 256-wide GEMM shape that splits K, a (tap, cin) width of 1152, and
# a halving conv on the merged-class tiling
KNOBS = ["ICE_NO_DUAL", "ICE_NO_STAGE", "ICE_NO_SPLITK", "ICE_NO_WGRAD_TRANS256", "ICE_NO_REF_TMA",
         "ICE_NO_HALO_WGRAD", "ICE_NO_HALVE_MERGE", "ICE_NO_PAIR"]


@pytest.mark.parametrize("knob", KNOBS)
def test_tiling_switches(knob, conv_knobs):
    conv_knobs(**{knob: "1"})
    for shape in [(1, 4, 256, 64, 64, 64, 3), (8, 8, 8, 256, 256, 512, 3), (2, 16, 16, 128, 0, 256, 3)]:
        test_fprop(shape)
        test_dgrad(shape)
        test_wgrad(shape)
    test_halve_fprop_dgrad_wgrad((2, 64, 64, 128, 64))


@pytest.mark.parametrize("shape", [(32, 32, 32, 512, 256), (32, 64, 64, 128, 64), (16, 16, 16, 1024, 512)], ids=str)
def test_halve_m2_tiles_forced(shape, conv_knobs):
    """Halving conv with 256-row tiles forced on (256x256 and 256x128 dgrad tiles, 256-row wgrad)."""
    conv_knobs(ICE_CONV_M2="1", ICE_WG_M2="1")
    test_halve_fprop_dgrad_wgrad(shape)


@pytest.mark.parametrize("shape", [(3, 8, 16), (2, 5, 7), (1, 256, 256), (4, 33, 64)], ids=str)
def test_stem_im2col(shape):
    """ice_stem_im2col: u8 NHWC RGB -> [px][64] bf16 rows of the 27 3x3x3 taps (/255, zero
    padded; column 3 t + c for tap t = 3 (dy + 1) + (dx + 1)), columns 27-63 zero."""
    from paper_2403_13135_b200 import _native
    n, h, w = shape
    g = torch.Generator().manual_seed(5)
    img = torch.randint(0, 256, (n, h, w, 3), generator=g, dtype=torch.uint8).cuda()
    out = torch.full((n * h * w, 64), 7, dtype=torch.int16, device="cuda")
    _native.call("ice_stem_im2col", img.data_ptr(), n, h, w, out.data_ptr(), _native.stream_handle())
    torch.cuda.synchronize()
    x = (img.float() / 255.0).permute(0, 3, 1, 2)
    cols = F.unfold(x, 3, padding=1)  # [n][c * 9 + t][px]
    ref = cols.view(n, 3, 9, h * w).permute(0, 3, 2, 1).reshape(n * h * w, 27)
    want = torch.zeros(n * h * w, 64, dtype=torch.bfloat16, device="cuda")
    want[:, :27] = ref.to(torch.bfloat16)
    assert torch.equal(out.view(torch.bfloat16), want)


def _stem_ref(img, wt, bias):
    """fp32 reference of the stem on the kernel's exact operands: bf16(x / 255) and bf16 weights."""
    x = (img.float() / 255.0).to(torch.bfloat16).float().permute(0, 3, 1, 2)
    w27 = wt[:, :27].float().view(64, 3, 3, 3).permute(0, 3, 1, 2)  # [co][(r*3+s)*3+c] -> OIHW
    return F.conv2d(x, w27, bias, padding=1)


@pytest.mark.parametrize("shape", [(3, 8, 16), (2, 5, 7), (2, 256, 256), (4, 33, 64), (1, 64, 32)], ids=str)
def test_stem_fused_fprop_and_wgrad(shape):
    """ice_stem_fprop / ice_stem_wgrad (the first conv straight from u8 pixels, mma.sync with
    gathered im2col fragments) against torch fp32 on the same bf16 operands; the ReLU mask
    words agree with the stored activations bit for bit."""
    from paper_2403_13135_b200 import _native
    n, h, w = shape
    g = torch.Generator().manual_seed(11)
    img = torch.randint(0, 256, (n, h, w, 3), generator=g, dtype=torch.uint8).cuda()
    wt = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    wt[:, :27] = (torch.randn(64, 27, generator=g) * 0.3).to(torch.bfloat16).cuda()
    bias = (torch.randn(64, generator=g) * 0.1).cuda()
    y = torch.empty(n, h, w, 64, dtype=torch.bfloat16, device="cuda")
    bits = torch.zeros(2, n * h * w, dtype=torch.int32, device="cuda")
    st = _native.stream_handle()
    _native.call("ice_stem_fprop", img.data_ptr(), n, h, w, wt.data_ptr(), bias.data_ptr(), y.data_ptr(),
                 bits.data_ptr(), st)
    torch.cuda.synchronize()
    ref = torch.relu(_stem_ref(img, wt, bias)).permute(0, 2, 3, 1)
    assert rel(y, ref) < 4e-3
    pos = (y.view(-1, 64).float() > 0).to(torch.int64)
    want = torch.stack([(pos[:, 32 * c:32 * c + 32] << torch.arange(32, device="cuda")).sum(1) for c in range(2)])
    assert torch.equal(bits.to(torch.int64) & 0xffffffff, want & 0xffffffff)
    # weight gradient: dW[co][k] = sum_p dz[p][co] col[p][k]; columns 27..63 untouched
    dz = rnd(n, h, w, 64, scale=0.5)
    dw = torch.full((64, 64), 0.25, device="cuda")
    _native.call("ice_stem_wgrad", img.data_ptr(), n, h, w, dz.data_ptr(), dw.data_ptr(), st)
    torch.cuda.synchronize()
    x = (img.float() / 255.0).to(torch.bfloat16).float().permute(0, 3, 1, 2)
    cols = F.unfold(x, 3, padding=1).view(n, 3, 9, h * w).permute(0, 3, 2, 1).reshape(n * h * w, 27)
    want_w = dz.view(-1, 64).float().t() @ cols
    assert rel(dw[:, :27] - 0.25, want_w) < 1e-4
    assert torch.equal(dw[:, 27:], torch.full((64, 37), 0.25, device="cuda"))
    # the same, deterministic: a second call adds bit-identical partial sums
    dw2 = torch.full((64, 64), 0.25, device="cuda")
    _native.call("ice_stem_wgrad", img.data_ptr(), n, h, w, dz.data_ptr(), dw2.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(dw, dw2)
