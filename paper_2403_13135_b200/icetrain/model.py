"""U-Net on the B200: spec, parameter layout, and the training engine.

Mirrors icetrain.model (/root/reference/pkg/trainer/src/icetrain/model.py):
  * UNetSpec (model.py:29-61) -- same fields, defaults, validation messages;
  * UNet (model.py:91-137)    -- same topology (depth x DoubleConv + MaxPool, bottleneck,
    depth x (Upsample -> HalvingConv -> cat([skip, x]) -> DoubleConv), 1x1 head), same
    parameter initialisation (nn.Conv2d defaults drawn in the reference's construction
    order, so torch.manual_seed(s) gives bit-identical initial weights), same state_dict
    keys/shapes (OIHW fp32) for checkpoints.
The arithmetic runs in libicelabel_b200.so: tcgen05 implicit-GEMM convolutions
(conv_tc.cu) and the fused stem/pool/head/Adam kernels (unet_ops.cu).  Activations are
NHWC bf16 with channel counts padded to multiples of 64 (the padding is exact: padded
channels carry zero weights, zero activations and zero gradients forever).
"""

from __future__ import annotations

import os

from collections import OrderedDict
from dataclasses import asdict, dataclass

import torch

from .. import _native
from . import ops

DROPOUT_CHOICES = (0.0, 0.1, 0.2, 0.3)


@dataclass(frozen=True)
class UNetSpec:
    input_size: int = 256
    in_channels: int = 3
    classes: int = 3
    depth: int = 5
    base_channels: int = 64
    dropout: float = 0.1

    def __post_init__(self) -> None:
        for name in ("input_size", "in_channels", "classes", "depth", "base_channels"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.input_size % (2 ** self.depth):
            raise ValueError(
                f"input_size {self.input_size} is not divisible by "
                f"2^depth = {2 ** self.depth}; the pooling chain would not close")
        if self.dropout not in DROPOUT_CHOICES:
            raise ValueError(f"dropout {self.dropout} not in {DROPOUT_CHOICES} (0.0 disables)")

    @property
    def conv_layers(self) -> int:
        return 5 * self.depth + 3

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, data: dict) -> "UNetSpec":
        return cls(**{f: data[f] for f in cls.__dataclass_fields__ if f in data})


def phys(c: int) -> int:
    return (c + 63) // 64 * 64


def check_tile(h: int, w: int, depth: int) -> None:
    """Tile sides the B200 engine runs: divisible by 2^depth (the reference's own rule,
    model.py:42-45,116-119) and powers of two (the conv kernels' shift/mask index math)."""
    step = 2 ** depth
    if h % step or w % step:
        raise ValueError(f"spatial dims {(h, w)} not divisible by {step}")
    if h & (h - 1) or w & (w - 1):
        raise ValueError(f"tile sides {(h, w)} must be powers of two on the B200 engine "
                         "(the reference accepts any multiple of 2^depth)")


def check_supported(spec: UNetSpec) -> None:
    """Limits of the B200 kernels (the reference accepts more; those raise loudly here)."""
    if spec.in_channels != 3:
        raise ValueError("the B200 stem kernel is specialised for in_channels == 3")
    if spec.classes != 3:
        raise ValueError("the B200 head kernel is specialised for classes == 3")
    if spec.base_channels > 64:
        raise ValueError("the B200 head kernel supports base_channels <= 64")


class Layer:
    """One convolution: logical shapes (reference) and physical slices (flat buffers)."""

    def __init__(self, name, kind, cin, cout, k, c1=None):
        self.name, self.kind, self.cin, self.cout, self.k = name, kind, cin, cout, k
        self.c1 = c1  # logical skip channels of a concat input (up.*.block.0)
        self.cout_p = cout if kind == "out" else phys(cout)
        if kind == "stem":
            self.cin_p, self.k_p = 64, 1  # im2col columns (27 used)
        elif kind == "concat":
            self.cin_p, self.k_p = 2 * phys(c1), k
        else:
            self.cin_p, self.k_p = phys(cin), k
        self.w_shape = (self.cout_p, self.k_p, self.k_p, self.cin_p)
        self.w_off = self.b_off = 0

    @property
    def w_numel(self):
        return self.cout_p * self.k_p * self.k_p * self.cin_p

    def oihw_shape(self):
        return (self.cout, self.cin, self.k, self.k)

    # --- layout conversion (reference OIHW fp32 <-> physical KRSC fp32) -------------
    def to_phys(self, w: torch.Tensor) -> torch.Tensor:
        out = torch.zeros(self.w_shape, dtype=torch.float32)
        if self.kind == "stem":  # [cout][ (r*3+s)*3 + c ]
            out[: self.cout, 0, 0, :27] = w.permute(0, 2, 3, 1).reshape(self.cout, 27)
        elif self.kind == "out":
            out[:, 0, 0, : self.cin] = w[:, :, 0, 0]
        elif self.kind == "concat":
            krsc = w.permute(0, 2, 3, 1)
            p1 = phys(self.c1)
            out[: self.cout, :, :, : self.c1] = krsc[..., : self.c1]
            out[: self.cout, :, :, p1: p1 + self.cin - self.c1] = krsc[..., self.c1:]
        else:
            out[: self.cout, :, :, : self.cin] = w.permute(0, 2, 3, 1)
        return out

    def from_phys(self, p: torch.Tensor) -> torch.Tensor:
        if self.kind == "stem":
            return p[: self.cout, 0, 0, :27].reshape(self.cout, 3, 3, 3).permute(0, 3, 1, 2).contiguous()
        if self.kind == "out":
            return p[:, 0, 0, : self.cin].reshape(self.cout, self.cin, 1, 1).contiguous()
        if self.kind == "concat":
            p1 = phys(self.c1)
            krsc = torch.cat([p[: self.cout, :, :, : self.c1], p[: self.cout, :, :, p1: p1 + self.cin - self.c1]], 3)
            return krsc.permute(0, 3, 1, 2).contiguous()
        return p[: self.cout, :, :, : self.cin].permute(0, 3, 1, 2).contiguous()


def build_layers(spec: UNetSpec):
    """(registration-order list, name -> Layer).  Registration order = the reference's
    state_dict order and its nn.Conv2d construction (= RNG) order (model.py:91-109)."""
    chans = [spec.base_channels * 2 ** i for i in range(spec.depth + 1)]
    layers = []
    cin = spec.in_channels
    for i, c in enumerate(chans[:-1]):
        layers.append(Layer(f"down.{i}.block.0", "stem" if i == 0 else "conv", cin, c, 3))
        layers.append(Layer(f"down.{i}.block.2", "conv", c, c, 3))
        cin = c
    layers.append(Layer("bottleneck.block.0", "conv", chans[-2], chans[-1], 3))
    layers.append(Layer("bottleneck.block.2", "conv", chans[-1], chans[-1], 3))
    for j, c in enumerate(reversed(chans[1:])):
        layers.append(Layer(f"halve.{j}.conv", "halve", c, c // 2, 2))
    for j, c in enumerate(reversed(chans[1:])):
        layers.append(Layer(f"up.{j}.block.0", "concat", c, c // 2, 3, c1=c // 2))
        layers.append(Layer(f"up.{j}.block.2", "conv", c // 2, c // 2, 3))
    layers.append(Layer("out", "out", chans[0], spec.classes, 1))
    return layers, {l.name: l for l in layers}


def readiness_order(spec: UNetSpec):
    """Order in which backward completes each layer's gradient (out first, stem last);
    the flat parameter/gradient buffers are laid out in this order so gradient buckets
    are contiguous slices."""
    d = spec.depth
    names = ["out"]
    for j in reversed(range(d)):
        names += [f"up.{j}.block.2", f"up.{j}.block.0", f"halve.{j}.conv"]
    names += ["bottleneck.block.2", "bottleneck.block.0"]
    for i in reversed(range(d)):
        names += [f"down.{i}.block.2", f"down.{i}.block.0"]
    return names


def flat_layout(spec: UNetSpec):
    """(layers, name -> Layer, numel): each layer's weight and bias slice of the flat
    fp32/bf16 parameter buffers, in readiness order, 256-byte aligned (TMA needs 16 B)."""
    layers, by_name = build_layers(spec)
    off = 0
    for name in readiness_order(spec):
        L = by_name[name]
        L.w_off = off
        off += (L.w_numel + 63) // 64 * 64
        L.b_off = off
        off += (L.cout_p + 63) // 64 * 64
    return layers, by_name, (off + 63) // 64 * 64


def init_reference_params(spec: UNetSpec) -> "OrderedDict[str, torch.Tensor]":
    """nn.Conv2d default init drawn in the reference's construction order (model.py:91-109):
    under torch.manual_seed(s) this equals icetrain.model.UNet(spec).state_dict()."""
    sd = OrderedDict()
    for layer in build_layers(spec)[0]:
        conv = torch.nn.Conv2d(layer.cin, layer.cout, layer.k, padding=1 if layer.k == 3 else 0)
        sd[layer.name + ".weight"] = conv.weight.detach().clone()
        sd[layer.name + ".bias"] = conv.bias.detach().clone()
    return sd


class _Acts:
    """Per-batch-shape activation / gradient buffers (NHWC bf16) for B tiles of H x W."""

    def __init__(self, spec: UNetSpec, B: int, H: int, W: int, device):
        d = spec.depth
        chans = [spec.base_channels * 2 ** i for i in range(d + 1)]
        cp = [phys(c) for c in chans]
        e = lambda *shape: torch.empty(shape, dtype=torch.bfloat16, device=device)  # noqa: E731
        lv = lambda L, c, n=B: e(n, H >> L, W >> L, c)  # noqa: E731  (level-L tensor)
        self.B, self.H, self.W = B, H, W
        self.stem = None    # im2col buffer, only for float input / the unfused stem (lazy)
        self.images = None  # u8 input of the fused stem (its weight gradient re-reads it)
        self.a1 = [lv(i, cp[i]) for i in range(d)]
        self.a2 = [lv(i, cp[i]) for i in range(d)]
        self.pool = [lv(i + 1, cp[i]) for i in range(d)]
        self.b1, self.b2 = lv(d, cp[d]), lv(d, cp[d])
        self.hv = [lv(d - 1 - j, cp[d - 1 - j]) for j in range(d)]
        self.u1 = [lv(d - 1 - j, cp[d - 1 - j]) for j in range(d)]
        self.u2 = [lv(d - 1 - j, cp[d - 1 - j]) for j in range(d)]
        # backward scratch, per level: two dZ ping-pong buffers, the skip gradient, the
        # halving-conv output gradient (sub-pixel planes) and the pooled gradient
        self.dz_a = [lv(L, cp[L]) for L in range(d + 1)]
        self.dz_b = [lv(L, cp[L]) for L in range(d + 1)]
        self.dskip = [lv(L, cp[L]) for L in range(d)]
        self.dhv = [e(4, B, H >> (L + 1), W >> (L + 1), cp[L]) for L in range(d)]
        self.dpool = [lv(L + 1, cp[L]) for L in range(d)]
        # packed ReLU masks of the DoubleConv middle activations (a1, b1, u1): the forward writes
        # them, the backward's dgrad reads 4 B per 32 channels instead of the bf16 tensor
        bits = lambda L, c: torch.empty((c // 32, B * (H >> L) * (W >> L)), dtype=torch.int32, device=device)  # noqa: E731
        self.a1_bits = [bits(i, cp[i]) for i in range(d)]
        self.b1_bits = bits(d, cp[d])
        self.u1_bits = [bits(d - 1 - j, cp[d - 1 - j]) for j in range(d)]
        # ... and of the up-block outputs that feed the next halving conv (its dgrad's ReLU mask)
        self.u2_bits = [bits(d - 1 - j, cp[d - 1 - j]) for j in range(d - 1)]
        self.labels = torch.empty((B, H, W), dtype=torch.uint8, device=device)
        self.drop = {}  # block name -> fp32 [B][c_p] Dropout2d scales (train mode, p > 0)


class UNetEngine:
    """Parameters (flat fp32 master + grads + Adam moments + bf16 working copy) and the
    forward/backward schedule of one replica on one GPU."""

    def __init__(self, spec: UNetSpec, device=None):
        check_supported(spec)
        _native.require_cuda()
        self.spec = spec
        self.device = torch.device(device or "cuda")
        self.layers, self.by_name, self.numel = flat_layout(spec)
        f32 = dict(dtype=torch.float32, device=self.device)
        self.params = torch.zeros(self.numel, **f32)
        self.grads = torch.zeros(self.numel, **f32)
        self.exp_avg = torch.zeros(self.numel, **f32)
        self.exp_avg_sq = torch.zeros(self.numel, **f32)
        self.wbf16 = torch.zeros(self.numel, dtype=torch.bfloat16, device=self.device)
        self.halve_wc = {}
        for L in self.layers:
            if L.kind == "halve":
                self.halve_wc[L.name] = torch.zeros((L.cout_p, 9, L.cin_p), dtype=torch.bfloat16, device=self.device)
        self.acts = None
        self._acts_cache = {}
        # loss sum / correct count of the current step, shared by all shard shapes
        self.stats = torch.zeros(2, dtype=torch.float32, device=self.device)
        # optimizer step counter on the device: Adam bias corrections and dropout seeds read it,
        # so a captured CUDA graph of a whole train step replays correctly
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.training = True
        self.n_real_params = sum(L.cout * L.cin * L.k * L.k + L.cout for L in self.layers)

    # ---- views -----------------------------------------------------------------------
    def w(self, name, buf=None):
        L = self.by_name[name]
        buf = self.params if buf is None else buf
        return buf[L.w_off: L.w_off + L.w_numel].view(L.w_shape)

    def b(self, name, buf=None):
        L = self.by_name[name]
        buf = self.params if buf is None else buf
        return buf[L.b_off: L.b_off + L.cout_p]

    def wb16(self, name):
        return self.w(name, self.wbf16)

    # ---- state ---------------------------------------------------------------------------
    def load_state_dict(self, sd) -> None:
        host = torch.zeros(self.numel, dtype=torch.float32)
        for L in self.layers:
            w = sd[L.name + ".weight"].detach().to("cpu", torch.float32)
            bvec = sd[L.name + ".bias"].detach().to("cpu", torch.float32)
            if tuple(w.shape) != L.oihw_shape() or tuple(bvec.shape) != (L.cout,):
                raise ValueError(f"{L.name}: shape {tuple(w.shape)} does not match {L.oihw_shape()}")
            host[L.w_off: L.w_off + L.w_numel] = L.to_phys(w).reshape(-1)
            host[L.b_off: L.b_off + L.cout] = bvec
        self.params.copy_(host)
        self.refresh_working_weights()

    def state_dict(self) -> "OrderedDict[str, torch.Tensor]":
        host = self.params.detach().cpu()
        sd = OrderedDict()
        for L in self.layers:
            sd[L.name + ".weight"] = L.from_phys(host[L.w_off: L.w_off + L.w_numel].view(L.w_shape))
            sd[L.name + ".bias"] = host[L.b_off: L.b_off + L.cout].clone()
        return sd

    def grad_dict(self) -> "OrderedDict[str, torch.Tensor]":
        host = self.grads.detach().cpu()
        out = OrderedDict()
        for L in self.layers:
            out[L.name + ".weight"] = L.from_phys(host[L.w_off: L.w_off + L.w_numel].view(L.w_shape))
            out[L.name + ".bias"] = host[L.b_off: L.b_off + L.cout].clone()
        return out

    def refresh_working_weights(self) -> None:
        st = _native.stream_handle()
        _native.call("ice_cast_bf16", self.params.data_ptr(), self.numel, self.wbf16.data_ptr(), st)
        self.prep_halves()

    def prep_halves(self, stream=None) -> None:
        st = _native.stream_handle(stream)
        for name, wc in self.halve_wc.items():
            L = self.by_name[name]
            _native.call("ice_halve_prep", self.w(name).data_ptr(), L.cout_p, L.cin_p, wc.data_ptr(), st)

    # ---- buffers ---------------------------------------------------------------------------
    def ensure(self, B: int, H: int, W: int = None) -> _Acts:
        W = H if W is None else W
        check_tile(H, W, self.spec.depth)
        key = (B, H, W)
        if key not in self._acts_cache:
            if len(self._acts_cache) >= 4:  # ragged tails etc.: keep a few shapes resident
                self._acts_cache.pop(next(iter(self._acts_cache)))
                torch.cuda.empty_cache()
            acts = _Acts(self.spec, B, H, W, self.device)
            acts.stats = self.stats
            self._acts_cache[key] = acts
        self.acts = self._acts_cache[key]
        return self.acts

    def _drop_masks(self, A: _Acts, seed: int, train: bool) -> None:
        """Dropout2d scales for every DoubleConv output of this step, one launch."""
        A.drop = {}
        p = self.spec.dropout
        if not train or p == 0.0:
            return
        d = self.spec.depth
        blocks = [f"down.{i}" for i in range(d)] + ["bottleneck"] + [f"up.{j}" for j in range(d)]
        widths = [self.by_name[blk + ".block.2"].cout_p for blk in blocks]
        total = A.B * sum(widths)
        if getattr(A, "drop_buf", None) is None or A.drop_buf.numel() != total:
            A.drop_buf = torch.empty(total, dtype=torch.float32, device=self.device)
        _native.call("ice_dropout_scale", total, float(p), seed & (2 ** 63 - 1), self.step_dev.data_ptr(),
                     A.drop_buf.data_ptr(), _native.stream_handle())
        off = 0
        for blk, c in zip(blocks, widths):
            A.drop[blk] = A.drop_buf[off: off + A.B * c].view(A.B, c)
            off += A.B * c

    # ---- forward ------------------------------------------------------------------------
    def forward(self, images, train: bool, seed: int = 0, float_input: bool = False) -> _Acts:
        """images: u8 [B, H, W, 3] (or fp32 in [0,1] with float_input) device tensor."""
        spec = self.spec
        d = spec.depth
        B, H, W = images.shape[0], images.shape[1], images.shape[2]
        A = self.ensure(B, H, W)
        st = _native.stream_handle()
        fused = self.fused_stem and not float_input
        if fused:
            images = images.contiguous()
        A.images = images if fused else None
        if not fused:
            if A.stem is None:
                A.stem = torch.empty((B, H, W, 64), dtype=torch.bfloat16, device=self.device)
            fn = "ice_stem_im2col_f32" if float_input else "ice_stem_im2col"
            _native.call(fn, images.data_ptr(), B, H, W, A.stem.data_ptr(), st)
        self._drop_masks(A, seed, train)
        dr = A.drop.get
        x = A.stem
        for i in range(d):
            n0, n2 = f"down.{i}.block.0", f"down.{i}.block.2"
            if i == 0 and fused:  # stem straight from the u8 images (csrc/stem.cu)
                _native.call("ice_stem_fprop", _native.ptr(images), B, H, W, self.wb16(n0).data_ptr(),
                             self.b(n0).data_ptr(), A.a1[0].data_ptr(), A.a1_bits[0].data_ptr(), st)
            else:
                ops.conv_fprop(x, self.wb16(n0), self.b(n0), relu=True, ksize=1 if i == 0 else 3, out=A.a1[i],
                               relu_bits=A.a1_bits[i])
            ops.conv_fprop(A.a1[i], self.wb16(n2), self.b(n2), relu=True, drop=dr(f"down.{i}"), out=A.a2[i])
            a2 = A.a2[i]
            _native.call("ice_maxpool_fwd", a2.data_ptr(), B, a2.shape[1], a2.shape[2], a2.shape[3],
                         A.pool[i].data_ptr(), st)
            x = A.pool[i]
        ops.conv_fprop(x, self.wb16("bottleneck.block.0"), self.b("bottleneck.block.0"), relu=True, out=A.b1,
                       relu_bits=A.b1_bits)
        ops.conv_fprop(A.b1, self.wb16("bottleneck.block.2"), self.b("bottleneck.block.2"), relu=True,
                       drop=dr("bottleneck"), out=A.b2)
        x = A.b2
        for j in range(d):
            L = d - 1 - j
            hn = f"halve.{j}.conv"
            hl = self.by_name[hn]
            _native.call("ice_halve_fprop", x.data_ptr(), hl.cin_p, B, x.shape[1], x.shape[2],
                         self.halve_wc[hn].data_ptr(), self.b(hn).data_ptr(), hl.cout_p, A.hv[j].data_ptr(), st)
            n0, n2 = f"up.{j}.block.0", f"up.{j}.block.2"
            ops.conv_fprop(A.a2[L], self.wb16(n0), self.b(n0), x2=A.hv[j], relu=True, out=A.u1[j],
                           relu_bits=A.u1_bits[j])
            ops.conv_fprop(A.u1[j], self.wb16(n2), self.b(n2), relu=True, drop=dr(f"up.{j}"), out=A.u2[j],
                           relu_bits=A.u2_bits[j] if j < d - 1 else None)
            x = A.u2[j]
        return A

    def head(self, A: _Acts, labels, train: bool, grad_scale: float = 0.0, logits=None):
        """Cross-entropy head over the last activation; accumulates A.stats (loss sum,
        correct) and, in training, the head gradients and dZ of up.{d-1}.block.2."""
        d = self.spec.depth
        h = A.u2[d - 1]
        B, hw = h.shape[0], h.shape[1] * h.shape[2]
        st = _native.stream_handle()
        dz = A.dz_a[0] if train else None
        overwrite = train and self.grads_stale  # the head's gradients open the backward (see backward)
        if overwrite:
            _native.call("ice_grad_overwrite", 1)
        try:
            _native.call("ice_head_ce", h.data_ptr(), B * hw, hw, labels.data_ptr(),
                         self.w("out").data_ptr(), self.b("out").data_ptr(),
                         _native.ptr(A.drop.get(f"up.{d - 1}")) if train else None, float(grad_scale),
                         _native.ptr(dz), _native.ptr(self.w("out", self.grads)) if train else None,
                         _native.ptr(self.b("out", self.grads)) if train else None, A.stats.data_ptr(),
                         _native.ptr(logits),
                         _native.ptr(self.b(f"up.{d - 1}.block.2", self.grads)) if train else None, st)
        finally:
            if overwrite:
                _native.call("ice_grad_overwrite", 0)
        return dz

    # ---- backward -----------------------------------------------------------------------
    @staticmethod
    def _relu(ref, bits):
        """The ReLU mask a dgrad applies: the forward's packed bits (default) or the bf16 tensor."""
        return {"ref1": ref} if os.environ.get("ICE_NO_RELU_BITS") else {"bits1": bits}

    def _bias_grad(self, name, dz):
        L = self.by_name[name]
        rows = dz.numel() // dz.shape[-1]
        _native.call("ice_bias_grad", dz.data_ptr(), rows, dz.shape[-1], self.b(name, self.grads).data_ptr(),
                     _native.stream_handle())

    # Deferred finishing (ice_finish_defer): the ~50 fixed-order finishers of the weight / bias
    # gradient reductions run as ONE kernel per flush instead of one launch each (bit-identical
    # results); every backward call then gets its own scratch slice (bump mode).
    defer_finish = os.environ.get("ICE_DEFER_FINISH", "1") != "0"  # A/B switch, read once
    # The first conv straight from the u8 images (ice_stem_fprop / ice_stem_wgrad) instead of
    # a bf16 im2col buffer + GEMMs; float input always takes the im2col path.
    fused_stem = os.environ.get("ICE_FUSED_STEM", "1") != "0"  # A/B switch, read once
    side_flush = os.environ.get("ICE_SIDE_FLUSH", "1") != "0"  # A/B switch, read once
    # The fused Adam leaves the gradients unzeroed ("stale"); the next backward then runs in
    # gradient overwrite mode (every producer stores instead of adding): 4 B/param less for Adam
    # and no read of the old value by the split-0 weight-gradient epilogues.
    lazy_zero = os.environ.get("ICE_LAZY_ZERO", "1") != "0"  # A/B switch, read once
    grads_stale = False

    def backward(self, A: _Acts, dz, on_layer_done=None) -> None:
        """Accumulate parameter gradients into self.grads (dz: dZ of up.{d-1}.block.2).
        on_layer_done(name) fires after each layer's gradient is complete (DP buckets); a
        callback that reads gradients before backward returns calls flush_deferred() first."""
        overwrite = self.grads_stale  # the optimizer step left the gradients logically zero
        self.grads_stale = False
        if overwrite:
            _native.call("ice_grad_overwrite", 1)
        try:
            if self.defer_finish:
                self._backward_deferred(A, dz, on_layer_done)
            else:
                self._backward(A, dz, on_layer_done)
        finally:
            if overwrite:
                _native.call("ice_grad_overwrite", 0)

    def _backward_deferred(self, A: _Acts, dz, on_layer_done=None) -> None:
        _native.call("ice_finish_defer", 1)
        _native.scratch.begin_bump()
        self._side_events = []
        try:
            self._backward(A, dz, on_layer_done)
            self.flush_deferred()
            cur = torch.cuda.current_stream()
            for ev in self._side_events:  # finishers flushed early on the side stream
                cur.wait_event(ev)
        finally:
            self._side_events = []
            _native.call("ice_finish_defer", 0)
            _native.scratch.end_bump()

    def flush_deferred(self, stream=None) -> None:
        """Run the gradient finishers recorded so far (one launch; no-op when none).  On the
        current stream it also joins the finishers flushed early on the side stream, so every
        gradient is complete after it in stream order (the bucketer relies on that)."""
        if stream is None:
            cur = torch.cuda.current_stream()
            for ev in getattr(self, "_side_events", ()):
                cur.wait_event(ev)
        _native.call("ice_finish_flush", _native.stream_handle(stream))

    def _flush_side(self) -> None:
        """Flush the finishers recorded so far on a side stream, so their (HBM-bound) slice
        sums overlap the rest of the (tensor-bound) backward; backward() joins it before it
        returns.  Their gradients are complete once their producers ran (ordered by the event);
        no later kernel of the backward touches them, and bump-mode scratch keeps their
        partial sums."""
        if not self.defer_finish or not self.grads.is_cuda or not self.side_flush:
            return
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        self._side.wait_event(ev)
        self.flush_deferred(self._side)
        done = torch.cuda.Event()
        done.record(self._side)
        self._side_events.append(done)

    def _backward(self, A: _Acts, dz, on_layer_done=None) -> None:
        d = self.spec.depth
        B = A.B
        st = _native.stream_handle()
        G = self.grads
        done = on_layer_done or (lambda name: None)
        done("out")
        for j in reversed(range(d)):
            L = d - 1 - j
            n0, n2, hn = f"up.{j}.block.0", f"up.{j}.block.2", f"halve.{j}.conv"
            # up.j.block.2 : u1 -> u2
            ops.conv_wgrad(A.u1[j], dz, self.w(n2, G))
            dz1 = A.dz_b[L]
            ops.conv_dgrad(dz, self.wb16(n2), A.u1[j].shape[3], out1=dz1, **self._relu(A.u1[j], A.u1_bits[j]), db1=self.b(n0, G))
            done(n2)
            # up.j.block.0 : cat(skip, hv) -> u1
            ops.conv_wgrad(A.a2[L], dz1, self.w(n0, G), x2=A.hv[j])
            c = A.a2[L].shape[3]
            _native.call("ice_conv_dgrad", dz1.data_ptr(), dz1.shape[3], B, dz1.shape[1], dz1.shape[2], 3,
                         self.wb16(n0).data_ptr(), c, c, A.dskip[L].data_ptr(), None, None, None,
                         A.dhv[L].data_ptr(), None, None, None, 1, None, self.b(hn, G).data_ptr(), None, st)
            done(n0)
            # halve.j : x_prev -> hv
            xprev = A.b2 if j == 0 else A.u2[j - 1]
            hl = self.by_name[hn]
            s = xprev.shape[1]
            _native.call("ice_halve_wgrad", xprev.data_ptr(), hl.cin_p, A.dhv[L].data_ptr(), hl.cout_p, B, s, s,
                         self.w(hn, G).data_ptr(), st)
            dz = A.dz_a[L + 1]
            drop_prev = A.drop.get("bottleneck" if j == 0 else f"up.{j - 1}")
            prev_name = "bottleneck.block.2" if j == 0 else f"up.{j - 1}.block.2"
            bits_prev = A.u2_bits[j - 1] if j > 0 else None  # (the bottleneck output keeps split-K: no bits)
            _native.call("ice_halve_dgrad", A.dhv[L].data_ptr(), hl.cout_p, B, s, s, self.halve_wc[hn].data_ptr(),
                         hl.cin_p, dz.data_ptr(), xprev.data_ptr(), _native.ptr(bits_prev), _native.ptr(drop_prev),
                         self.b(prev_name, G).data_ptr(), st)
            done(hn)
        self._flush_side()  # the up path's finishers overlap the bottleneck and down path
        # bottleneck
        ops.conv_wgrad(A.b1, dz, self.w("bottleneck.block.2", G))
        dz1 = A.dz_b[d]
        ops.conv_dgrad(dz, self.wb16("bottleneck.block.2"), A.b1.shape[3], out1=dz1, **self._relu(A.b1, A.b1_bits),
                       db1=self.b("bottleneck.block.0", G))
        done("bottleneck.block.2")
        ops.conv_wgrad(A.pool[d - 1], dz1, self.w("bottleneck.block.0", G))
        ops.conv_dgrad(dz1, self.wb16("bottleneck.block.0"), A.pool[d - 1].shape[3], out1=A.dpool[d - 1])
        done("bottleneck.block.0")
        # down path
        for i in reversed(range(d)):
            n0, n2 = f"down.{i}.block.0", f"down.{i}.block.2"
            a2 = A.a2[i]
            dz2 = A.dz_a[i]
            _native.call("ice_maxpool_bwd", a2.data_ptr(), A.dpool[i].data_ptr(), A.dskip[i].data_ptr(),
                         _native.ptr(A.drop.get(f"down.{i}")), B, a2.shape[1], a2.shape[2], a2.shape[3],
                         dz2.data_ptr(), self.b(n2, G).data_ptr(), st)
            ops.conv_wgrad(A.a1[i], dz2, self.w(n2, G))
            dz1 = A.dz_b[i]
            ops.conv_dgrad(dz2, self.wb16(n2), A.a1[i].shape[3], out1=dz1, **self._relu(A.a1[i], A.a1_bits[i]), db1=self.b(n0, G))
            done(n2)
            if i == 0 and A.images is not None:
                _native.call("ice_stem_wgrad", A.images.data_ptr(), B, A.H, A.W, dz1.data_ptr(),
                             self.w(n0, G).data_ptr(), st)
            elif i == 0:
                ops.conv_wgrad(A.stem, dz1, self.w(n0, G), ksize=1)
            else:
                ops.conv_wgrad(A.pool[i - 1], dz1, self.w(n0, G))
            if i > 0:
                ops.conv_dgrad(dz1, self.wb16(n0), A.pool[i - 1].shape[3], out1=A.dpool[i - 1])
            done(n0)

    # ---- optimizer ------------------------------------------------------------------------
    def advance_step(self, stream=None) -> None:
        _native.call("ice_counter_add", self.step_dev.data_ptr(), 1, _native.stream_handle(stream))

    def adam(self, step: int, lr: float, betas=(0.9, 0.999), eps: float = 1e-8) -> None:
        self.advance_step()
        self.adam_slice(0, self.numel, step, lr, betas, eps)
        self.prep_halves()

    def adam_slice(self, start: int, stop: int, step: int, lr: float, betas=(0.9, 0.999), eps: float = 1e-8,
                   stream=None) -> None:
        """Fused Adam on flat elements [start, stop) (a gradient bucket); 4-element aligned.
        With lazy_zero the gradients are not zeroed: they become logically zero ("stale") and
        the next backward writes them in overwrite mode (ice_grad_overwrite)."""
        st = _native.stream_handle(stream)
        off4, off2 = start * 4, start * 2
        _native.call("ice_adam", self.params.data_ptr() + off4, self.grads.data_ptr() + off4,
                     self.exp_avg.data_ptr() + off4, self.exp_avg_sq.data_ptr() + off4, stop - start, int(step),
                     self.step_dev.data_ptr(), float(lr), float(betas[0]), float(betas[1]), float(eps),
                     0 if self.lazy_zero else 1, self.wbf16.data_ptr() + off2, st)
        if self.lazy_zero:
            self.grads_stale = True

    def zero_grad(self) -> None:
        _native.call("ice_fill_f32", self.grads.data_ptr(), self.numel, 0.0, _native.stream_handle())
        self.grads_stale = False

    def layer_slice(self, name):
        """(start, stop) of a layer's weight+bias in the flat buffers."""
        L = self.by_name[name]
        return L.w_off, L.b_off + L.cout_p


class ParamList(list):
    """UNet.parameters(): one torch.nn.Parameter per reference parameter (state_dict order),
    each a VIEW of the engine's flat fp32 master buffer in its physical layout (KRSC, channels
    padded to 64 -- padded entries are zero and get zero gradients), with `.grad` a view of the
    flat gradient buffer.  So any torch optimizer can step them in place
    (`torch.optim.SGD(m.parameters(), lr)` as in the reference's own tests); synchronized_step
    then refreshes the bf16 working weights.  `.engine` lets the fused Adam find its buffers."""

    def __init__(self, engine):
        super().__init__()
        self.engine = engine
        for L in engine.layers:
            for view, grad in ((engine.w(L.name), engine.w(L.name, engine.grads)),
                               (engine.b(L.name), engine.b(L.name, engine.grads))):
                prm = torch.nn.Parameter(view, requires_grad=True)
                prm.grad = grad
                self.append(prm)
        self._grads = [p.grad for p in self]

    def attach_grads(self) -> None:
        """Re-point every .grad at its flat-buffer view (after a zero_grad(set_to_none=True))."""
        for prm, g in zip(self, self._grads):
            prm.grad = g


class UNet:
    """Drop-in for icetrain.model.UNet (model.py:91-137) running on the B200 engine."""

    def __init__(self, spec: UNetSpec, device=None) -> None:
        self.spec = spec
        check_supported(spec)
        params = init_reference_params(spec)  # same RNG draws as the reference constructor
        self.engine = UNetEngine(spec, device)
        self.engine.load_state_dict(params)
        self.training = True
        self._params = None

    # nn.Module-like surface
    def train(self, mode: bool = True):
        self.training = mode
        return self

    def eval(self):
        return self.train(False)

    def state_dict(self):
        return self.engine.state_dict()

    def load_state_dict(self, sd):
        missing = [L.name + s for L in self.engine.layers for s in (".weight", ".bias")
                   if L.name + s not in sd]
        unexpected = [k for k in sd if k not in {L.name + s for L in self.engine.layers
                                                 for s in (".weight", ".bias")}]
        if missing or unexpected:
            raise RuntimeError(f"Error(s) in loading state_dict for UNet: missing keys {missing}, "
                               f"unexpected keys {unexpected}")
        self.engine.load_state_dict(sd)

    def parameters(self) -> ParamList:
        if self._params is None:
            self._params = ParamList(self.engine)
        return self._params

    def zero_grad(self, set_to_none: bool = True) -> None:
        """nn.Module.zero_grad: the engine accumulates into one flat buffer, which is zeroed."""
        self.engine.zero_grad()

    def named_parameters(self):
        names = [L.name + s for L in self.engine.layers for s in (".weight", ".bias")]
        return list(zip(names, self.parameters()))

    def conv_layer_count(self) -> int:
        return len(self.engine.layers)

    def _check(self, x):
        if x.ndim != 4 or x.shape[1] != self.spec.in_channels:
            raise ValueError(f"expected (n, {self.spec.in_channels}, h, w) input, got {tuple(x.shape)}")
        check_tile(x.shape[2], x.shape[3], self.spec.depth)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """Class logits (n, classes, h, w) fp32, on x's device (model.py:111-130).  In train mode
        (the default, as an nn.Module) Dropout2d drops whole (sample, channel) planes with a
        mask seeded from torch's default generator (so torch.manual_seed fixes it); eval()
        makes the forward deterministic, as the reference's model.eval()."""
        self._check(x)
        dev = x.device
        xin = x.detach().to(self.engine.device, torch.float32).permute(0, 2, 3, 1).contiguous()
        n, h, w = xin.shape[0], xin.shape[1], xin.shape[2]
        drop = self.training and self.spec.dropout > 0
        seed = int(torch.randint(0, 2 ** 62, (1,)).item()) if drop else 0
        A = self.engine.forward(xin, train=drop, seed=seed, float_input=True)
        logits = torch.empty((n, h, w, 3), dtype=torch.float32, device=self.engine.device)
        labels = torch.zeros((n, h, w), dtype=torch.uint8, device=self.engine.device)
        A.stats.zero_()
        self.engine.head(A, labels, train=False, logits=logits)
        return logits.permute(0, 3, 1, 2).contiguous().to(dev)

    __call__ = forward

    def probabilities(self, x: torch.Tensor) -> torch.Tensor:
        return torch.softmax(self.forward(x), dim=1)
