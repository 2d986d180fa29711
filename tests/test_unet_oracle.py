"""Pin the CPU U-Net oracle (oracle/unet_ref.py) and the product's seeded init / layout
conversions to vectors produced by the reference trainer (tests/golden/unet_golden.pt)."""
import hashlib
import os

import pytest
import torch

from oracle import unet_ref
from paper_2403_13135_b200.icetrain.model import UNetSpec, build_layers, init_reference_params

GOLD = torch.load(os.path.join(os.path.dirname(__file__), "golden", "unet_golden.pt"))


def digest(sd):
    h = hashlib.sha256()
    for k, v in sd.items():
        h.update(k.encode())
        h.update(v.detach().contiguous().numpy().tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["desk", "deep"])
def test_product_init_equals_reference_init(name):
    spec = UNetSpec(**GOLD[name]["spec"])
    torch.manual_seed(0)
    assert digest(init_reference_params(spec)) == GOLD[name]["init_digest"]


@pytest.mark.parametrize("name", ["desk", "deep"])
def test_oracle_forward_backward_matches_reference(name):
    g = GOLD[name]
    spec = UNetSpec(**g["spec"])
    torch.manual_seed(0)
    model = unet_ref.RefUNet(spec)
    assert digest(model.state_dict()) == g["init_digest"]
    x = unet_ref.images_to_input(g["images"])
    loss, logits, grads = unet_ref.loss_and_grads(model, x, g["labels"].long())
    assert torch.allclose(logits, g["logits"], rtol=1e-5, atol=1e-6)
    assert abs(loss - g["loss"]) < 1e-6
    for k, v in grads.items():
        ref = g["grads"][k]
        if isinstance(ref, dict):
            assert abs(float(v.norm()) - ref["norm"]) <= 1e-5 * max(ref["norm"], 1e-12) + 1e-12
            assert torch.allclose(v.reshape(-1)[:256], ref["head"], rtol=1e-4, atol=1e-9)
        else:
            assert torch.allclose(v, ref, rtol=1e-4, atol=1e-9), k


def test_oracle_synchronized_steps_match_reference():
    g = GOLD["desk"]
    spec = UNetSpec(**g["spec"])
    torch.manual_seed(0)
    m0 = unet_ref.RefUNet(spec)
    m1 = unet_ref.RefUNet(spec)
    m1.load_state_dict(m0.state_dict())
    opts = [torch.optim.Adam(m.parameters(), lr=1e-3) for m in (m0, m1)]
    x = unet_ref.images_to_input(g["images"])
    y = g["labels"].long()
    losses = []
    for step in range(5):
        perm = torch.randperm(len(x), generator=torch.Generator().manual_seed(step))
        shards = [(x[p], y[p]) for p in torch.tensor_split(perm, 2)]
        losses.append(unet_ref.synchronized_step([m0, m1], opts, shards)[0])
    assert losses == pytest.approx(g["step_losses"], rel=1e-5)
    for k, v in m0.state_dict().items():
        assert torch.allclose(v, g["final_state"][k], rtol=1e-4, atol=1e-7), k
        assert torch.equal(v, m1.state_dict()[k])  # replicas never drift


@pytest.mark.parametrize("spec", [UNetSpec(input_size=32, base_channels=8, depth=2),
                                  UNetSpec(), UNetSpec(input_size=64, base_channels=16, depth=3)])
def test_layout_round_trip(spec):
    torch.manual_seed(1)
    sd = init_reference_params(spec)
    layers, _ = build_layers(spec)
    assert len(layers) == spec.conv_layers
    for L in layers:
        w = sd[L.name + ".weight"]
        assert tuple(w.shape) == L.oihw_shape()
        p = L.to_phys(w)
        assert torch.equal(L.from_phys(p), w)
        assert float(p.abs().sum()) == pytest.approx(float(w.abs().sum()), rel=1e-6)


def test_paper_spec_parameter_count():
    spec = UNetSpec()
    sd = init_reference_params(spec)
    assert sum(v.numel() for v in sd.values()) == 124_362_307
    assert len(sd) == 56


def test_oracle_trajectory_matches_reference():
    """The oracle port reproduces the reference's 200-step loss trajectory (first 20 steps
    checked here to keep the CPU suite fast)."""
    from tests.golden.trajectory_data import SEED, batch_order, corpus
    gold = torch.load(os.path.join(os.path.dirname(__file__), "golden", "unet_trajectory.pt"))
    spec = UNetSpec(**gold["spec"])
    x_u8, y = corpus()
    x = unet_ref.images_to_input(x_u8)
    yt = torch.from_numpy(y)
    torch.manual_seed(SEED)
    model = unet_ref.RefUNet(spec)
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    for step, idx in enumerate(batch_order()[:20]):
        loss, _ = unet_ref.synchronized_step([model], [opt], [(x[idx], yt[idx])])
        assert loss == pytest.approx(gold["losses"][step], rel=1e-4), step
