"""A CUDA-graph-captured train step replays as real consecutive steps: same parameters as
eager steps (Adam bias corrections and dropout seeds come from the device step counter)."""
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "unet_golden.pt")


@pytest.mark.parametrize("dropout", [0.0, 0.1])
def test_graph_replay_equals_eager(dropout):
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec
    from paper_2403_13135_b200.icetrain.train import GradBucketer, GraphedStep, device_step
    g = torch.load(GOLD)["desk"]
    spec = UNetSpec(**{**g["spec"], "dropout": dropout})
    x = g["images"].cuda()
    y = g["labels"].cuda()
    runs = []
    for graphed in (False, True):
        torch.manual_seed(0)
        m = UNet(spec)
        opt = Adam(m.parameters())
        b = GradBucketer(m.engine, bucket_bytes=1 << 16, optimizer=opt)
        if graphed:
            step = GraphedStep(m, opt, x, y, len(x), b, warmup=2)  # warm-up runs 2 real steps
            for _ in range(3):
                step(x, y)
        else:
            for _ in range(5):
                device_step(m, opt, x, y, len(x), b)
        torch.cuda.synchronize()
        assert opt.step_count == 5
        assert int(m.engine.step_dev.item()) == 5
        runs.append(m.engine.params.clone())
    # every fp32 reduction is fixed-order (no atomics), so replays equal eager steps bit for bit
    assert torch.equal(runs[0], runs[1])

