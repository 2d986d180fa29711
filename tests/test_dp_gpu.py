"""Two ranks on one GPU (gloo over CUDA tensors, since NCCL needs distinct GPUs): the
bucketed, overlapped DP step equals the single-process step on the union batch, and the
ranks stay bit-identical (trainer/tests/test_acceptance.py:53-87)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "unet_golden.pt")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec, synchronized_step
    from paper_2403_13135_b200.icetrain.train import rank_shards
    g = torch.load(GOLD)["desk"]
    spec = UNetSpec(**g["spec"])
    torch.manual_seed(0)
    m = UNet(spec)
    opt = Adam(m.parameters())
    losses = []
    for step in range(3):
        union = torch.randperm(len(g["images"]), generator=torch.Generator().manual_seed(step))
        (p,) = rank_shards(union[:3] if step == 2 else union, world, rank, 1)  # ragged last step
        losses.append(synchronized_step([m], [opt], [(g["images"][p], g["labels"][p])]))
    out[rank] = (losses, m.engine.params.cpu())
    dist.destroy_process_group()


def test_two_ranks_equal_union_batch_step():
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec, synchronized_step
    out = mp.Manager().dict()
    mp.spawn(_rank, args=(2, _port(), out), nprocs=2, join=True)
    g = torch.load(GOLD)["desk"]
    spec = UNetSpec(**g["spec"])
    torch.manual_seed(0)
    m = UNet(spec)
    opt = Adam(m.parameters())
    ref = []
    for step in range(3):
        union = torch.randperm(len(g["images"]), generator=torch.Generator().manual_seed(step))
        union = union[:3] if step == 2 else union
        ref.append(synchronized_step([m], [opt], [(g["images"][union], g["labels"][union])]))
    (l0, p0), (l1, p1) = out[0], out[1]
    assert torch.equal(p0, p1)  # replica drift == 0.0
    for (a, na), (b, nb), (c, nc) in zip(l0, l1, ref):
        assert na == nb == nc
        assert a == b
        assert abs(a - c) <= 1e-5 * abs(c) + 1e-6
    rel = float((p0 - m.engine.params.cpu()).norm() / m.engine.params.cpu().norm())
    assert rel < 1e-5
