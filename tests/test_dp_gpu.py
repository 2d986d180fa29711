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


def _al_rank(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_13135_b200 import icelabel as il
    from tests.fixtures import synth
    tiles = torch.from_numpy(__import__("numpy").stack([t for t, _ in synth.corpus(23, 7, 0.5)]))
    res, (lo, hi), totals = il.autolabel_sharded(tiles)  # host corpus: each rank copies its shard
    out[rank] = (lo, hi, res["label"].cpu() if res is not None else None, totals.cpu())
    dist.destroy_process_group()


def test_autolabel_sharded_two_ranks():
    """BASELINE configs[3] layout on two ranks (one GPU, gloo): contiguous tile shards with no
    data-path collective, the per-class / masked totals summed by ONE small all-reduce; the
    shards' labels and the totals equal the single-process labeling of the whole corpus."""
    import numpy as np
    from paper_2403_13135_b200 import icelabel as il
    from tests.fixtures import synth
    out = mp.Manager().dict()
    mp.spawn(_al_rank, args=(2, _port(), out), nprocs=2, join=True)
    tiles = torch.from_numpy(np.stack([t for t, _ in synth.corpus(23, 7, 0.5)])).cuda()
    ref = il.autolabel(tiles)
    (lo0, hi0, lab0, tot0), (lo1, hi1, lab1, tot1) = out[0], out[1]
    assert (lo0, hi0, lo1, hi1) == (0, 3, 3, 7)  # shard_bounds(7, 2, r)
    assert torch.equal(torch.cat([lab0, lab1]), ref["label"].cpu())
    assert torch.equal(tot0, tot1)
    want = torch.tensor(ref["counts"].to(torch.int64).sum(0).tolist() + [int(ref["affected"].sum()),
                                                                         int((ref["unmatched"] >= 0).sum())])
    assert torch.equal(tot0, want)
