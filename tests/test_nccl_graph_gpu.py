"""The NCCL data-parallel step inside a CUDA graph, on one GPU: a 1-rank NCCL group with the
bucketed all-reduce forced on (GradBucketer(force_collective=True)) exercises the same
capture path as N > 1 -- collectives on the comm stream, Adam on the opt stream, all in one
graph -- and must equal eager steps bit for bit, with fp32 or bf16 on the wire."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "unet_golden.pt")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, port, wire, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec
    from paper_2403_13135_b200.icetrain.train import GradBucketer, GraphedStep, device_step
    g = torch.load(GOLD)["desk"]
    spec = UNetSpec(**{**g["spec"], "dropout": 0.1})
    x, y = g["images"].cuda(), g["labels"].cuda()
    runs = []
    for graphed in (False, True):
        torch.manual_seed(0)
        m = UNet(spec)
        opt = Adam(m.parameters())
        b = GradBucketer(m.engine, bucket_bytes=1 << 18, optimizer=opt, force_collective=True,
                         comm_dtype=torch.bfloat16 if wire == "bf16" else None)
        if graphed:
            step = GraphedStep(m, opt, x, y, len(x), b, warmup=2)
            for _ in range(3):
                step(x, y)
        else:
            for _ in range(5):
                device_step(m, opt, x, y, len(x), b)
        torch.cuda.synchronize()
        runs.append(m.engine.params.cpu())
    out[wire] = (bool(torch.equal(runs[0], runs[1])), len(b.buckets))
    dist.destroy_process_group()


@pytest.mark.parametrize("wire", ["fp32", "bf16"])
def test_nccl_bucketed_step_captured_in_a_graph(wire):
    out = mp.Manager().dict()
    mp.spawn(_run, args=(_port(), wire, out), nprocs=1, join=True)
    same, nbuckets = out[wire]
    assert nbuckets > 3 and same
