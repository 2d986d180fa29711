"""Data-parallel host logic at world size 2 on CPU (gloo): bucket planning, the bucketed
SUM all-reduce of pre-scaled gradients == the reference's shard-size-weighted average
(train.py:108-117), and the union-batch sharding (train.py:161-163)."""
import os
import socket
from types import SimpleNamespace

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_13135_b200.icetrain.model import UNetSpec, flat_layout, readiness_order
from paper_2403_13135_b200.icetrain.train import GradBucketer, plan_buckets, rank_shards

SPEC = UNetSpec(input_size=64, base_channels=8, depth=3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, counts, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, _, numel = flat_layout(SPEC)
    total = sum(counts)
    torch.manual_seed(100 + rank)
    local_mean_grad = torch.randn(numel)            # d(mean loss over this shard)/dθ
    grads = local_mean_grad * counts[rank] / total   # what the CE head pre-scaling produces
    eng = SimpleNamespace(spec=SPEC, grads=grads.clone())
    b = GradBucketer(eng, bucket_bytes=4096)
    for name in readiness_order(SPEC):
        b.on_layer_done(name)
    b.finish()
    out[rank] = (local_mean_grad, eng.grads)
    dist.destroy_process_group()


@pytest.mark.parametrize("counts", [(3, 5), (4, 0)])
def test_bucketed_allreduce_is_the_weighted_average(counts):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, counts, out), nprocs=2, join=True)
    g0, r0 = out[0]
    g1, r1 = out[1]
    want = (counts[0] * g0 + counts[1] * g1) / sum(counts)  # train.py:111-114
    assert torch.equal(r0, r1)                                # identical on every rank
    assert torch.allclose(r0, want, rtol=1e-6, atol=1e-7)


def test_buckets_partition_the_flat_buffer():
    for spec in (SPEC, UNetSpec()):
        _, by_name, numel = flat_layout(spec)
        for size in (4096, 64 << 20):
            b = plan_buckets(spec, size)
            assert b[0][0] == 0 and b[-1][1] == numel
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
            order = readiness_order(spec)
            assert [order.index(x[2]) for x in b] == sorted(order.index(x[2]) for x in b)


def test_rank_shards_match_reference_tensor_split():
    union = torch.randperm(70)
    for world, local in ((2, 1), (4, 1), (1, 3), (2, 2)):
        n = world * local
        ref = torch.tensor_split(union, n)
        got = [p for r in range(world) for p in rank_shards(union, n, r, local)]
        assert all(torch.equal(a, b) for a, b in zip(ref, got))
    # ragged final union batch and empty shards (trainer/tests/test_train.py:102-130)
    tail = union[:3]
    shards = [p for r in range(4) for p in rank_shards(tail, 4, r, 1)]
    assert [len(p) for p in shards] == [1, 1, 1, 0]


def test_autolabel_shards_cover_the_corpus_once():
    """Tile sharding of the auto-labeler: contiguous, disjoint, complete."""
    from paper_2403_13135_b200.icelabel import shard_bounds
    for n in (0, 1, 7, 100, 100000):
        for world in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _count_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_13135_b200.icelabel import shard_bounds
    n = 11
    per_tile = torch.arange(n * 5, dtype=torch.int64).view(n, 5)  # stand-in per-tile counts
    lo, hi = shard_bounds(n, world, rank)
    totals = per_tile[lo:hi].sum(0)
    dist.all_reduce(totals)  # the one collective autolabel_sharded issues
    out[rank] = totals
    dist.destroy_process_group()


def test_autolabel_sharded_totals_allreduce_gloo():
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_count_worker, args=(2, port, out), nprocs=2, join=True)
    want = torch.arange(55, dtype=torch.int64).view(11, 5).sum(0)
    assert torch.equal(out[0], want) and torch.equal(out[1], want)
