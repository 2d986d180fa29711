"""The training-loop API on the B200 path (reference: pkg/trainer/src/icetrain/train.py:123-234,
pkg/trainer/tests/test_train.py), and run-to-run determinism of the train step.

Every fp32 reduction on the training path is fixed-order (no atomics: see
paper_2403_13135_b200/csrc/reduce.cuh), so the reference's "fixed seed, reproducible history"
contract holds bit for bit: same seed -> identical history, identical weights.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2403_13135_b200.icetrain import (TABLE_COLUMNS, Adam, TrainConfig, UNet, UNetSpec,  # noqa: E402
                                            synchronized_step, table_csv, throughput_table, train,
                                            train_distributed)

pytestmark = pytest.mark.gpu

SMALL_SPEC = UNetSpec(input_size=32, depth=3, base_channels=4, dropout=0.0)


def small_pairs(count=10, size=32, seed=0):
    """pkg/trainer/tests/test_train.py:16-20."""
    rng = np.random.default_rng(seed)
    return [(rng.integers(0, 256, (size, size, 3)).astype(np.uint8),
             rng.integers(0, 3, (size, size)).astype(np.int64))
            for _ in range(count)]


def test_loss_drops_on_small_corpus():
    result = train(small_pairs(), SMALL_SPEC, TrainConfig(batch_size=4, epochs=5))
    losses = [h["train_loss"] for h in result.history]
    assert len(losses) == 5
    assert losses[-1] < losses[0]


def test_history_records_validation_metrics():
    result = train(small_pairs(), SMALL_SPEC, TrainConfig(batch_size=4, epochs=1))
    assert set(result.history[0]) == {"epoch", "train_loss", "train_acc", "val_loss", "val_acc"}


def test_same_seed_reproduces_history_exactly():
    """test_train.py:71-75: bit-identical histories (no fp32 atomics on the path)."""
    config = TrainConfig(batch_size=4, epochs=2, seed=9)
    a = train(small_pairs(), SMALL_SPEC, config)
    b = train(small_pairs(), SMALL_SPEC, config)
    assert a.history == b.history
    assert torch.equal(a.model.engine.params, b.model.engine.params)


def test_distributed_single_device_matches_train():
    config = TrainConfig(batch_size=4, epochs=2, seed=3)
    lone = train(small_pairs(), SMALL_SPEC, config)
    result, row = train_distributed(small_pairs(), SMALL_SPEC, config, devices=1)
    assert result.history == lone.history
    assert row["devices"] == 1
    assert set(row) == set(TABLE_COLUMNS)


def test_two_local_replicas_match_union_training():
    """train_distributed(devices=2) on one GPU: two lockstep replicas, union batch 2 x 4.
    Same data order as a single replica at batch 8, so the losses agree to rounding."""
    pairs = small_pairs(18, seed=4)
    a, row_a = train_distributed(pairs, SMALL_SPEC, TrainConfig(batch_size=4, epochs=2, seed=5), devices=2)
    b, _ = train_distributed(pairs, SMALL_SPEC, TrainConfig(batch_size=8, epochs=2, seed=5), devices=1)
    assert row_a["devices"] == 2
    for ha, hb in zip(a.history, b.history):
        assert abs(ha["train_loss"] - hb["train_loss"]) <= 1e-4 * abs(hb["train_loss"])


def test_throughput_table_schema_and_speedups():
    cfg = TrainConfig(batch_size=4, epochs=1, seed=0)
    rows = throughput_table(small_pairs(12), SMALL_SPEC, cfg, device_counts=(1, 2))
    assert [r["devices"] for r in rows] == [1, 2]
    assert all(set(r) == set(TABLE_COLUMNS) for r in rows)
    assert rows[0]["speedup"] == 1.0
    assert rows[1]["speedup"] == round(rows[1]["samples_per_s"] / rows[0]["samples_per_s"], 3)
    csv = table_csv(rows).splitlines()
    assert csv[0] == ",".join(TABLE_COLUMNS) and len(csv) == 3
    with pytest.raises(ValueError, match="device_counts"):
        throughput_table(small_pairs(4), SMALL_SPEC, cfg, device_counts=())


def test_paper_spec_step_is_bit_reproducible():
    """Paper U-Net (124.4M params) at 256^2, batch 8: two train steps from the same weights
    give bit-identical gradients, loss and updated weights.  This batch exercises every
    fixed-order reduction: split-K weight-gradient slices (levels 0-4), per-CTA bias-gradient
    rows of the fused dgrad epilogues, the split fprop/dgrad finishers of the deep levels, the
    max-pool and head partial rows."""
    from paper_2403_13135_b200.icetrain.train import device_step
    spec = UNetSpec(dropout=0.1)
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.integers(0, 256, (8, 256, 256, 3), dtype=np.uint8)).cuda()
    y = torch.from_numpy(rng.integers(0, 3, (8, 256, 256), dtype=np.uint8)).cuda()
    out = []
    for _ in range(2):
        torch.manual_seed(0)
        m = UNet(spec)
        opt = Adam(m.parameters())
        eng = m.engine
        eng.stats.zero_()
        A = eng.forward(x, train=True, seed=5)
        dz = eng.head(A, y, train=True, grad_scale=1.0 / y.numel())
        eng.backward(A, dz)
        grads = eng.grads.clone()
        stats = eng.stats.clone()
        device_step(m, opt, x, y, 8)
        torch.cuda.synchronize()
        out.append((grads, stats, eng.params.clone()))
    (g0, s0, p0), (g1, s1, p1) = out
    assert torch.equal(s0, s1)
    assert torch.equal(g0, g1)
    assert torch.equal(p0, p1)
    assert float(g0.abs().sum()) > 0


def test_deferred_finishers_match_immediate_bit_for_bit():
    """ice_finish_defer / ice_finish_flush: the gradient finishers of a paper-spec backward run
    as one batched launch with the same partitions and summation orders, so the gradients are
    bit-identical to launching each finisher on its own -- with far fewer launches."""
    from paper_2403_13135_b200 import _native
    spec = UNetSpec(dropout=0.1)
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.integers(0, 256, (8, 256, 256, 3), dtype=np.uint8)).cuda()
    y = torch.from_numpy(rng.integers(0, 3, (8, 256, 256), dtype=np.uint8)).cuda()
    torch.manual_seed(0)
    eng = UNet(spec).engine
    res = {}
    for defer in (False, True, True):
        eng.defer_finish = defer
        eng.grads.zero_()
        A = eng.forward(x, train=True, seed=5)
        dz = eng.head(A, y, train=True, grad_scale=1.0 / y.numel())
        torch.cuda.synchronize()
        k0 = _native.kernel_launches()
        eng.backward(A, dz)
        torch.cuda.synchronize()
        res.setdefault(defer, []).append((eng.grads.clone(), _native.kernel_launches() - k0))
    eng.defer_finish = True
    (g_imm, n_imm), = res[False]
    (g_def, n_def), (g_def2, _) = res[True]
    assert torch.equal(g_imm, g_def) and torch.equal(g_def, g_def2)
    assert n_def <= n_imm - 30, (n_def, n_imm)


def test_synchronized_step_same_inputs_same_bits():
    """synchronized_step twice from the same state (two lockstep replicas, ragged shards)."""
    spec = UNetSpec(input_size=64, base_channels=16, depth=4, dropout=0.0)
    pairs = small_pairs(7, size=64, seed=2)
    x = torch.from_numpy(np.stack([p[0] for p in pairs]))
    y = torch.from_numpy(np.stack([p[1] for p in pairs]))
    res = []
    for _ in range(2):
        torch.manual_seed(1)
        ms = [UNet(spec), UNet(spec)]
        ms[1].load_state_dict(ms[0].state_dict())
        opts = [Adam(m.parameters()) for m in ms]
        losses = [synchronized_step(ms, opts, [(x[:4], y[:4]), (x[4:], y[4:])])[0] for _ in range(3)]
        res.append((losses, ms[0].engine.params.clone(), ms[1].engine.params.clone()))
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][1], res[0][2])  # replica drift == 0


def _clone_replicas(spec, count, seed=0):
    """pkg/trainer/tests/test_train.py:23-33 verbatim: torch.optim.SGD over model.parameters()."""
    torch.manual_seed(seed)
    first = UNet(spec)
    models = [first]
    for _ in range(count - 1):
        twin = UNet(spec)
        twin.load_state_dict(first.state_dict())
        models.append(twin)
    optimizers = [torch.optim.SGD(m.parameters(), lr=0.05) for m in models]
    return models, optimizers


def _batch_tensors(pairs):
    x = torch.from_numpy(np.stack([p[0] for p in pairs])).permute(0, 3, 1, 2)
    y = torch.from_numpy(np.stack([p[1] for p in pairs]))
    return x.float() / 255.0, y.long()


def _max_param_diff(a, b):
    with torch.no_grad():
        return max(float((p - q).abs().max()) for p, q in zip(a.parameters(), b.parameters()))


def test_reference_dp_tests_with_torch_sgd():
    """The reference's own DP-exactness tests (test_train.py:86-130) with its own optimizer
    choice -- torch.optim.SGD over UNet.parameters() (flat-buffer views): two replicas equal
    the union batch, ragged shards too; torch-style zero_grad keeps the gradient views."""
    x, y = _batch_tensors(small_pairs(8, seed=2))
    models, optimizers = _clone_replicas(SMALL_SPEC, 2, seed=4)
    loss, count = synchronized_step(models, optimizers, [(x[:4], y[:4]), (x[4:], y[4:])])
    assert count == 8
    solo, solo_opt = _clone_replicas(SMALL_SPEC, 1, seed=4)
    solo_loss, _ = synchronized_step(solo, solo_opt, [(x, y)])
    assert abs(loss - solo_loss) <= 1e-5
    assert _max_param_diff(models[0], solo[0]) <= 1e-5
    assert _max_param_diff(models[0], models[1]) == 0.0
    x, y = _batch_tensors(small_pairs(7, seed=6))
    models, optimizers = _clone_replicas(SMALL_SPEC, 3, seed=8)
    pieces = torch.tensor_split(torch.arange(7), 3)
    loss, count = synchronized_step(models, optimizers, [(x[p], y[p]) for p in pieces])
    assert count == 7
    solo, solo_opt = _clone_replicas(SMALL_SPEC, 1, seed=8)
    solo_loss, _ = synchronized_step(solo, solo_opt, [(x, y)])
    assert abs(loss - solo_loss) <= 1e-5
    assert _max_param_diff(models[0], solo[0]) <= 1e-5
    # the SGD step moved the weights by exactly -lr * grad (the reference's optimizer semantics)
    m, (opt,) = _clone_replicas(SMALL_SPEC, 1, seed=1)
    before = [p.detach().clone() for p in m[0].parameters()]
    opt.zero_grad(set_to_none=True)  # a torch-style zero_grad must not break the gradient views
    synchronized_step(m, [opt], [(x, y)])
    moved = sum(float((p - q).abs().sum()) for p, q in zip(m[0].parameters(), before))
    assert moved > 0


def test_forward_train_mode_applies_dropout2d():
    """model.py:64-76: Dropout2d acts in train mode only; eval() forwards are deterministic."""
    spec = UNetSpec(input_size=64, base_channels=16, depth=3, dropout=0.3)
    torch.manual_seed(0)
    m = UNet(spec)
    x = torch.rand(2, 3, 64, 64)
    m.eval()
    e1, e2 = m(x), m(x)
    assert torch.equal(e1, e2)
    m.train()
    torch.manual_seed(5)
    t1 = m(x)
    torch.manual_seed(5)
    t2 = m(x)
    t3 = m(x)
    assert torch.equal(t1, t2) and not torch.equal(t1, t3) and not torch.equal(t1, e1)
    assert len(list(m.parameters())) == 2 * m.conv_layer_count()
    names = [n for n, _ in m.named_parameters()]
    assert names == list(m.state_dict().keys())


def test_gradient_overwrite_mode_equals_zero_and_accumulate():
    """ice_grad_overwrite: after the fused Adam (which then skips zeroing, lazy_zero), the next
    head + backward STORE every gradient instead of adding: bit-identical to zeroing the buffer
    and accumulating, even when the buffer holds garbage; and three fused-Adam training steps
    match a run that zeroes explicitly, bit for bit."""
    from paper_2403_13135_b200.icetrain.train import device_step
    spec = UNetSpec(dropout=0.1)
    rng = np.random.default_rng(21)
    x = torch.from_numpy(rng.integers(0, 256, (4, 256, 256, 3), dtype=np.uint8)).cuda()
    y = torch.from_numpy(rng.integers(0, 3, (4, 256, 256), dtype=np.uint8)).cuda()
    torch.manual_seed(0)
    eng = UNet(spec).engine
    grads = []
    for ow in (False, True):
        eng.grads.fill_(123.0 if ow else 0.0)  # overwrite mode must not read the old values
        eng.grads_stale = ow
        A = eng.forward(x, train=True, seed=5)
        dz = eng.head(A, y, train=True, grad_scale=1.0 / y.numel())
        eng.backward(A, dz)
        torch.cuda.synchronize()
        grads.append(eng.grad_dict())
    for k in grads[0]:
        assert torch.equal(grads[0][k], grads[1][k]), k
    params = []
    for lazy in (True, False):
        torch.manual_seed(0)
        m = UNet(spec)
        m.engine.lazy_zero = lazy
        opt = Adam(m.parameters())
        for _ in range(3):
            device_step(m, opt, x, y, 4)
        torch.cuda.synchronize()
        params.append(m.engine.params.clone())
    assert torch.equal(params[0], params[1])
