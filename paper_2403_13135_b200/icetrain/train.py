"""Synchronous data-parallel U-Net training on B200s.

Mirrors icetrain.train (/root/reference/pkg/trainer/src/icetrain/train.py):
  * TrainConfig / TrainResult / TABLE_COLUMNS / BATCH_CHOICES  (train.py:25-57)
  * synchronized_step(models, optimizers, shards) -> (mean_loss, total)   (train.py:85-120)
  * train / train_distributed / throughput_table / table_csv            (train.py:188-234)

The reference runs one thread replica per "device" on the CPU and averages gradients in
Python, weighted by shard size.  Here every shard's cross-entropy gradient is pre-scaled by
1 / (union pixels), so a plain SUM over shards is exactly that weighted average:
  * local replicas (several shards on one GPU) accumulate into one gradient buffer
    (every gradient kernel accumulates);
  * across processes (one per GPU, torch.distributed/NCCL) the flat gradient buffer is
    all-reduced in buckets laid out in backward-readiness order, each bucket launched on a
    side stream as soon as backward has produced it (overlap with the rest of backward).
Every replica then applies the identical fused Adam step, so replicas never drift.
"""

from __future__ import annotations

import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from .data import train_val_split
from .model import UNet, UNetSpec, check_tile
from .optim import Adam

BATCH_CHOICES = (16, 32, 64)
TABLE_COLUMNS = ("devices", "total_s", "s_per_epoch", "samples_per_s", "speedup")


@dataclass(frozen=True)
class TrainConfig:
    batch_size: int = 32
    epochs: int = 5
    lr: float = 1e-3
    val_fraction: float = 0.2
    seed: int = 0
    device: str = "cpu"

    def __post_init__(self) -> None:
        if self.batch_size < 1:
            raise ValueError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.epochs < 1:
            raise ValueError(f"epochs must be >= 1, got {self.epochs}")
        if self.lr <= 0:
            raise ValueError(f"lr must be positive, got {self.lr}")
        if self.device not in ("cpu", "cuda"):
            raise ValueError(f"device must be cpu or cuda, got {self.device!r}")


@dataclass
class TrainResult:
    model: UNet
    spec: UNetSpec
    config: TrainConfig
    history: list = field(default_factory=list)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _as_nhwc(x: torch.Tensor, device) -> tuple:
    """Shard images -> (device tensor, float_input).  Accepts the reference's NCHW float
    in [0, 1] (train.py:63) or the GPU pipeline's NHWC uint8."""
    if x.dtype == torch.uint8:
        t = x if x.shape[-1] == 3 else x.permute(0, 2, 3, 1)
        return t.to(device, non_blocking=True).contiguous(), False
    t = x.permute(0, 2, 3, 1) if x.shape[1] == 3 and x.shape[-1] != 3 else x
    return t.to(device, torch.float32, non_blocking=True).contiguous(), True


# One process, one GPU: a single bucket, i.e. the fused Adam runs once after the backward.
# Overlapping per-bucket Adam with the backward made both contend for HBM and measured 1.3%
# slower per step on a B200 (bench ICE_BUCKET_MB sweep); with NCCL the 64 MB buckets let the
# all-reduce overlap the backward instead.
SINGLE_GPU_BUCKET = 4096 << 20


def plan_buckets(spec, bucket_bytes: int = 64 << 20):
    """Contiguous [start, stop) slices of the flat gradient buffer, in backward-readiness
    order, each closed by the layer whose gradient completes it: [(start, stop, last)]."""
    from .model import flat_layout, readiness_order
    _, by_name, numel = flat_layout(spec)
    names = readiness_order(spec)
    buckets, start, limit = [], 0, bucket_bytes // 4
    for k, name in enumerate(names):
        L = by_name[name]
        hi = L.b_off + L.cout_p
        last = k == len(names) - 1
        if hi - start >= limit or last:
            buckets.append((start, numel if last else hi, name))
            start = hi
    return buckets


class GradBucketer:
    """Bucketed SUM all-reduce of the flat gradient buffer, overlapped with backward,
    optionally fused with the optimizer (optimizer-in-backward).

    Buckets are contiguous slices of UNetEngine.grads (laid out in readiness order).  When
    backward reports the layer that completes a bucket, the bucket is all-reduced (under
    torch.distributed, NCCL over NVLink) on a COMM stream that waits on an event of the
    compute stream; if an optimizer is attached, the bucket's fused Adam runs on a separate
    OPT stream that waits on the bucket's all-reduce event -- so Adam(k) overlaps the
    all-reduce of bucket k+1, and both overlap the tensor-bound rest of backward.  `finish()`
    re-derives the halving-conv weight slabs and joins both streams back into the compute
    stream.  Every step is stream-ordered (no host sync), so a whole step -- collectives
    included -- can be captured in one CUDA graph (GraphedStep).

    comm_dtype=torch.bfloat16 sends each pre-scaled fp32 bucket as bf16 (half the NVLink
    bytes, 249 MB/step instead of 497 MB at the paper spec); the sum is cast back to fp32 on
    every rank identically, so replicas stay bit-identical.  force_collective issues the
    collective even in a 1-rank group (tests the captured NCCL path on one GPU).
    Works on CPU tensors too (gloo, synchronously, no Adam)."""

    def __init__(self, engine, bucket_bytes: int = 64 << 20, group=None, optimizer=None, comm_dtype=None,
                 force_collective: bool = False):
        self.engine, self.group, self.optimizer = engine, group, optimizer
        self.cuda = engine.grads.is_cuda
        self.comm_dtype = comm_dtype
        self.force = force_collective
        dev = engine.grads.device
        self.comm_stream = torch.cuda.Stream(device=dev) if self.cuda else None
        self.opt_stream = torch.cuda.Stream(device=dev) if self.cuda and optimizer is not None else None
        self.buckets = plan_buckets(engine.spec, bucket_bytes)
        self.by_last = {}
        for b in self.buckets:
            self.by_last.setdefault(b[2], []).append(b)
        self._wire = None
        self._comm_used = False
        if self.cuda and comm_dtype is not None:
            longest = max(stop - start for start, stop, _ in self.buckets)
            self._wire = torch.empty(longest, dtype=comm_dtype, device=dev)

    def _collective(self) -> bool:
        dist = _dist()
        return dist is not None and (self.force or dist.get_world_size() > 1)

    def begin(self) -> None:
        if self.optimizer is not None:
            self.optimizer.begin_overlapped_step()

    def on_layer_done(self, name: str) -> None:
        dist = _dist()
        if self.cuda and name in self.by_last and hasattr(self.engine, "flush_deferred"):
            self.engine.flush_deferred()  # the bucket's deferred gradient finishers, first
        for start, stop, _ in self.by_last.get(name, ()):
            g = self.engine.grads[start:stop]
            if not self.cuda:
                dist.all_reduce(g, group=self.group)
                continue
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            done = None
            if self._collective():
                self._comm_used = True
                with torch.cuda.stream(self.comm_stream):
                    self.comm_stream.wait_event(ev)
                    if self._wire is None:
                        dist.all_reduce(g, group=self.group)
                    else:  # bf16 on the wire, fp32 sum back into the gradient buffer
                        w = self._wire[: stop - start]
                        w.copy_(g)
                        dist.all_reduce(w, group=self.group)
                        g.copy_(w)
                    done = torch.cuda.Event()
                    done.record(self.comm_stream)
            if self.optimizer is not None:
                with torch.cuda.stream(self.opt_stream):
                    self.opt_stream.wait_event(done if done is not None else ev)
                    self.optimizer.step_slice(self.engine, start, stop, self.opt_stream)

    def finish(self) -> None:
        if not self.cuda:
            return
        cur = torch.cuda.current_stream()
        # join only streams that carry this step's work (a capture must not wait on a stream
        # with no captured work)
        comm, self._comm_used = self._comm_used, False
        if self.optimizer is not None:
            if comm:
                self.opt_stream.wait_stream(self.comm_stream)
            self.engine.prep_halves(self.opt_stream)
            cur.wait_stream(self.opt_stream)
        if comm:
            cur.wait_stream(self.comm_stream)


def device_step(model, optimizer, x, y, union_count: int, bucketer=None) -> None:
    """One data-parallel step with everything already on the device and no host sync:
    forward, fused CE head, backward (bucketed gradient all-reduce overlapped when a
    bucketer is given), fused Adam.  x: u8 NHWC [n, S, S, 3], y: u8 [n, S, S].
    The step's loss sum / hit count accumulate in model.engine.stats."""
    engine = model.engine
    hw = x.shape[1] * x.shape[2]
    # dropout masks: per-rank seed + the engine's device step counter (graph-replay safe)
    dist = _dist()
    A = engine.forward(x, train=model.training, seed=1 + (dist.get_rank() if dist else 0))
    dz = engine.head(A, y, train=True, grad_scale=1.0 / (union_count * hw))
    fused = bucketer is not None and bucketer.optimizer is optimizer
    if fused:
        bucketer.begin()
    engine.backward(A, dz, on_layer_done=bucketer.on_layer_done if bucketer else None)
    if bucketer:
        bucketer.finish()
    if not fused:
        optimizer.step()


class GraphedStep:
    """A whole device_step captured once as a CUDA graph and replayed (single process):
    ~140 kernel launches (+ the optimizer-in-backward side stream) become one graph launch.
    Inputs are copied into static device buffers before each replay; the Adam step count and
    dropout seeds advance through the engine's device step counter, so replays are real
    consecutive training steps."""

    def __init__(self, model, optimizer, x, y, union_count: int, bucketer=None, warmup: int = 2,
                 zero_stats: bool = False):
        self.model, self.optimizer = model, optimizer
        self.x = x.clone()
        self.y = y.clone()
        self.union, self.bucketer = union_count, bucketer
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                device_step(model, optimizer, self.x, self.y, union_count, bucketer)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            if zero_stats:  # the replay's loss sum / hit count start from zero
                model.engine.stats.zero_()
            device_step(model, optimizer, self.x, self.y, union_count, bucketer)
        # the capture itself did not run the step: undo its host-side step bookkeeping
        optimizer.step_count -= 1

    def __call__(self, x=None, y=None) -> None:
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        if y is not None:
            self.y.copy_(y, non_blocking=True)
        self.graph.replay()
        self.optimizer.step_count += 1


def synchronized_step(models: list, optimizers: list, shards: list) -> tuple:
    """One collective training step (train.py:85-120).  ``shards[i]`` is replica i's
    ``(x, y)`` slice of the union batch (may be empty).  Under torch.distributed each rank
    passes its own shard(s) and the union spans all ranks.  Returns the union-batch mean
    loss and the union sample count."""
    engine = models[0].engine
    device = engine.device
    counts = [len(x) for x, _ in shards]
    local = sum(counts)
    # union sample count and pixels per tile (tiles of one corpus share a shape; a rank with
    # an empty shard learns the tile size from the others)
    local_hw = next((x.shape[1] * x.shape[2] if x.shape[-1] == 3 else x.shape[2] * x.shape[3]
                     for x, _ in shards if len(x)), 0)
    dist = _dist()
    if dist is not None:
        t = torch.tensor([float(local), float(local * local_hw)], dtype=torch.float64, device=device)
        dist.all_reduce(t)
        total, pixels = int(t[0].item()), int(t[1].item())
    else:
        total, pixels = local, local * local_hw
    if total == 0:
        raise ValueError("synchronized step got only empty shards")
    A = None
    rank_seed = 1 + 1009 * (dist.get_rank() if dist is not None else 0)
    bucketer = None
    fused = len(models) == 1 and isinstance(optimizers[0], Adam)
    if fused or (dist is not None and dist.get_world_size() > 1):
        key = (id(optimizers[0]) if fused else None)
        bucketer = getattr(engine, "_bucketer", None)
        if bucketer is None or getattr(bucketer, "_key", None) != key:
            bucketer = GradBucketer(engine, bucket_bytes=(64 << 20) if dist else SINGLE_GPU_BUCKET,
                                    optimizer=optimizers[0] if fused else None)
            bucketer._key = key
            engine._bucketer = bucketer
        if fused:
            bucketer.begin()
    live = [(k, s) for k, s in enumerate(shards) if counts[k] > 0]
    for idx, (k, (x, y)) in enumerate(live):
        xin, is_float = _as_nhwc(x, device)
        A = engine.forward(xin, train=models[0].training, seed=rank_seed + k, float_input=is_float)
        if idx == 0:
            A.stats.zero_()
        A.labels.copy_(y.to(device, non_blocking=True), non_blocking=True)
        dz = engine.head(A, A.labels, train=True, grad_scale=1.0 / pixels)
        last = idx == len(live) - 1
        engine.backward(A, dz, on_layer_done=bucketer.on_layer_done if (bucketer and last) else None)
    if A is None:  # this rank had no samples: contribute zeros
        engine.stats.zero_()
        if bucketer:
            for _, _, last in bucketer.buckets:
                bucketer.on_layer_done(last)
    if bucketer:
        bucketer.finish()
    stats = engine.stats
    if dist is not None:
        dist.all_reduce(stats)
    mean_loss = float(stats[0].item()) / pixels
    if not fused:
        for m in models[1:]:
            m.engine.grads.copy_(engine.grads)
        for m, opt in zip(models, optimizers):
            if isinstance(opt, Adam):
                opt.step()
            else:  # any torch optimizer over m.parameters() (flat-buffer views): step in place,
                # then refresh the bf16 working weights and clear the accumulating gradients
                m.parameters().attach_grads()
                opt.step()
                m.engine.advance_step()
                m.engine.refresh_working_weights()
                m.engine.zero_grad()
    return mean_loss, total


def rank_shards(union: torch.Tensor, n_replicas: int, rank: int, local: int) -> tuple:
    """This process's replicas' slices of a union batch: torch.tensor_split of the union into
    n_replicas pieces exactly as the reference (train.py:161-163), replicas numbered
    rank-major (rank r owns pieces [r * local, (r + 1) * local))."""
    return torch.tensor_split(union, n_replicas)[rank * local:(rank + 1) * local]


def _validate_pairs(pairs: list, spec: UNetSpec) -> None:
    if not pairs:
        raise ValueError("training corpus is empty")
    step = 2 ** spec.depth
    shape = pairs[0][0].shape
    for i, (tile, mask) in enumerate(pairs):
        if tile.shape != shape or mask.shape != shape[:2]:
            raise ValueError(f"pair {i}: shape {tile.shape}/{mask.shape} does "
                             f"not match the corpus shape {shape}")
        if mask.min() < 0 or mask.max() >= spec.classes:
            raise ValueError(f"pair {i}: class index out of range for {spec.classes} classes")
    if shape[2] != spec.in_channels or shape[0] % step or shape[1] % step:
        raise ValueError(f"tile shape {shape} does not fit the model "
                         f"(needs {spec.in_channels} channels, dims divisible by {step})")
    check_tile(shape[0], shape[1], spec.depth)  # the B200 engine's own limit, raised up front


def _device_corpus(pairs: list, device):
    """uint8 NHWC images and uint8 labels, resident in HBM (the reference keeps float32
    NCHW copies in host RAM, train.py:60-65)."""
    x = torch.from_numpy(np.ascontiguousarray(np.stack([p[0] for p in pairs]))).to(device)
    y = torch.from_numpy(np.ascontiguousarray(np.stack([p[1] for p in pairs]).astype(np.uint8))).to(device)
    return x, y


def evaluate(model: UNet, x: torch.Tensor, y: torch.Tensor, batch: int) -> tuple:
    """(mean loss, pixel accuracy) in eval mode (train.py:123-134)."""
    eng = model.engine
    loss_sum, correct, pixels = 0.0, 0.0, 0
    for start in range(0, len(x), batch):
        xb, yb = x[start:start + batch], y[start:start + batch]
        A = eng.forward(xb, train=False)
        A.stats.zero_()
        eng.head(A, yb.contiguous(), train=False)
        st = A.stats.tolist()
        loss_sum += st[0]
        correct += st[1]
        pixels += yb.numel()
    return loss_sum / pixels, correct / pixels


def _validate_device(x, y, spec: UNetSpec) -> None:
    """_validate_pairs for a device corpus: u8 [n, h, w, 3] tiles, [n, h, w] class ids."""
    if x.ndim != 4 or len(x) == 0:
        raise ValueError("training corpus is empty" if x.ndim == 4 else f"expected (n, h, w, 3) tiles, got {tuple(x.shape)}")
    if x.dtype != torch.uint8 or not x.is_cuda:
        raise ValueError("device corpus tiles must be a uint8 CUDA tensor")
    if tuple(y.shape) != tuple(x.shape[:3]):
        raise ValueError(f"labels {tuple(y.shape)} do not match tiles {tuple(x.shape)}")
    step = 2 ** spec.depth
    if x.shape[3] != spec.in_channels or x.shape[1] % step or x.shape[2] % step:
        raise ValueError(f"tile shape {tuple(x.shape[1:])} does not fit the model "
                         f"(needs {spec.in_channels} channels, dims divisible by {step})")
    if int(y.max()) >= spec.classes or (y.dtype.is_signed and int(y.min()) < 0):
        raise ValueError(f"class index out of range for {spec.classes} classes")
    check_tile(x.shape[1], x.shape[2], spec.depth)


def _fit(pairs, spec: UNetSpec, config: TrainConfig, replicas: int, device_corpus=None) -> tuple:
    """train.py:137-185.  `pairs` (host (tile, mask) list, the reference's input) or
    `device_corpus` = (u8 [n, h, w, 3], [n, h, w]) already resident in HBM (K1 output)."""
    device = torch.device("cuda", torch.cuda.current_device())
    if device_corpus is None:
        _validate_pairs(pairs, spec)
    else:
        _validate_device(*device_corpus, spec)
    torch.manual_seed(config.seed)
    if device_corpus is None:
        train_pairs, val_pairs = train_val_split(pairs, config.val_fraction, config.seed)
        x_train, y_train = _device_corpus(train_pairs, device)
        x_val, y_val = _device_corpus(val_pairs, device) if val_pairs else (None, None)
    else:  # the same seeded split, on indices; the tiles never leave the GPU
        x_all, y_all = device_corpus
        tr, va = train_val_split(list(range(len(x_all))), config.val_fraction, config.seed)
        pick = lambda t, idx: t[torch.as_tensor(idx, device=t.device)].contiguous()  # noqa: E731
        x_train, y_train = pick(x_all, tr), pick(y_all, tr).to(torch.uint8)
        x_val, y_val = (pick(x_all, va), pick(y_all, va).to(torch.uint8)) if va else (None, None)
    dist = _dist()
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1

    local = replicas if dist is None else 1
    models = [UNet(spec, device)]
    for _ in range(local - 1):
        twin = UNet(spec, device)
        twin.load_state_dict(models[0].state_dict())
        models.append(twin)
    if dist is not None:  # parameter broadcast from rank 0 (train.py:144-148)
        dist.broadcast(models[0].engine.params, 0)
        models[0].engine.refresh_working_weights()
    optimizers = [Adam(m.parameters(), lr=config.lr) for m in models]

    shuffler = torch.Generator().manual_seed(config.seed)
    history = []
    n_replicas = local * world
    torch.cuda.synchronize()
    started = time.perf_counter()
    for epoch in range(config.epochs):
        for m in models:
            m.train()
        order = torch.randperm(len(x_train), generator=shuffler)
        span = config.batch_size * n_replicas
        loss_sum, seen = 0.0, 0
        for start in range(0, len(order), span):
            mine = rank_shards(order[start:start + span], n_replicas, rank, local)
            shards = [(x_train[p.to(device)], y_train[p.to(device)]) for p in mine]
            loss, count = synchronized_step(models, optimizers, shards)
            loss_sum += loss * count
            seen += count
        entry = {"epoch": epoch, "train_loss": loss_sum / seen}
        entry["train_acc"] = evaluate(models[0], x_train, y_train, config.batch_size)[1]
        if x_val is not None:
            entry["val_loss"], entry["val_acc"] = evaluate(models[0], x_val, y_val, config.batch_size)
        history.append(entry)
    torch.cuda.synchronize()
    total_s = time.perf_counter() - started
    result = TrainResult(models[0], spec, config, history)
    row = {
        "devices": n_replicas,
        "total_s": round(total_s, 3),
        "s_per_epoch": round(total_s / config.epochs, 3),
        "samples_per_s": round(config.epochs * len(x_train) / total_s, 3) if total_s > 0 else 0.0,
        "speedup": 1.0,
    }
    return result, row


def train(pairs: list, spec: UNetSpec, config: TrainConfig) -> TrainResult:
    result, _ = _fit(pairs, spec, config, replicas=1)
    return result


def train_device(tiles, labels, spec: UNetSpec, config: TrainConfig, devices: int = 1) -> tuple:
    """train / train_distributed on a corpus already in HBM -- e.g. icelabel.autolabel's
    labels of icelabel.tiling.split_scene_device tiles (K1 -> training
    with no host round trip).  Same split, shuffle, steps and history as train() on the
    equivalent host pairs.  Returns (TrainResult, throughput row)."""
    return _fit(None, spec, config, _available_replicas(config, devices), device_corpus=(tiles, labels))


def _available_replicas(config: TrainConfig, requested: int) -> int:
    if requested < 1:
        raise ValueError(f"devices must be >= 1, got {requested}")
    dist = _dist()
    if dist is not None and requested not in (1, dist.get_world_size()):
        warnings.warn(f"requested {requested} devices but the process group has "
                      f"{dist.get_world_size()} ranks; using the process group")
    return requested


def train_distributed(pairs: list, spec: UNetSpec, config: TrainConfig, devices: int = 1) -> tuple:
    """Synchronous data-parallel training.  Under torch.distributed (one process per GPU,
    launched by torchrun) the replicas are the ranks; otherwise ``devices`` lockstep
    replicas share the current GPU (same math, for equivalence testing)."""
    replicas = _available_replicas(config, devices)
    return _fit(pairs, spec, config, replicas)


def throughput_table(pairs: list, spec: UNetSpec, config: TrainConfig, device_counts: tuple = (1, 2)) -> list:
    if not device_counts:
        raise ValueError("device_counts must list at least one count")
    rows = []
    for n in device_counts:
        _, row = train_distributed(pairs, spec, config, devices=n)
        rows.append(row)
    base = rows[0]["samples_per_s"]
    for row in rows:
        row["speedup"] = round(row["samples_per_s"] / base, 3) if base > 0 else 1.0
    return rows


def table_csv(rows: list) -> str:
    lines = [",".join(TABLE_COLUMNS)]
    for row in rows:
        lines.append(",".join(str(row[c]) for c in TABLE_COLUMNS))
    return "\n".join(lines) + "\n"
