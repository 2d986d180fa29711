"""Benchmark: paper U-Net training images/s on B200 (+ auto-label Mpixel/s), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): the paper U-Net (UNetSpec(): depth 5, base 64,
124.4M params, Dropout2d 0.1) trained with Adam on synthetic 256x256 sea-ice tiles
(T-gray corpus) auto-labelled on the GPU by K1, batch 32 per GPU, bf16
compute / fp32 accumulate.  A "step" = forward + CE + backward + (N>1: bucketed NCCL
all-reduce) + Adam over one batch.  Per-step activations are GBs, far larger than the
126 MB L2, so no L2 flush is needed between steps.

  value  = N * 32 * K / (max over ranks of the CUDA-event time of K steps), inputs in HBM
  e2e    = the same through the public API synchronized_step() with pinned host batches
           copied in and the loss read back every step
  roofline = dominant kernel class of one instrumented step vs MEASURED_PEAKS bf16 sustained
  cpu_baseline = the reference CPU fp32 train step (oracle/unet_ref.py port), bounded sample
Under torchrun each rank drives one GPU (NCCL); rank 0 prints.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "U-Net train images/sec @256^2 (paper U-Net, batch 32/GPU)"
UNIT = "images/s"
BATCH = 32
SIZE = 256
CORPUS = 4224
AUTOLABEL_TILES = 100_000
WORKLOAD_CONFIG = {"workload": "paper U-Net (depth 5, base 64, dropout 0.1) train step on 4224 synthetic 256x256 "
                               "tiles, batch 32/GPU, Adam", "seq_len": None}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        # the driver-measured figures of this pool as recorded in SURVEY.md 8(d)
        return 6447.5, 1613.4, 1392.1, "measured (SURVEY.md 8(d) copy of MEASURED_PEAKS)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows)}


def _scene_chunk(args):
    from tests.fixtures import synth
    seed, count, haze, lo, hi = args
    flags = synth.haze_flags(seed, count, haze)
    return np.stack([synth.scene(seed, i, SIZE, bool(flags[i]))[0] for i in range(lo, hi)])


def _scene512_chunk(args):
    from tests.fixtures import synth
    seed, count, haze, lo, hi = args
    flags = synth.haze_flags(seed, count, haze)
    out = [synth.scene(seed, i, 512, bool(flags[i])) for i in range(lo, hi)]
    return np.stack([o[0] for o in out]), np.stack([o[1] for o in out])


def config5_bench(dev, dist, world, rank, steps: int = 10, warmup: int = 3, count: int = 64):
    """BASELINE config 5 geometry on this job's GPUs: the paper U-Net on 512 x 512 tiles
    (generate_corpus(101, 64, 0.3, size=512) labelled by K1 at 512^2), batch 16 per
    GPU, device-timed like the headline.  Returns a dict for the JSON line."""
    import multiprocessing as mp
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec
    from paper_2403_13135_b200.icetrain.train import SINGLE_GPU_BUCKET, GradBucketer, GraphedStep, device_step
    bounds = np.linspace(0, count, 9).astype(int)
    with mp.get_context("fork").Pool(8) as pool:
        parts = pool.map(_scene512_chunk, [(101, count, 0.3, int(bounds[i]), int(bounds[i + 1])) for i in range(8)])
    x_all = torch.from_numpy(np.concatenate([p[0] for p in parts])).to(dev)
    # labels by K1 at 512^2 (the multi-CTA region path, ice_autolabel_scene), timed on its own
    from paper_2403_13135_b200 import icelabel as il
    lab = il.autolabel(x_all)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(5):
        il.autolabel(x_all, out=lab)
    a1.record()
    torch.cuda.synchronize()
    al_ms = a0.elapsed_time(a1) / 5
    y_all = lab["label"].clone()
    batch = 16
    torch.manual_seed(0)
    model = UNet(UNetSpec(input_size=512), dev)
    if dist:
        dist.broadcast(model.engine.params, 0)
        model.engine.refresh_working_weights()
    opt = Adam(model.parameters(), lr=1e-3)
    bucketer = GradBucketer(model.engine, bucket_bytes=(64 << 20) if dist else SINGLE_GPU_BUCKET, optimizer=opt)
    gen = torch.Generator().manual_seed(55)
    union = batch * world
    idx = [torch.randperm(count, generator=gen)[:union][rank * batch:(rank + 1) * batch].to(dev)
           for _ in range(warmup + steps)]
    xs = [x_all[i].contiguous() for i in idx]
    ys = [y_all[i].contiguous() for i in idx]
    graphed = GraphedStep(model, opt, xs[0], ys[0], union, bucketer) if not os.environ.get("ICE_NO_GRAPH") else None
    run = (lambda i: graphed(xs[i], ys[i])) if graphed else (lambda i: device_step(model, opt, xs[i], ys[i], union, bucketer))
    for i in range(warmup):
        run(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(warmup, warmup + steps):
        run(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = union * steps / (ms / 1000.0)
    del model, opt, bucketer, graphed
    torch.cuda.empty_cache()
    return {"metric": "U-Net train images/sec @512^2 (config 5 geometry: paper U-Net, batch 16/GPU)",
            "value": round(value, 2), "unit": UNIT, "ms_per_step": round(ms / steps, 3), "steps": steps,
            "warmup": warmup, "n_gpus": world, "global_batch": union,
            "tflops": round(1622.4e9 * union / (ms / steps / 1000.0) / 1e12, 1),
            "data": "synthetic generate_corpus(101, 64, 0.3, size=512) tiles, labels by K1 on GPU (512^2 region path)",
            "autolabel_512": {"value": round(count * 512 * 512 / (al_ms / 1000.0) / 1e6, 1), "unit": "Mpixel/s",
                              "ms": round(al_ms, 3), "tiles": count,
                              "path": "ice_autolabel_scene region path: 3 x 3 cores per tile, each on a SWAR 256^2 window"}}


def config0_bench():
    """BASELINE configs[0] through the reference-facing API, on this GPU: 64 T-gray tiles ->
    icelabel.process_tile (one call per tile, as engine.run_sequential) -> icetrain
    train_distributed(pairs, UNetSpec(), TrainConfig(batch_size=8, epochs=1), devices=1).
    Reports the reference's own throughput row (samples_per_s counts the 51 training tiles of
    the epoch over total_s, which includes the per-epoch train/val evaluation, train.py:166-185)."""
    import paper_2403_13135_b200.icelabel as il
    from paper_2403_13135_b200.icelabel.types import FilterConfig, SceneRaster, Tile, get_preset
    from paper_2403_13135_b200.icetrain import TrainConfig, UNetSpec, train_distributed
    from tests.fixtures import synth
    tiles = [t for t, _ in synth.corpus(101, 64, 0.3)]
    scheme = get_preset("ross-sea-summer")
    t0 = time.perf_counter()
    results = [il.process_tile(Tile(SceneRaster(t, f"s{i}"), f"s{i}", 0, 0), FilterConfig(), scheme)
               for i, t in enumerate(tiles)]
    label_s = time.perf_counter() - t0
    assert all(r.ok for r in results)
    pairs = [(t, r.label.astype(np.int64)) for t, r in zip(tiles, results)]
    result, row = train_distributed(pairs, UNetSpec(), TrainConfig(batch_size=8, epochs=1), devices=1)
    return {"metric": "configs[0]: 64 tiles -> process_tile -> train_distributed(batch 8, 1 epoch) samples_per_s",
            "value": row["samples_per_s"], "unit": "samples/s", "row": row, "label_s": round(label_s, 3),
            "history": result.history,
            "reference_survey_probe": {"total_s": 81.05, "note": "reference CPU run of this config in the survey "
                                                                 "container (SURVEY.md 8(a) U12), not re-measured here"}}


def make_corpus(count: int, workers: int = 8) -> np.ndarray:
    """T-gray tiles generate_corpus(101, count, 0.3), in parallel."""
    import multiprocessing as mp
    bounds = np.linspace(0, count, workers + 1).astype(int)
    jobs = [(101, count, 0.3, int(bounds[i]), int(bounds[i + 1])) for i in range(workers)]
    with mp.get_context("fork").Pool(workers) as pool:
        return np.concatenate(pool.map(_scene_chunk, jobs))


def conv_flops(name, args):
    """Algorithmic (reference-nominal) FLOPs of one ice_* launch, or 0."""
    if name == "ice_conv_fprop":
        c1, c2, n, h, w, k, cout = args[1], args[3], args[4], args[5], args[6], args[7], args[10]
        kk = 27 if (k == 1 and c1 == 64 and c2 == 0 and cout <= 64) else k * k * (c1 + c2)
        return 2.0 * n * h * w * cout * kk
    if name == "ice_conv_dgrad":
        cout, n, h, w, k, c1, c2 = args[1], args[2], args[3], args[4], args[5], args[7], args[8]
        return 2.0 * n * h * w * cout * k * k * (c1 + c2)
    if name == "ice_conv_wgrad":
        c1, c2, cout, n, h, w, k = args[1], args[3], args[5], args[6], args[7], args[8], args[9]
        kk = 27 if k == 1 else k * k * (c1 + c2)
        return 2.0 * n * h * w * cout * kk
    if name == "ice_halve_fprop":  # nominal: 2x2 taps on the 2h x 2w output
        c, n, h, w, cout = args[1], args[2], args[3], args[4], args[7]
        return 2.0 * n * (2 * h) * (2 * w) * cout * 4 * c
    if name == "ice_halve_dgrad":
        cout, n, h, w, c = args[1], args[2], args[3], args[4], args[6]
        return 2.0 * n * (2 * h) * (2 * w) * cout * 4 * c
    if name == "ice_halve_wgrad":
        c, cout, n, h, w = args[1], args[3], args[4], args[5], args[6]
        return 2.0 * n * (2 * h) * (2 * w) * cout * 4 * c
    return 0.0


def instrumented_step(fn):
    """Run fn() once with per-launch CUDA events; returns {entry: (launches, ms, flops)}."""
    from paper_2403_13135_b200 import _native
    torch.cuda.synchronize()
    _native.counter.events = []
    fn()
    torch.cuda.synchronize()
    evs, _native.counter.events = _native.counter.events, None
    out = {}
    for name, args, e0, e1 in evs:
        k = out.setdefault(name, [0, 0.0, 0.0])
        k[0] += 1
        k[1] += e0.elapsed_time(e1)
        k[2] += conv_flops(name, args)
    return out


def cpu_reference_step_rate(batch: int, steps: int, warmup: int = 0):
    """Reference CPU fp32 train step (oracle/unet_ref.py restating model.py + train.py:85-120)
    on the host cores: returns (images/s, threads, seconds)."""
    from oracle import unet_ref
    from paper_2403_13135_b200.icetrain import UNetSpec
    from tests.fixtures import synth
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    spec = UNetSpec()
    torch.manual_seed(0)
    model = unet_ref.RefUNet(spec)
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    tiles = synth.corpus(101, batch, 0.3)
    x = unet_ref.images_to_input(np.stack([t for t, _ in tiles]))
    y = torch.from_numpy(np.stack([l for _, l in tiles])).long()
    for _ in range(warmup):
        unet_ref.synchronized_step([model], [opt], [(x, y)])
    t0 = time.perf_counter()
    for _ in range(steps):
        unet_ref.synchronized_step([model], [opt], [(x, y)])
    dt = time.perf_counter() - t0
    return batch * steps / dt, threads, dt


def run_reference(args, rank, world):
    """The reference arm: the reference's train step (oracle/unet_ref.py, pinned to the
    reference's own outputs) at the headline config -- paper U-Net, batch 32, torch CPU fp32
    on all host threads.  A batch-32 CPU step takes ~10-30 s, so the run is bounded to
    min(K, 2) timed steps after min(W, 1) warm-up steps (stated in the line)."""
    if rank != 0:
        return
    steps, warmup = max(1, min(args.steps, 2)), min(args.warmup, 1)
    rate, threads, dt = cpu_reference_step_rate(BATCH, steps, warmup=warmup)
    line = {"metric": METRIC, "value": round(rate, 4), "unit": UNIT, "impl": "reference", "n_gpus": 0,
            "steps": steps, "warmup": warmup, "ms_per_step": round(1000 * dt / steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (T-gray tiles, SURVEY.md 8(d))", "config": dict(WORKLOAD_CONFIG, global_batch=BATCH,
                                                                          parallelism=f"cpu{threads}"),
            "cpu_baseline": {"value": round(rate, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{steps} timed (+{warmup} warm-up) reference-equivalent synchronized_step(s) "
                                       f"(oracle/unet_ref.py) at batch {BATCH}, {threads} host threads, torch CPU fp32"},
            "e2e": {"value": round(rate, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _cv_chunk(tiles):
    import cv2
    cv2.setNumThreads(1)  # as the reference (kernels.py:18)
    from oracle import autolabel_cv
    for t in tiles:
        autolabel_cv.process_tile(t)
    return len(tiles)


def cpu_autolabel_rate(corpus: np.ndarray, per_core: int = 24):
    """Reference-algorithm CPU labeler (oracle/autolabel_cv.py: OpenCV + NumPy, the calls the
    reference's process_tile makes) on all host cores, one process per core as the
    reference's run_local (engine.py:236-325).  Returns (Mpixel/s, cores, tiles, seconds)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    n = min(len(corpus), cores * per_core)
    chunks = [corpus[i::cores][: per_core] for i in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_cv_chunk, [c[:1] for c in chunks])  # warm the workers (imports)
        t0 = time.perf_counter()
        done = sum(pool.map(_cv_chunk, chunks))
        dt = time.perf_counter() - t0
    return done * corpus.shape[1] * corpus.shape[2] / dt / 1e6, cores, done, dt


def tint_corpus(corpus: np.ndarray) -> np.ndarray:
    """T-tint: per-pixel per-channel offsets in [-12, 12] on the T-gray tiles."""
    from tests.fixtures import synth
    return np.stack([synth.tint(t, 101, i) for i, t in enumerate(corpus)])


def rand_corpus(count: int) -> np.ndarray:
    """T-rand: uniform random RGB tiles default_rng([0, i])."""
    from tests.fixtures import synth
    return np.stack([synth.random_tile(i) for i in range(count)])


def autolabel_bench(corpus_dev, n_tiles: int, reps: int):
    """K1 over n_tiles tiles (tile i = corpus[i mod len]) resident in HBM."""
    from paper_2403_13135_b200 import icelabel as il
    idx = torch.arange(n_tiles, device=corpus_dev.device) % corpus_dev.shape[0]
    tiles = corpus_dev[idx]
    out = None
    out = il.autolabel(tiles, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        il.autolabel(tiles, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del tiles
    return ms, out


def segment_bench(corpus_dev, n_tiles: int, reps: int):
    """K1s (segment only, `icelabel label`) over n_tiles resident tiles: HBM-bound, 4 B/px."""
    from paper_2403_13135_b200 import icelabel as il
    idx = torch.arange(n_tiles, device=corpus_dev.device) % corpus_dev.shape[0]
    tiles = corpus_dev[idx]
    out = il.segment_batch(tiles)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        il.segment_batch(tiles, out=out)
    e1.record()
    torch.cuda.synchronize()
    del tiles
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--corpus", type=int, default=CORPUS)
    ap.add_argument("--no-autolabel", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--no-config0", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import paper_2403_13135_b200.icelabel as il
    from paper_2403_13135_b200 import _native
    from paper_2403_13135_b200.icetrain import Adam, UNet, UNetSpec, synchronized_step
    from paper_2403_13135_b200.icetrain.train import SINGLE_GPU_BUCKET, GradBucketer, device_step

    # one GPU per rank; modulo the device count only matters for functional runs of
    # several ranks on one GPU (ICE_DIST_BACKEND=gloo), NCCL needs distinct GPUs
    local_rank %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        backend = os.environ.get("ICE_DIST_BACKEND", "nccl")
        # NCCL's init lines (ranks, channels, NVLS / NVLink transport) on stderr as evidence
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        tdist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
        dist = tdist
    _native.require_cuda()

    # ---- data: T-gray corpus, auto-labelled on the GPU (K1), resident in HBM -----------
    corpus = make_corpus(args.corpus)
    corpus_dev = torch.from_numpy(corpus).to(dev)
    labelled = il.autolabel(corpus_dev)
    labels_dev = labelled["label"]
    torch.cuda.synchronize()

    spec = UNetSpec()  # paper spec, dropout 0.1
    torch.manual_seed(0)
    model = UNet(spec, dev)
    if dist:
        dist.broadcast(model.engine.params, 0)
        model.engine.refresh_working_weights()
    opt = Adam(model.parameters(), lr=1e-3)
    # optimizer-in-backward: each gradient bucket is (all-reduced and) Adam-stepped on a side
    # stream as soon as backward completes it
    bucket_mb = int(os.environ.get("ICE_BUCKET_MB", "64" if dist else str(SINGLE_GPU_BUCKET >> 20)))
    comm_bf16 = bool(os.environ.get("ICE_COMM_BF16"))
    bucketer = GradBucketer(model.engine, bucket_bytes=bucket_mb << 20, optimizer=opt,
                            comm_dtype=torch.bfloat16 if comm_bf16 else None)
    union = BATCH * world
    gen = torch.Generator().manual_seed(1234)

    def batch_indices():
        order = torch.randperm(args.corpus, generator=gen)[:union]
        return order[rank * BATCH:(rank + 1) * BATCH].to(dev)

    batches = [batch_indices() for _ in range(args.warmup + args.steps)]
    xs = [corpus_dev[b].contiguous() for b in batches]
    ys = [labels_dev[b].contiguous() for b in batches]

    graphed = None
    if not os.environ.get("ICE_NO_GRAPH"):
        # one CUDA graph per step, the NCCL bucket all-reduces included at N > 1 (launch
        # overhead off the critical path); batches are copied into the graph's static inputs
        from paper_2403_13135_b200.icetrain.train import GraphedStep
        graphed = GraphedStep(model, opt, xs[0], ys[0], union, bucketer)

    def step(i):
        if graphed is not None:
            graphed(xs[i], ys[i])
        else:
            device_step(model, opt, xs[i], ys[i], union, bucketer)

    # ---- device-timed loop ------------------------------------------------------------
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.kernel_launches()
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for i in range(args.warmup, args.warmup + args.steps):
            step(i)
        e1.record()
        torch.cuda.synchronize()
    launches = _native.kernel_launches() - launches0
    if graphed is not None:  # replays make no host-side launches: count one eager step's kernels
        c0 = _native.kernel_launches()
        device_step(model, opt, xs[0], ys[0], union, bucketer)
        torch.cuda.synchronize()
        launches = (_native.kernel_launches() - c0) * args.steps
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    value = union * args.steps / (ms / 1000.0)

    # ---- e2e through the public API: pinned host batch in, loss out, every step --------
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    host_x = [xs[i % len(xs)].cpu().pin_memory() for i in range(e2e_steps)]
    host_y = [ys[i % len(ys)].cpu().pin_memory() for i in range(e2e_steps)]
    synchronized_step([model], [opt], [(host_x[0], host_y[0])])  # warm the path
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(e2e_steps):
        loss, total = synchronized_step([model], [opt], [(host_x[i], host_y[i])])
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = union * e2e_steps / (e2e_ms / 1000.0)
    h2d = host_x[0].numel() + host_y[0].numel()

    # ---- per-kernel breakdown of one step and the dominant kernel's roofline ----------
    breakdown = instrumented_step(lambda: device_step(model, opt, xs[args.warmup], ys[args.warmup], union, bucketer))
    step_ms = sum(v[1] for v in breakdown.values())
    dom = max(breakdown.items(), key=lambda kv: kv[1][1])
    hbm, bf16_burst, bf16_sust, peak_src = peaks()
    conv_names = [k for k in breakdown if k.startswith(("ice_conv", "ice_halve_f", "ice_halve_d", "ice_halve_w"))]
    conv_ms = sum(breakdown[k][1] for k in conv_names)
    conv_flops = sum(breakdown[k][2] for k in conv_names)
    roofline = {"bound": "tensor", "kernel": dom[0], "launches_per_step": dom[1][0],
                "achieved": round(dom[1][2] / (dom[1][1] / 1000.0) / 1e12, 2), "peak": bf16_sust,
                "unit": "TFLOP/s", "peak_source": f"{peak_src} bf16 sustained (kernel timed inside the step)",
                "traffic": None}
    roofline["frac"] = round(roofline["achieved"] / roofline["peak"], 4)
    roofline["all_convs"] = {"ms_per_step": round(conv_ms, 3), "share_of_step": round(conv_ms / step_ms, 3),
                             "achieved": round(conv_flops / (conv_ms / 1000.0) / 1e12, 2),
                             "frac": round(conv_flops / (conv_ms / 1000.0) / 1e12 / bf16_sust, 4)}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            roofline["traffic"] = json.load(open(prof_path)).get(dom[0])
        except Exception:
            pass
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3),
                   "tflops": round(v[2] / (v[1] / 1000.0) / 1e12, 1) if v[2] else None}
               for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][1])}

    # ---- auto-label throughput (secondary metric), tiles sharded over ranks ------------
    autolabel = None
    if not args.no_autolabel:
        n_tiles = AUTOLABEL_TILES // world
        al_ms, _ = autolabel_bench(corpus_dev, n_tiles, reps=2)
        if dist:
            t = torch.tensor([al_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            al_ms = float(t.item())
        px = n_tiles * world * SIZE * SIZE
        gbs = px * 7 / (al_ms / 1000.0) / 1e9
        seg_ms = segment_bench(corpus_dev, n_tiles, reps=5)
        if dist:
            t = torch.tensor([seg_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            seg_ms = float(t.item())
        seg_gbs = px * 4 / (seg_ms / 1000.0) / 1e9
        al_traffic = None
        try:
            tj = json.load(open(prof_path))
            if tj.get("ice_autolabel_bytes_per_tile"):
                al_traffic = tj["ice_autolabel_bytes_per_tile"] * n_tiles
        except Exception:
            pass
        al_compute = None  # K1's integer-pipe utilisation, from the committed ncu full capture
        try:
            for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "r0*_ncu_full_summary.json")), reverse=True):
                hit = [k for k in json.load(open(fn)) if "autolabel256" in k.get("kernel", "")]
                if hit:
                    k = hit[0]
                    num = lambda v: float(str(v).split()[0])  # noqa: E731
                    al_compute = {"bound": "int-alu", "alu_pipe_pct": num(k["alu_pipe_pct"]),
                                  "fma_pipe_pct": num(k.get("fma_pipe_pct", 0)), "dram_pct": num(k["dram_pct"]),
                                  "source": os.path.relpath(fn, ROOT) + " (ncu --set full, one K1 launch, T-gray)"}
                    break
        except Exception:
            pass
        variants = {}
        for name, make in (("t_tint", lambda: tint_corpus(corpus)), ("t_rand", lambda: rand_corpus(len(corpus)))):
            vdev = torch.from_numpy(make()).to(dev)
            v_ms, _ = autolabel_bench(vdev, n_tiles, reps=1)
            if dist:
                t = torch.tensor([v_ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                v_ms = float(t.item())
            v_gbs = px * 7 / (v_ms / 1000.0) / 1e9
            variants[name] = {"value": round(px / (v_ms / 1000.0) / 1e6, 1), "unit": "Mpixel/s", "ms": round(v_ms, 2),
                              "hbm_frac": round(v_gbs / hbm, 4)}
            del vdev
        autolabel = {"metric": "auto-label Mpixel/s (fused filter + HSV labeler, 100k 256^2 tiles)",
                     "value": round(px / (al_ms / 1000.0) / 1e6, 1), "unit": "Mpixel/s",
                     "ms": round(al_ms, 2), "tiles": n_tiles * world,
                     "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                                  "frac": round(gbs / hbm, 4), "traffic": al_traffic,
                                  "note": "7 B/px algorithmic (RGB in, filtered + label out); "
                                          "the 21x21 medians make K1 integer-ALU-bound (SWAR kernel)",
                                  "compute": al_compute},
                     "segment_only": {"metric": "label-only (K1s, icelabel label) Mpixel/s",
                                      "value": round(px / (seg_ms / 1000.0) / 1e6, 1), "unit": "Mpixel/s",
                                      "ms": round(seg_ms, 3),
                                      "roofline": {"bound": "hbm", "achieved": round(seg_gbs, 1), "peak": hbm,
                                                   "unit": "GB/s", "frac": round(seg_gbs / hbm, 4),
                                                   "traffic": None, "note": "4 B/px (RGB in, label out); a 3:1 read-dominated stream can exceed the copy-measured peak (read+write of b.copy_(a))"}},
                     "corpus": "T-gray (headline); T-tint / T-rand below (SURVEY.md 8(d)), tile i = corpus[i mod 4224]",
                     **variants}

    if autolabel is not None and rank == 0 and world == 1 and not args.no_cpu:
        try:
            rate, cores, done, dt = cpu_autolabel_rate(corpus)
            autolabel["cpu_baseline"] = {
                "value": round(rate, 3), "unit": "Mpixel/s", "cores": cores, "kind": "port",
                "sample": f"{done} T-gray tiles through oracle/autolabel_cv.py process_tile (OpenCV + NumPy, "
                          f"the reference's own calls), {cores} processes, {dt:.1f} s"}
        except Exception as exc:  # the GPU number stands without it
            autolabel["cpu_baseline"] = {"unavailable": f"{type(exc).__name__}: {exc}"}

    launch_mode = "CUDA graph per step" if graphed is not None else "eager"
    config0 = None
    if world == 1 and not args.no_config0:
        try:
            config0 = config0_bench()
        except Exception as exc:  # the headline stands without it
            config0 = {"unavailable": f"{type(exc).__name__}: {exc}"}
    config5 = None
    if not args.no_config5:
        del graphed
        torch.cuda.empty_cache()
        graphed = None
        try:
            config5 = config5_bench(dev, dist, world, rank)
        except Exception as exc:  # the headline stands without it
            config5 = {"unavailable": f"{type(exc).__name__}: {exc}"}

    # ---- CPU baseline (rank 0, N = 1 only): bounded sample of the reference step -------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, threads, dt = cpu_reference_step_rate(batch=BATCH, steps=1, warmup=0)
        cpu = {"value": round(rate, 4), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"1 reference-equivalent synchronized_step (oracle/unet_ref.py) at batch {BATCH}, torch CPU "
                         f"fp32, {threads} threads, {dt:.1f} s"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": f"synthetic (T-gray tiles generate_corpus(101, {args.corpus}, 0.3), labels by K1 on GPU)",
                "config": {**WORKLOAD_CONFIG,
                           "global_batch": union, "parallelism": f"dp{world}",
                           "grad_allreduce": (f"NCCL SUM, {bucket_mb} MB buckets, "
                                              f"{'bf16' if comm_bf16 else 'fp32'} on the wire") if world > 1 else None,
                           "l2": "per-step working set (activations, 124M params) >> 126 MB L2; no flush",
                           "launch": launch_mode},
                "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": 8, "steps": e2e_steps,
                        "api": "icetrain.synchronized_step([model], [opt], [(pinned u8 NHWC, pinned u8)])"},
                "gpu_launches": int(launches), "clocks": clocks.summary(), "roofline": roofline,
                "cpu_baseline": cpu, "autolabel": autolabel, "config0": config0, "config5": config5,
                "kernels": kernels,
                "tflops_step": round(405.6e9 * BATCH / (ms / args.steps / 1000.0) / 1e12, 1),
                "loss_last": round(loss, 4)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
