#!/usr/bin/env python
"""Benchmark: training images/sec of the batched raster fwd+bwd step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C2]

Workload (BASELINE.json configs[1], "paper default"): synthetic head avatar,
20 blendshapes, 50,176 Gaussians (UV 224), 512x512, batch 16 frames per GPU,
random-init weights perturbed per SURVEY §8d, synthetic u8 RGBA targets.  A step
is one full ``train_step`` (S/train.py:214-260): mesh frames from theta (device
rig), MLP, blend, projection, tile
binning + radix sort (one host sync), forward compositing with the fused L1
loss, the full adjoint chain, the gradient reduction (NCCL allreduce for N>1),
the multi-group Adam update and the colour-initialisation estimate.

Multi-GPU (torchrun, one process per GPU): weak scaling, 16 frames per GPU,
global batch 16*N, one NCCL allreduce of the flat gradient per step; the timed
region is max over ranks.

``--impl reference`` times the CPU reference path on the host cores (the float64
oracle port of headsplat's train_step under oracle/, all host threads) on the same
config, metric and unit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training images/sec (batched raster fwd+bwd)"
UNIT = "images/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0          # GB/s, /opt/skills/guides/B200_PROFILING.md fallback
L2_FLUSH_BYTES = 256 << 20


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


# ------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.  nvidia-smi
    writes its samples to a file (-f) from its own process: no reader thread in the
    benchmark process (a Python thread would contend for the GIL with the host-side
    kernel enqueue of the timed steps)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        import tempfile
        try:
            fd, self.path = tempfile.mkstemp(prefix="hs_clocks_", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        try:
            with open(self.path) as f:
                lines = f.read().splitlines()
            os.unlink(self.path)
        except Exception:
            lines = []
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "0x1", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ algorithmic bytes

def stage_bytes(B, N, K, H, D, W, Hh, keys, params, color_init=True, passes=6):
    """Algorithmic (ideal-fusion) DRAM bytes per launch of each stage."""
    HW = W * Hh
    rec = 48
    out = {
        "mlp_fwd": 4 * (H * D + D * D + K * D + B * (H + 4 * D + K)),
        "blend_fwd": 4 * (10 * N * K + 10 * N + B * 10 * N),
        "rig_frames": B * 1024 * 22 * 4 + 561 * 11 * 3 * 8,
        "project_fwd": B * N * (40 + rec + 4 + 4) + N * 32 + B * 1024 * 22 * 4,
        "bin_sort": keys * (12 + 8 + passes * 24 + 8),   # emit, histogram, passes, ranges
        # tile-major: count + scatter read the bbox words, scatter writes key + value,
        # the list sort reads value + depth and writes the value
        "bin_tiles": keys * (8 + 12) + B * N * 2 * (8 + 4),
        "raster_fwd": keys * (4 + rec) + B * HW * (4 + 4 + 4) + (B * N * 20 if color_init else 0),
        "raster_bwd": keys * (4 + rec) + B * HW * 8 + B * N * 36,
        # fused forward + adjoint: both key walks, targets once, no per-pixel state round trip
        "raster": 2 * keys * (4 + rec) + B * HW * 4 + B * N * 36 + (B * N * 20 if color_init else 0),
        "project_bwd": B * N * (36 + 40 + 56) + N * 32 + B * 1024 * 22 * 4,
        "blend_bwd": 4 * (B * 14 * N + 2 * 10 * N * K + 14 * N),
        "adam": 28 * params,
    }
    return out


def mufu_bound(keys_per_image, sm_mhz, value):
    """The SFU (MUFU) bound on images/s: 256 evaluations per (splat, tile) key, ~3 MUFU
    ops per evaluation, 148 SMs x 16 MUFU/clk at the measured SM clock."""
    import torch
    if not sm_mhz:
        return None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peak = sms * 16 * sm_mhz * 1e6
    per_image = 256.0 * keys_per_image * 3.0
    bound = peak / per_image
    return {"evals_per_image": 256.0 * keys_per_image, "mufu_per_eval": 3, "peak_mufu_per_s": peak,
            "bound_images_s": bound, "frac": value / bound}


# --------------------------------------------------------------- workloads

CONFIGS = {
    "C1": dict(uv=141, batch=4, size=256, desc="synthetic head avatar: 20 bases, 19,881 Gaussians, 256x256, batch 4"),
    "C2": dict(uv=224, batch=16, size=512, desc="paper default: 20 bases, 50,176 Gaussians, 512x512, batch 16"),
    # BASELINE configs[3]: global batch 128 split over the ranks (strong scaling)
    "C4": dict(uv=317, global_batch=128, size=512,
               desc="batch-sharded training: 20 bases, 100,489 Gaussians, 512x512, global batch 128"),
}


def per_rank_batch(cfg, world):
    if "batch" in cfg:
        return cfg["batch"], cfg["batch"] * world, "weak"
    gb = cfg["global_batch"]
    if gb % world:
        raise SystemExit(f"global batch {gb} does not split over {world} ranks")
    return gb // world, gb, "strong"


def make_trainer(cfg, rank=0, world=1, pg=None):
    import torch
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    B, GB, _ = per_rank_batch(cfg, world)
    # theta ~ N(0, 0.3) per frame: every frame of every rank distinct
    wl = synth.make_workload(cfg["uv"], B, cfg["size"], frames_seed=1 + rank)
    av = wl.avatar
    dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp,
                                 av.tri_index, av.barycentric)
    # mesh frames come from theta on the device (hs_rig_frames) inside every step
    tr = Trainer(dev, cfg["size"], cfg["size"], B, process_group=pg, global_batch=GB, frame_offset=B * rank,
                 rig=DeviceRig(wl.rig))
    d = {
        "thetas": torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda(),
        "targets": torch.from_numpy(wl.targets).cuda(),
        "frames": torch.from_numpy(wl.frames).cuda(),
        "cameras": torch.from_numpy(np.tile(wl.camera.packed(), (B, 1))).cuda(),
        "backgrounds": torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda(),
    }
    return tr, d, wl


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def port_step_fn(cfg, frames_per_step, workers):
    """The oracle port (float64 C restatement under oracle/) of train_step on a
    bounded sample of the workload (host cores)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from bench_support import synth
    wl = synth.make_workload(cfg["uv"], frames_per_step, cfg["size"])
    av = wl.avatar
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)
    model = O.Model(O.GSet(*(f(av.base[a]) for a in ("position", "rotation", "scale", "opacity", "color"))),
                    f(av.deltas), {k: f(v) for k, v in av.mlp.items()}, av.tri_index, f(av.barycentric))
    c = wl.camera
    cam = O.Cam(c.fx, c.fy, c.cx, c.cy, np.asarray(c.rotation, np.float64), np.asarray(c.translation, np.float64),
                c.width, c.height)
    frames = [O.Frames(m.rotation, m.quat, m.tri_vertices) for m in wl.mesh]
    state = O.State(model, cam, workers=workers)
    images = wl.targets.astype(np.float64) / 255.0

    def step():
        O.train_step(state, wl.thetas, images, frames, wl.backgrounds)
    return step, state.close


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "headsplat"))


def reference_step_fn(cfg, frames_per_step, workers):
    """The reference package's own train_step (S/train.py:214-260: numpy + numba,
    BatchRenderer two-stage schedule on ``workers`` threads) from baseline/_ref, on the
    same synthetic avatar (identical bindings, perturbations, theta, targets and
    backgrounds as the device arm's workload), mesh frames cached per sample like
    SequenceDataset.mesh_for (S/dataset.py:54-57)."""
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "hs_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from headsplat.binding import mesh_frames
    from headsplat.color_init import ColorInitState
    from headsplat.dataset import FrameSample
    from headsplat.render import Camera
    from headsplat.rig import build_head_rig, rig_evaluate
    from headsplat.scheduler import BatchRenderer
    from headsplat.train import Optimizer, TrainConfig, TrainState, init_avatar, train_step
    from bench_support import synth
    wl = synth.make_workload(cfg["uv"], frames_per_step, cfg["size"])
    av = wl.avatar
    rig = build_head_rig()
    tcfg = TrainConfig(uv_resolution=cfg["uv"], num_blendshapes=av.K, batch_size=frames_per_step, workers=workers)
    model = init_avatar(rig, tcfg)
    n = model.count
    if n != av.count:
        raise RuntimeError(f"reference binding count {n} != workload {av.count}")
    for a in ("position", "rotation", "scale", "opacity", "color"):
        getattr(model.base, a)[...] = np.asarray(av.base[a], np.float64).reshape(getattr(model.base, a).shape)
    for k, dl in enumerate(model.deltas):
        row = np.asarray(av.deltas[k], np.float64)
        dl.position[...] = row[:3 * n].reshape(n, 3)
        dl.rotation[...] = row[3 * n:7 * n].reshape(n, 4)
        dl.color[...] = row[7 * n:].reshape(n, 3)
    for k in ("w1", "b1", "w2", "b2", "w3", "b3"):
        getattr(model.mlp, k)[...] = np.asarray(av.mlp[k], np.float64)
    cam = Camera.frontal(cfg["size"])
    samples = [FrameSample(i + 1, wl.targets[i].astype(np.float64) / 255.0, np.asarray(wl.thetas[i], np.float64))
               for i in range(frames_per_step)]

    def mesh_of(sample):
        if sample.mesh is None:
            sample.mesh = mesh_frames(rig, rig_evaluate(rig, sample.theta))
        return sample.mesh
    renderer = BatchRenderer(workers)
    state = TrainState(model, Optimizer(model, tcfg), renderer, ColorInitState.create(n, 0.1), tcfg, cam)
    bgs = np.asarray(wl.backgrounds, np.float64)

    def step():
        train_step(state, samples, bgs, mesh_of)
    return step, renderer.close


def time_cpu(step_fn, cfg, frames, cores, warmup, steps):
    step, close = step_fn(cfg, frames, cores)
    try:
        for _ in range(warmup):
            step()
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            step()
            times.append(time.perf_counter() - t0)
    finally:
        close()
    return statistics.median(times), times


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_frames(cfg, world=1):
    """Frames per reference step: the config's per-GPU batch (the whole C2 step),
    capped at 16 so a step stays a bounded sample."""
    b, _, _ = per_rank_batch(cfg, world)
    return min(b, 16)


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU train_step (baseline/_ref, numba) on the
    host cores, rank 0 only; the oracle port when baseline/_ref is absent."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = host_cores()
    fps = cpu_frames(cfg)
    kind = "reference" if reference_available() else "port"
    fn = reference_step_fn if kind == "reference" else port_step_fn
    # the first reference call JIT-compiles the numba kernels: one extra untimed step
    med, _ = time_cpu(fn, cfg, fps, cores, max(1, min(args.warmup, 2)), args.steps)
    ms = 1000.0 * med
    value = fps / med
    what = ("headsplat train_step (the reference package itself, numpy + numba, baseline/_ref)" if kind == "reference"
            else "oracle train_step (float64 C port of headsplat, oracle/; baseline/_ref missing)")
    sample = (f"{what} on {fps} frames of the {args.config} workload per step, BatchRenderer with {cores} "
              f"workers, median of {args.steps} steps after warm-up")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": per_rank_batch(cfg, 1)[2], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "frames_per_step": fps},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; HS_BENCH_BACKEND=gloo lets several ranks share one GPU to
    # exercise the multi-rank code path where fewer GPUs than ranks are available
    backend = os.environ.get("HS_BENCH_BACKEND", "nccl")
    if backend == "nccl" and world > torch.cuda.device_count():
        # NCCL cannot put two ranks on one GPU: fall back to gloo (host-mediated
        # allreduce) and say so in the line rather than fail
        backend = "gloo"
        if rank == 0:
            print(f"bench: {world} ranks on {torch.cuda.device_count()} GPU(s): gloo backend", file=sys.stderr)
    dev_index = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    pg = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator / NVLS lines on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
        pg = dist.group.WORLD
    tr, d, wl = make_trainer(cfg, rank, world, pg)
    B, GB, scaling = per_rank_batch(cfg, world)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])

    clocks = ClockSampler(dev_index)
    clocks.start()                      # sampled through warm-up + timed region (>= 1 s of load)
    # warm-up: W steps (>= 3), continued until ~2 s of load so the SM clock and the
    # caching allocator have settled (a 5-step warm-up left the first timed steps ~10 %
    # slower than steady state)
    t_w = time.perf_counter()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    per = (time.perf_counter() - t_w) / max(args.warmup, 3)
    extra = torch.tensor([max(0.0, (2.0 - (time.perf_counter() - t_w)) / max(per, 1e-4))], device="cuda")
    if world > 1:                       # every rank runs the same number of steps (collectives)
        dist.all_reduce(extra, op=dist.ReduceOp.MAX)
    for _ in range(int(min(extra.item(), 5000))):
        step()
    barrier()
    # ---- device-resident timed region: K consecutive steps between one pair of events,
    # barrier + synchronize on both sides.  No L2 flush between steps: every step touches
    # ~0.4 GB (params, grads, Adam moments, records, keys, per-frame buffers), far more
    # than the 126 MB L2.  No per-stage events (their host cost would be timed).
    launches0 = tr.launches
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        step()
    e.record()
    e.synchronize()
    total_ms = s.elapsed_time(e)
    barrier()
    launches = tr.launches - launches0
    clk = clocks.stop()
    # ---- per-stage breakdown: a separate profiled run of the same steps (stages_ms)
    tr.enable_profiling(True)
    nprof = min(args.steps, 10)
    for _ in range(nprof):
        flush.fill_(1.0)
        step()
    stages = {k: v * args.steps / nprof for k, v in tr.stage_ms().items()}
    tr.enable_profiling(False)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    value = B * world * args.steps / (float(t.item()) / 1000.0)

    # ---- end-to-end through the host API (pinned H2D inputs, D2H losses) every step
    h = {k: v.cpu().numpy() for k, v in d.items()}
    # a training loop's input pipeline: each call uploads the next step's inputs on the
    # copy stream under its own compute (double-buffered), so every step of the timed
    # region still pays one batch of H2D copies and one D2H read
    hb = (h["thetas"], h["targets"], None, h["cameras"], h["backgrounds"])
    for _ in range(2):
        tr.step_from_host(*hb, prefetch=hb)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()            # host wall clock over K steps back to back (each
    for _ in range(args.steps):         # step returns after its loss read, a host sync on the
        tr.step_from_host(*hb, prefetch=hb)     # loss copy; the backward finishes under the next)
    torch.cuda.synchronize()            # the last step's backward and Adam are in the region
    e2e_ms = (time.perf_counter() - t0) * 1000.0
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = B * world * args.steps / (float(t.item()) / 1000.0)
    F = d["frames"].shape[1]

    if rank == 0:
        av = tr.av
        peak, peak_kind = load_peaks()
        sb = stage_bytes(B, av.N, av.K, av.H, av.D, tr.W, tr.H, tr.last_total, av.size,
                         passes=tr.binner.passes)
        per_step = {k: v / args.steps for k, v in stages.items()}
        kern = {k: v for k, v in per_step.items() if k in sb}
        dom = max(kern, key=kern.get)
        achieved = sb[dom] / (kern[dom] / 1000.0) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(dom)
        except Exception:
            pass
        issue = None                     # the bound that actually limits the rasterizer
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_issue.json")) as f:
                issue = json.load(f).get(dom)
        except Exception:
            pass
        step_bytes = sum(sb.values())
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "gaussians": av.N, "blendshapes": av.K, "image": tr.W,
                       "frames_per_gpu": B, "global_batch": GB, "parallelism": f"dp{world}",
                       "backend": backend if world > 1 else None,
                       "l2": "inputs larger than L2: each step touches ~0.4 GB (> 126 MB L2); the K steps are timed "
                             "back to back",
                       "keys_per_step": tr.last_total, "colour_init": "active (unvisited Gaussians)",
                       "mesh_frames": "computed from theta on the device every step (hs_rig_frames)"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                         else "fallback (B200_PROFILING.md)",
                         "algorithmic_bytes_per_launch": sb[dom],
                         "issue_bound": issue},
            "step_roofline": {"algorithmic_bytes_per_step": step_bytes,
                              "achieved_gbs": step_bytes / (ms / 1000.0) / 1e9,
                              "frac": step_bytes / (ms / 1000.0) / 1e9 / peak},
            # SURVEY 8(d)'s secondary bound: 256 pixel evaluations per key, ~3 MUFU ops each
            # (ex2 forward; ex2 + rcp in the adjoint) at 16 MUFU/clk/SM
            "mufu_bound": mufu_bound(tr.last_total / B, clk.get("sm_mhz") or clk.get("sm_max_mhz"), value / world),
            "stages_ms": {k: round(v, 4) for k, v in per_step.items()},
            "clocks": clk,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": tr.h2d_bytes(F, frames=False),
                    "d2h_bytes_per_step": tr.d2h_bytes()},
            "gpu_launches": launches,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"], port = cpu_baseline(cfg, args)
            if port is not None:
                line["cpu_port"] = port
        if world == 1 and not args.no_render:
            line["e2e_compat"] = compat_e2e(cfg, min(args.steps, 20))
    if not args.no_render:
        # render batches are independent per rank (no collective): every rank renders its
        # own 64 frames, the time is the max over ranks
        render = render_fps(args, world=world, pg=pg)
        online = online_rate(args, rank=rank, world=world, pg=pg)
        if rank == 0:
            line["render"] = render
            line["online"] = online
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(cfg, args):
    """The reference's own train_step (baseline/_ref) on the box's host cores: median
    of 3 steps after one warm-up step (which also JIT-compiles the numba kernels), on
    the config's whole per-GPU frame batch; the oracle port beside it."""
    cores = host_cores()
    fps = cpu_frames(cfg)
    out = {}
    if reference_available():
        med, ts = time_cpu(reference_step_fn, cfg, fps, cores, 1, 3)
        out = {"value": fps / med, "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"headsplat train_step (baseline/_ref, numpy + numba) on {fps} frames of the {args.config} "
                         f"workload, BatchRenderer with {cores} workers: median of 3 steps after 1 warm-up "
                         f"({', '.join(f'{t:.2f}' for t in ts)} s)"}
    med, ts = time_cpu(port_step_fn, cfg, fps, cores, 1, 3)
    port = {"value": fps / med, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle train_step (float64 C port, oracle/) on {fps} frames of the {args.config} workload, "
                      f"{cores} threads: median of 3 steps after 1 warm-up ({', '.join(f'{t:.2f}' for t in ts)} s)"}
    if not out:
        return port, None
    return out, port


def compat_e2e(cfg, steps):
    """images/s through compat.train_step -- the drop-in for S/train.py:214 with the
    reference's own argument types: FrameSample-like items holding float64 RGBA images,
    cached MeshFrames, float64 backgrounds, and the updated parameters written back into
    the caller's float64 model every step (wall clock, K steps after 2 warm-up)."""
    from types import SimpleNamespace as NS
    from bench_support import synth
    from paper_2503_12886_b200 import compat
    B, _, _ = per_rank_batch(cfg, 1)
    wl = synth.make_workload(cfg["uv"], B, cfg["size"])
    av = wl.avatar
    n = av.count
    f64 = lambda a: np.array(a, np.float64)
    base = NS(**{a: f64(av.base[a]) for a in ("position", "rotation", "scale", "opacity", "color")})
    deltas = [NS(position=f64(x[:3 * n].reshape(n, 3)), rotation=f64(x[3 * n:7 * n].reshape(n, 4)),
                 color=f64(x[7 * n:].reshape(n, 3))) for x in av.deltas]
    mlp = NS(**{k: f64(v) for k, v in av.mlp.items()})
    model = NS(base=base, deltas=deltas, mlp=mlp,
               bindings=NS(triangle_index=av.tri_index, barycentric=f64(av.barycentric)))
    tcfg = NS(lr_position=0.0008, lr_opacity=0.25, lr_scale=0.025, lr_rotation=0.005, lr_color=0.0125,
              delta_position_scale=0.05, delta_rotation_scale=0.5, delta_color_scale=0.5, lr_mlp=0.001,
              color_init=True, use_mlp=True)
    state = NS(model=model, config=tcfg, camera=wl.camera, color_state=NS(visited=np.zeros(n, bool), threshold=0.1))
    samples = [NS(index=i + 1, image=wl.targets[i].astype(np.float64) / 255.0, theta=f64(wl.thetas[i]), mesh=None)
               for i in range(B)]
    meshes = list(wl.mesh)
    mesh_of = lambda smp: meshes[smp.index - 1]
    bgs = np.asarray(wl.backgrounds, np.float64)
    for _ in range(2):
        compat.train_step(state, samples, bgs, mesh_of)
    t0 = time.perf_counter()
    for _ in range(steps):
        compat.train_step(state, samples, bgs, mesh_of)
    dt = time.perf_counter() - t0
    return {"value": B * steps / dt, "unit": UNIT, "ms_per_step": 1000.0 * dt / steps,
            "path": ("compat.train_step (reference signature; each sample's u8 target and mesh frames uploaded "
                     "once and cached on the sample; float64 model written back each step)"),
            "d2h_bytes_per_step": 4 * (14 * n + 10 * av.K * n) + 4 * int(sum(np.size(v) for v in av.mlp.values()))
            + n}


def render_fps(args, world=1, pg=None):
    """Render-only FPS (BASELINE configs[2]: 100,489 Gaussians, 512^2, batch 64 per GPU),
    device-resident; on N ranks each renders its own batch (frames are independent: no
    collective) and the time is the max over ranks, so the value is 64 N frames / time."""
    import torch
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    wl = synth.make_workload(317, 64, 512, distinct_frames=8)
    av = wl.avatar
    dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp,
                                 av.tri_index, av.barycentric)
    tr = Trainer(dev, 512, 512, 64, color_init=False, rig=DeviceRig(wl.rig))
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    fr = None                                   # mesh frames from theta on the device (unseen theta)
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (64, 1))).cuda()
    bg = torch.zeros(64, 3, device="cuda")
    out = torch.empty(64, 512, 512, 3, device="cuda")
    for _ in range(3):
        tr.render(th, fr, cams, bg, out)
    torch.cuda.synchronize()
    if pg is not None:
        torch.distributed.barrier(group=pg)
    reps = 10
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        tr.render(th, fr, cams, bg, out)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / reps
    if pg is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=pg)
        ms = float(t.item())
    return {"metric": "render FPS (rig + MLP + blend + transform + project + bin/sort + composite)",
            "value": 64 * world / (ms / 1000.0),
            "unit": "frames/s", "ms_per_batch": ms, "n_gpus": world, "scaling": "weak",
            "config": "20 bases, 100,489 Gaussians, 512x512, batch 64 per GPU",
            "keys_per_batch": tr.last_total}


def online_rate(args, frames=120, steps=200, rank=0, world=1, pg=None):
    """Online stream (BASELINE configs[4]: 10 frames/step per GPU, 512^2, pools 150 /
    1000, eta 0.7): optimisation steps/s on device-resident frame pools and the
    ingestion rate that sustains 25 steps per arriving frame (S/stream.py run_online).
    On N ranks every rank ingests the stream and trains on its slice of the same global
    draw of 10 N frames (OnlineTrainer, sharded draws); the time is the max over ranks."""
    import torch
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    from paper_2503_12886_b200.online import OnlineConfig, OnlineTrainer
    B = 10
    wl = synth.make_workload(224, frames, 512)
    av = wl.avatar
    dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp,
                                 av.tri_index, av.barycentric)
    tr = Trainer(dev, 512, 512, B, process_group=pg, global_batch=B * world, frame_offset=B * rank,
                 rig=DeviceRig(wl.rig))
    cfg = OnlineConfig(batch_size=B * world, steps_per_frame=0, check_every=10_000)
    on = OnlineTrainer(tr, wl.camera.packed(), cfg)
    for i in range(frames):
        on.ingest(i + 1, wl.targets[i], wl.thetas[i])
    for _ in range(5):
        on.optimize_once()
    torch.cuda.synchronize()
    if pg is not None:
        torch.distributed.barrier(group=pg)
    t0 = time.perf_counter()
    for _ in range(steps):
        on.optimize_once()
    on.flush()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if pg is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=pg)
        dt = float(t.item())
    sps = steps / dt
    return {"metric": f"online optimisation steps/s (device frame pools, {B} frames/step per GPU, global batch "
                      f"{B * world}, 512^2, 50,176 Gaussians)",
            "value": sps, "unit": "steps/s", "ms_per_step": 1000.0 / sps, "n_gpus": world,
            "training_frames_per_s": sps * B * world,
            "sustained_ingest_fps_at_25_steps_per_frame": sps / 25.0,
            "pooled_frames": frames,
            "timing": "host wall clock incl. draws, gathers and the per-step sync (max over ranks)"}


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: re-run this script under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous); rank 0 prints the
    line.  NCCL needs one GPU per rank; HS_BENCH_BACKEND=gloo lets N ranks share fewer
    GPUs (host-mediated allreduce) to exercise the multi-rank path."""
    import socket
    import torch
    backend = os.environ.get("HS_BENCH_BACKEND", "nccl")
    ngpu = torch.cuda.device_count()
    env = dict(os.environ)
    if backend == "nccl" and ngpu < args.gpus:
        print(f"bench: --gpus {args.gpus} with {ngpu} GPU(s) visible: ranks share GPUs over gloo", file=sys.stderr)
        env["HS_BENCH_BACKEND"] = "gloo"
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    return run_b200(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
