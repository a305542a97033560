"""On-the-fly reconstruction from a frame stream on device-resident frame pools.

B200 counterpart of S/stream.py.  The reference keeps FrameSample
objects in a local FIFO and a reservoir-sampled global pool and re-uploads nothing
only because it never leaves the host; here every pooled frame lives in HBM
(u8 RGBA image + theta in a slot of a DeviceFramePool, 1,151 slots x 1 MiB at
512^2 for the paper's 150 + 1000 pools), the bookkeeping stays on the host with the
reference's exact rule and random draws, and a step gathers its sampled slots on
the device (hs_gather_rows) -- the only per-step H2D traffic is the B slot ids and
the B background colours.  Mesh frames come from theta through the Trainer's
DeviceRig, so nothing per frame is cached on the host.

  SamplePools / process_frame / _reservoir_insert   S/stream.py:27-66
  sample_batch                                      S/stream.py:73-90
  OnlineConfig / run_online (sampling modes,        S/stream.py:93-172
    steps_per_frame, wall-clock ingestion)
  forgetting_gap                                    S/stream.py:191-197

Deviation: the reference raises on a non-finite loss at the failing step; the
device loop keeps the step losses on the device and raises the same RuntimeError
(with the step index) when they are read back -- every ``check_every`` steps and at
the end of the stream -- so the step loop has no extra host sync.
"""

from __future__ import annotations

import ctypes
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import Trainer, _p, _stream


@dataclass
class FrameRef:
    """A pooled frame: its 1-based stream index and its slot in the device pool."""
    index: int
    slot: int


@dataclass
class SamplePools:
    """S/stream.py:27-66, over FrameRefs; ``release`` is told about every frame
    that leaves both pools so its device slot can be reused."""
    local_capacity: int = 150
    global_capacity: int = 1000
    keep_evicted: bool = True
    local: deque = field(default_factory=deque)
    global_pool: list = field(default_factory=list)
    last_index: int = 0
    evictions: int = 0
    discarded: int = 0
    reservoir_inserts: int = 0
    release: object = None

    def _drop(self, ref):
        if self.release is not None:
            self.release(ref)

    def process_frame(self, sample, rng):
        if sample.index != self.last_index + 1:
            raise ValueError(f"frame index {sample.index} does not follow {self.last_index}")
        self.last_index = sample.index
        if len(self.local) >= self.local_capacity:
            evicted = self.local.popleft()
            self.evictions += 1
            if self.keep_evicted:
                self._reservoir_insert(evicted, rng)
            else:
                self.discarded += 1
                self._drop(evicted)
        self.local.append(sample)

    def _reservoir_insert(self, sample, rng):
        if len(self.global_pool) < self.global_capacity:
            self.global_pool.append(sample)
            self.reservoir_inserts += 1
            return
        k = int(rng.integers(0, sample.index))
        if k < self.global_capacity:
            displaced = self.global_pool[k]
            self.global_pool[k] = sample
            self.reservoir_inserts += 1
            self._drop(displaced)
        else:
            self._drop(sample)
        self.discarded += 1


def process_frame(sample, pools: SamplePools, rng):
    pools.process_frame(sample, rng)


def sample_batch(pools: SamplePools, batch_size: int, eta: float, rng):
    """S/stream.py:73-90: B_l = round-half-up(eta * B) uniform draws (with
    replacement) from the local FIFO, the rest from the reservoir (all local
    while the reservoir is empty)."""
    if len(pools.local) == 0:
        raise ValueError("local pool is empty" if pools.global_pool else "both pools are empty")
    b_local = int(np.floor(eta * batch_size + 0.5))
    b_global = batch_size - b_local
    if len(pools.global_pool) == 0:
        b_local, b_global = batch_size, 0
    local_items = list(pools.local)
    picks = [local_items[int(i)] for i in rng.integers(0, len(local_items), size=b_local)]
    if b_global:
        picks += [pools.global_pool[int(i)] for i in rng.integers(0, len(pools.global_pool), size=b_global)]
    return picks


def draw_step(pools: SamplePools, cfg, rng, batch_size):
    """One step's draws (S/stream.py:124-137): the sampled frames by the configured
    mode, then the per-item backgrounds, from one rng."""
    if cfg.sampling == "no_global":
        batch = sample_batch(pools, batch_size, 1.0, rng)
    elif cfg.sampling == "no_local":
        if len(pools.global_pool) == 0:
            batch = sample_batch(pools, batch_size, 1.0, rng)
        else:
            batch = [pools.global_pool[int(i)] for i in rng.integers(0, len(pools.global_pool), size=batch_size)]
    else:
        batch = sample_batch(pools, batch_size, cfg.eta, rng)
    bgs = rng.uniform(0.0, 1.0, size=(batch_size, 3))
    return batch, bgs


class DeviceFramePool:
    """HBM-resident slots of (u8 RGBA image, theta); slot 0..capacity-1."""

    def __init__(self, capacity, height, width, param_dim, device="cuda"):
        self.capacity = int(capacity)
        self.images = torch.empty(self.capacity, height, width, 4, dtype=torch.uint8, device=device)
        self.thetas = torch.empty(self.capacity, param_dim, dtype=torch.float32, device=device)
        self.free = list(range(self.capacity - 1, -1, -1))
        self.device = device

    def put(self, image, theta) -> int:
        """Upload one frame (image (H,W,4) u8 or float in [0,1], theta) into a free slot."""
        if not self.free:
            raise RuntimeError("device frame pool is full")
        slot = self.free.pop()
        img = image if torch.is_tensor(image) else torch.from_numpy(np.ascontiguousarray(_to_u8(image)))
        self.images[slot].copy_(img, non_blocking=True)
        th = theta if torch.is_tensor(theta) else torch.from_numpy(np.asarray(theta, np.float32))
        self.thetas[slot].copy_(th, non_blocking=True)
        return slot

    def release(self, ref: FrameRef):
        self.free.append(ref.slot)

    def gather(self, slots_dev, images_out, thetas_out):
        B = slots_dev.numel()
        L.call("hs_gather_rows", B, self.images[0].numel(), _p(slots_dev), _p(self.images), _p(images_out), _stream())
        L.call("hs_gather_rows", B, self.thetas.shape[1] * 4, _p(slots_dev), _p(self.thetas), _p(thetas_out),
               _stream())


def _to_u8(image):
    a = np.asarray(image)
    if a.dtype == np.uint8:
        return a
    return np.clip(np.floor(a * 255.0 + 0.5), 0, 255).astype(np.uint8)     # PNG-backed [0,1] floats


@dataclass
class OnlineConfig:
    """S/stream.py:93-101 (the TrainConfig part lives in the Trainer)."""
    batch_size: int = 10
    local_capacity: int = 150
    global_capacity: int = 1000
    eta: float = 0.7
    steps_per_frame: int = 25
    sampling: str = "full"        # "full" | "no_global" | "no_local"
    wall_clock_fps: float = 0.0   # > 0: ingest in real time instead
    seed: int = 0
    check_every: int = 64         # steps between loss read-backs


class OnlineTrainer:
    """run_online (S/stream.py:104-172) on one device Trainer holding a DeviceRig.

    ``trainer.global_batch`` must equal ``config.batch_size``; every step draws its
    batch with the reference's rule and rng order (sample_batch, then the backgrounds)
    and trains on the gathered device frames.

    Data-parallel (a Trainer with a process group, SURVEY §8e / BASELINE configs[4]):
    every rank ingests every frame into its own HBM pool and keeps identical host
    bookkeeping (same seed, same stream), draws the same GLOBAL batch, and trains on
    its slice [frame_offset, frame_offset + B) of it -- so the ranks together take
    exactly the single-process step of S/stream.py:73-90 on the whole batch, with the
    gradients summed by the Trainer's allreduce."""

    def __init__(self, trainer: Trainer, camera, config: OnlineConfig):
        if config.sampling not in ("full", "no_global", "no_local"):
            raise ValueError(f"unknown sampling mode {config.sampling!r}")
        if trainer.rig is None:
            raise ValueError("OnlineTrainer needs a Trainer with a DeviceRig (frames from theta)")
        if trainer.global_batch != config.batch_size:
            raise ValueError(f"trainer global batch {trainer.global_batch} != config.batch_size {config.batch_size}")
        if trainer.frame_offset % trainer.B or trainer.frame_offset + trainer.B > trainer.global_batch:
            raise ValueError("trainer.frame_offset must be rank * trainer.B")
        self.tr = trainer
        self.cfg = config
        self.rng = np.random.default_rng(config.seed)
        lc = 1 if config.sampling == "no_local" else config.local_capacity
        self.pool = DeviceFramePool(lc + config.global_capacity + 1, trainer.H, trainer.W, trainer.rig.param_dim,
                                    trainer.av.device)
        self.pools = SamplePools(lc, config.global_capacity, keep_evicted=config.sampling != "no_global",
                                 release=self.pool.release)
        d = trainer.av.device
        B = trainer.B
        self.cameras = torch.as_tensor(np.asarray(camera, np.float32)).reshape(-1)[:16].to(d)
        self.targets = torch.empty(B, trainer.H, trainer.W, 4, dtype=torch.uint8, device=d)
        self.thetas = torch.empty(B, trainer.rig.param_dim, dtype=torch.float32, device=d)
        self._slots_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
        self._bg_host = torch.empty(B, 3, dtype=torch.float32, pin_memory=True)
        self.slots = torch.empty(B, dtype=torch.int32, device=d)
        self.bgs = torch.empty(B, 3, dtype=torch.float32, device=d)
        self._loss_log = []            # (step, device loss row [2B+1], frame indices)
        self.log = []
        self.min_l1 = {}
        self.steps = 0
        self.processed = 0

    # ------------------------------------------------------------------ ingest
    def ingest(self, index, image, theta):
        """One arriving frame (S/stream.py:37-49): upload into a free slot, then the
        FIFO / reservoir rule (which may free the slot of a dropped frame)."""
        slot = self.pool.put(image, theta)
        self.pools.process_frame(FrameRef(int(index), slot), self.rng)
        self.processed += 1

    # -------------------------------------------------------------------- step
    def _draw(self):
        """The global batch (the reference's draws, in its order), this rank's slice of
        it and the slice's backgrounds."""
        batch, bgs = draw_step(self.pools, self.cfg, self.rng, self.tr.global_batch)
        lo = self.tr.frame_offset
        return batch, batch[lo:lo + self.tr.B], bgs[lo:lo + self.tr.B]

    def optimize_once(self):
        full, batch, bgs = self._draw()
        # the slots and backgrounds of this step (B ints + 3B floats) are the only H2D bytes
        self._slots_host.numpy()[:] = [r.slot for r in batch]
        self._bg_host.numpy()[:] = bgs
        self.slots.copy_(self._slots_host, non_blocking=True)
        self.bgs.copy_(self._bg_host, non_blocking=True)
        self.pool.gather(self.slots, self.targets, self.thetas)
        self.tr.launches += 2
        loss = self.tr.step(self.thetas, self.targets, None, self.cameras, self.bgs)
        self._loss_log.append((self.steps, loss.clone(), [r.index for r in full]))
        self.steps += 1
        if len(self._loss_log) >= self.cfg.check_every:
            self.flush()

    def flush(self):
        """Read back the queued step losses (S/stream.py:141-148 bookkeeping).  With a
        process group the ranks' rows are all-gathered first, so every rank logs the
        global batch's loss (mean of the equal-sized slices) and per-frame L1s."""
        if not self._loss_log:
            return
        rows = torch.stack([r for _, r, _ in self._loss_log])
        B = self.tr.B
        pg = self.tr.pg
        if pg is not None:
            import torch.distributed as dist
            parts = [torch.empty_like(rows) for _ in range(dist.get_world_size(pg))]
            dist.all_gather(parts, rows, group=pg)
        else:
            parts = [rows]
        parts = [p.cpu().numpy() for p in parts]
        for j, (step, _, idx) in enumerate(self._loss_log):
            loss = float(np.mean([p[j, 2 * B] for p in parts]))
            if not np.isfinite(loss):
                self._loss_log = []
                raise RuntimeError(f"non-finite loss at online step {step}")
            black = np.concatenate([p[j, B:2 * B] for p in parts])
            for i, bl in zip(idx, black):
                prev = self.min_l1.get(i)
                if prev is None or bl < prev:
                    self.min_l1[i] = float(bl)
            self.log.append({"step": step, "loss": loss})
        self._loss_log = []

    # --------------------------------------------------------------------- run
    def run(self, stream):
        """stream: iterable of (index, image, theta) with consecutive 1-based indices
        (or objects with .index/.image/.theta).  Returns the per-step loss log."""
        cfg = self.cfg
        items = ((s.index, s.image, s.theta) if hasattr(s, "image") else s for s in stream)
        if cfg.wall_clock_fps > 0:
            interval = 1.0 / cfg.wall_clock_fps
            next_due = time.perf_counter()
            for index, image, theta in items:
                while time.perf_counter() < next_due:
                    if self.pools.local:
                        self.optimize_once()
                    else:
                        time.sleep(interval / 10.0)
                self.ingest(index, image, theta)
                next_due += interval
            for _ in range(cfg.steps_per_frame):
                self.optimize_once()
        else:
            for index, image, theta in items:
                self.ingest(index, image, theta)
                for _ in range(cfg.steps_per_frame):
                    self.optimize_once()
        self.flush()
        return self.log

    def forgetting_report(self, images, thetas):
        """S/stream.py:175-188: per processed frame, the minimum black-background L1
        seen while training and the final one (batched device render, fp32)."""
        tr = self.tr
        B = tr.B
        n = min(self.processed, len(images))
        report = []
        zero = torch.zeros(B, 3, dtype=torch.float32, device=tr.av.device)
        cams = self.cameras
        for s in range(0, n, B):
            idx = list(range(s, min(n, s + B)))
            th = np.zeros((B, tr.rig.param_dim), np.float32)
            th[:len(idx)] = np.asarray([thetas[i] for i in idx], np.float32)
            img = tr.render(torch.from_numpy(th).to(tr.av.device), None, cams, zero)
            for j, i in enumerate(idx):
                a = np.asarray(images[i])
                a = a / 255.0 if a.dtype == np.uint8 else a.astype(np.float64)
                t = torch.from_numpy(a).to(tr.av.device)
                black = t[..., :3] * t[..., 3:4]
                final = float(torch.mean(torch.abs(img[j].double() - black)))
                report.append({"frame": i + 1, "min_l1": self.min_l1.get(i + 1, float("nan")), "final_l1": final})
        return report


def forgetting_gap(report, first_fraction: float = 0.25):
    """S/stream.py:191-197."""
    cut = max(1, int(len(report) * first_fraction))
    gaps = [r["final_l1"] - r["min_l1"] for r in report[:cut] if np.isfinite(r["min_l1"])]
    return float(np.mean(gaps)) if gaps else float("nan")
